#!/bin/bash
# build variants of the FIT/APPLY kernel microbenchmark (run from the repo root)
set -e
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude"
nvcc $F -o tools/ubf_base tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=2 -DFLR_FIT_MAXW=14 -o tools/ubf_s2w14 tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=2 -DFLR_FIT_MAXW=16 -o tools/ubf_s2w16 tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=3 -DFLR_FIT_MAXW=12 -o tools/ubf_s3w12 tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=4 -DFLR_FIT_MAXW=8 -o tools/ubf_s4w8 tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=2 -DFLR_FIT_MAXW=8 -o tools/ubf_s2w8 tools/ubench_fit.cu &
wait
