#!/bin/bash
# build variants of the FIT/APPLY kernel microbenchmark (run from the repo root)
set -e
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude"
nvcc $F -o tools/ubf_base tools/ubench_fit.cu &
nvcc $F -DFLR_DBG_NOCOMPUTE -o tools/ubf_nocomp tools/ubench_fit.cu &
nvcc $F -DFLR_DBG_NOSTORE -o tools/ubf_nostore tools/ubench_fit.cu &
nvcc $F -DFLR_DBG_NOFENCE -o tools/ubf_nofence tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=2 -DFLR_FIT_MAXW=12 -o tools/ubf_s2w12 tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=4 -DFLR_FIT_MAXW=8 -o tools/ubf_s4w8 tools/ubench_fit.cu &
nvcc $F -DFLR_FIT_S=6 -DFLR_FIT_MAXW=8 -o tools/ubf_s6w8 tools/ubench_fit.cu &
wait
