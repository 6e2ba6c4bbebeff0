mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fit_stream|k_blur_solve|k_apply_stream" -s 3 -c 3 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
