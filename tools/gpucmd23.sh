mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --import-source on --cache-control none --clock-control none -k 'regex:k_fit_ws' -c 2 -f -o gpurun_out/prof_ws python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step 8 --steps 3 --warmup 3 --no-graph > gpurun_out/ncu_ws.log 2>&1; tail -1 gpurun_out/ncu_ws.log
