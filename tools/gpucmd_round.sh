# round deliverables: tests, smoke, bench (+reference arm), ncu launch lists + full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv 2>&1
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_default.log
timeout -s KILL 600 python bench.py --frames-per-step 8 --no-cpu-baseline > gpurun_out/bench_f8.log 2>&1; echo "bench f8 rc=$?"; tail -c 600 gpurun_out/bench_f8.log
timeout -s KILL 600 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 800 gpurun_out/bench_ref.log
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"^k_" -s 12 -c 12 --csv --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:"^k_" -s 12 -c 12 --csv --log-file gpurun_out/r01_launches_warm.csv $CMD > gpurun_out/ncu_list_warm.log 2>&1; echo "ncu warm list rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"k_fit_ws|k_apply_ws|k_blur_solve_tile" -s 6 -c 3 -o gpurun_out/r01_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
