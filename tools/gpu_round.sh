# round deliverables: tests, smoke, bench lines (+reference arm), ncu launch lists + full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --check > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_c2.log
for X in "--guides f16" "--config c4" "--config c4 --guides f16" "--config c5" "--frames-per-step 8" "--modulated" "--config c3" "--config c1"; do
  N=$(echo $X | tr -d ' -'); timeout -s KILL 600 python bench.py $X --no-cpu-baseline --check --steps 500 > gpurun_out/bench_$N.log 2>&1; echo "bench $X rc=$?"; tail -1 gpurun_out/bench_$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_frame']*1e3,2), 'us/frame', round(d['value']), d['unit'], 'frac', round(d['step_roofline']['frac'],3), 'parity', d.get('parity',{}).get('max_ratio'), d.get('parity',{}).get('violations'))"
done
timeout -s KILL 600 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.log
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"^k_" -s 12 -c 12 --csv --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:"^k_" -s 12 -c 12 --csv --log-file gpurun_out/r01_launches_warm.csv $CMD > gpurun_out/ncu_list_warm.log 2>&1; echo "ncu warm list rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"k_fit_ws|k_apply_ws|k_blur_solve_tile" -s 6 -c 3 -o gpurun_out/r01_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout -s KILL 60 tools/t_timeline > gpurun_out/timeline.txt 2>&1; cat gpurun_out/timeline.txt
