# round-2 evidence: gpu tests, smoke, bench lines for every config (+ the wave variant and the
# reference arm), the ncu launch list, one full ncu capture of the dominant kernels, the
# whole-step DRAM traffic (ncu app-range replay, steady state over 8 calls), CTA timelines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py --check > gpurun_out/r02_bench_c2.json 2>gpurun_out/bench_c2.err; echo "bench c2 rc=$?"; tail -c 300 gpurun_out/r02_bench_c2.json
for X in "--config c1" "--config c3" "--config c4" "--config c5 --steps 20 --warmup 3" "--frames-per-step 8" "--guides f16" "--config c4 --guides f16" "--modulated" "--variant 2"; do
  N=$(echo $X | tr -d ' -' | sed 's/steps.*//'); timeout -s KILL 900 python bench.py $X --no-cpu-baseline --check > gpurun_out/r02_bench_$N.json 2>gpurun_out/bench_$N.err; echo "bench $X rc=$?"; tail -1 gpurun_out/r02_bench_$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_frame']*1e3,2), 'us/frame', round(d['value']), d['unit'], 'frac', round(d['step_roofline']['frac'],3), 'parity', d.get('parity',{}).get('max_ratio'), d.get('parity',{}).get('violations'))"
done
timeout -s KILL 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02_bench_reference.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/r02_bench_reference.json
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"^k_" -s 12 -c 12 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"k_fit_ws|k_apply_ws|k_blur_solve_tile" -s 6 -c 3 -o gpurun_out/r02_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout -s KILL 600 ncu --replay-mode app-range --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r02_step_traffic_staged8.csv python tools/step_traffic.py staged 8 > gpurun_out/ncu_step_staged8.log 2>&1; echo "ncu step staged8 rc=$?"
timeout -s KILL 600 ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r02_step_traffic_staged.csv python tools/step_traffic.py staged 1 > gpurun_out/ncu_step_staged.log 2>&1; echo "ncu step staged rc=$?"
(timeout -s KILL 60 tools/t_timeline; timeout -s KILL 60 tools/t_timeline early) > gpurun_out/r02_timeline.txt 2>&1; cat gpurun_out/r02_timeline.txt | grep graph
