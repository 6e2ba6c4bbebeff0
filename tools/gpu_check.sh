# quick GPU validation: gpu tests, smoke, the c2 bench line with a parity check
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --check --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_frame']*1e3,2), 'us/frame', round(d['value']), d['unit'], 'frac', round(d['step_roofline']['frac'],3), d['kernel_us'], 'parity', d.get('parity',{}).get('max_ratio'), d.get('parity',{}).get('violations'))"
