mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_parity_gpu.py -q -rf -x -k "variants or fused or c1 or c2 or c4" > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_fused.log
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernel_us'], d['roofline'], d['step_roofline']['frac'], d['clocks'], d['e2e'])" || tail -5 gpurun_out/bench.log
