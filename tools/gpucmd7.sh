mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_parity_gpu.py -q -rf -x -k "not sweep_q" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for V in 1 2; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 3 --variant $V > gpurun_out/bench_v$V.log 2>&1; echo "bench v$V rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_v$V.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/bench_v$V.log
done
