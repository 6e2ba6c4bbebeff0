mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_parity_gpu.py -q -rf -x -k "not sweep_q" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for E in "" "FLR_NO_PDL=1"; do
env $E timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 3 --variant 1 > gpurun_out/bench_v1.log 2>&1; echo "bench [$E] rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_v1.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/bench_v1.log
done
