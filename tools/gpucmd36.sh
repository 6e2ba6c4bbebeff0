mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_tikhonov_gpu.py tests/test_modulated_gpu.py -q -rf > gpurun_out/pt_new.log 2>&1; echo "new rc=$?"; tail -15 gpurun_out/pt_new.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for F in 1 8; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --frames-per-step $F --steps 1000 > gpurun_out/b.log 2>&1; echo -n "frames $F: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v/$F,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log
done
