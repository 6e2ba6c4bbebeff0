mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
run() { timeout -s KILL 300 env "$@" python bench.py --no-cpu-baseline --e2e-steps 1 --steps 2000 > gpurun_out/b.log 2>&1; echo -n "$*: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log; }
for i in 1 2; do run FLR_X=0; run FLR_STATIC_ITEMS=1; run FLR_WAVE=1; done
run FLR_X=0 python bench.py --frames-per-step 8 2>/dev/null | true
