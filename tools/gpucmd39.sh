run() { timeout -s KILL 300 env "$@" python bench.py --no-cpu-baseline --e2e-steps 1 --steps 2000 > gpurun_out/b.log 2>&1; echo -n "$*: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log; }
mkdir -p gpurun_out
for i in 1 2; do run FLR_X=0; run FLR_APPLY_NSUB=4; run FLR_APPLY_NSUB=1; done
timeout -s KILL 60 tools/t_timeline
