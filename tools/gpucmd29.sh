mkdir -p gpurun_out
run() { timeout -s KILL 300 env "$@" python bench.py --no-cpu-baseline --e2e-steps 1 --steps 1000 > gpurun_out/b.log 2>&1; echo -n "$*: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log; }
run FLR_FIT_GPOL=0 FLR_APPLY_REV=1
run FLR_FIT_GPOL=0 FLR_APPLY_REV=1 FLR_MOM_POL=2
run FLR_FIT_GPOL=0 FLR_APPLY_REV=1 FLR_MOM_POL=2 FLR_K2_POL=0
for P in 1 2 3 4; do for R in 0 1; do run FLR_FIT_GPOL=$P FLR_APPLY_REV=$R FLR_MOM_POL=2 FLR_K2_POL=0; done; done
run FLR_FIT_GPOL=3 FLR_APPLY_REV=1 FLR_MOM_POL=1 FLR_K2_POL=0
run FLR_FIT_GPOL=2 FLR_APPLY_REV=1 FLR_MOM_POL=1 FLR_K2_POL=0
