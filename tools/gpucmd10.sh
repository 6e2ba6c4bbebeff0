mkdir -p gpurun_out
for L in 35 80 120 400; do for F in 1 4; do
FLR_FUSED_LAG=$L timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --variant 2 --frames-per-step $F --steps 100 > gpurun_out/b.log 2>&1; echo -n "lag $L frames $F: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,1), 'us/frame', round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log
done; done
