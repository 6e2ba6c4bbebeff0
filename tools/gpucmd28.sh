mkdir -p gpurun_out
run() { timeout -s KILL 300 env "$@" python bench.py --no-cpu-baseline --e2e-steps 1 --steps 1000 > gpurun_out/b.log 2>&1; echo -n "$*: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log; }
for P in 0 1 2; do for R in 0 1; do run FLR_FIT_GPOL=$P FLR_APPLY_REV=$R; done; done
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph"
for P in 0 2; do
FLR_FIT_GPOL=$P FLR_APPLY_REV=1 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:"^k_" -s 12 -c 12 --csv --log-file gpurun_out/l2exp_p$P.csv $CMD > /dev/null 2>&1; echo "ncu $P rc=$?"
done
