mkdir -p gpurun_out
for F in 1 8; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step $F --steps 300 > gpurun_out/b.log 2>&1; echo -n "frames $F: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,1), 'us/frame', {k: round(v/$F,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k 'regex:^k_' -c 40 --csv --log-file gpurun_out/warm$F.csv python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step $F --steps 4 --warmup 4 --no-graph > gpurun_out/ncu_w$F.log 2>&1
done
