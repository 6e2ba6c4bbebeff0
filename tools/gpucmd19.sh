mkdir -p gpurun_out
for F in 1 8; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step $F --steps 300 > gpurun_out/b.log 2>&1; echo -n "frames $F: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,1), 'us/frame', {k: round(v/$F,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log
done
timeout -s KILL 600 ncu --set full --import-source on --cache-control none --clock-control none -k 'regex:k_fit_stream' -c 2 -f -o gpurun_out/prof_fs python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step 8 --steps 3 --warmup 3 --no-graph > gpurun_out/ncu_fs.log 2>&1; tail -1 gpurun_out/ncu_fs.log
