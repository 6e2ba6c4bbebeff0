mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "not sweep_q" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for V in ws ring; do for F in 1 8; do
if [ $V = ring ]; then export FLR_APPLY_RING=1; else unset FLR_APPLY_RING; fi
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step $F --steps 300 > gpurun_out/b.log 2>&1; echo -n "$V frames $F: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,1), 'us/frame', {k: round(v/$F,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log
done; done
