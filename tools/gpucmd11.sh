mkdir -p gpurun_out
for L in 40 100; do timeout -s KILL 60 tools/t_fused $L; timeout -s KILL 60 tools/t_fused_fake $L | sed 's/^/FAKE /'; done
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -k "variants or fused" 2>&1 | tail -4
for V in 1 2; do for F in 1 8; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --variant $V --frames-per-step $F --steps 200 > gpurun_out/b.log 2>&1; echo -n "variant $V frames $F: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,1), 'us/frame', {k: round(v/$F,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log
done; done
