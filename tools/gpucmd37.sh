mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_half_guides_gpu.py -q -rf > gpurun_out/pt_half.log 2>&1; echo "half rc=$?"; tail -15 gpurun_out/pt_half.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for G in f32 f16; do for C in c2 c4; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --guides $G --config $C --steps 1000 --check > gpurun_out/b.log 2>&1; echo -n "$G $C: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3), d['parity']['max_ratio'], d['parity']['violations'])" || tail -3 gpurun_out/b.log
done; done
