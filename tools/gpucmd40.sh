mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_inputs_ready_gpu.py -q -rf > gpurun_out/pt_ir.log 2>&1; echo "ir rc=$?"; tail -5 gpurun_out/pt_ir.log
run() { timeout -s KILL 300 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 2000 "$@" > gpurun_out/b.log 2>&1; echo -n "$*: "; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()}, round(d['step_roofline']['frac'],3))" || tail -3 gpurun_out/b.log; }
for i in 1 2; do run; run --no-inputs-ready; done
run --guides f16; run --config c4; run --frames-per-step 8
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
