bash tools/gpu_check.sh
for X in "--config c3" "--config c4" "--config c5 --steps 20 --warmup 3"; do
  timeout -s KILL 600 python bench.py $X --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; echo -n "$X: "; tail -1 gpurun_out/b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,2) for k,v in d['kernel_us'].items()})"
done
