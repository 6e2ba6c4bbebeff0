for v in q8 noring; do cp gpurun_exp/$v.so paper_2410_11625_b200/libflr.so;
for X in "--frames-per-step 8" "--config c5 --steps 10 --warmup 3" "--config c3 --steps 200"; do
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 $X 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$X', round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,1) for k,v in d['kernel_us'].items()})"; done; done
cp gpurun_exp/full.so paper_2410_11625_b200/libflr.so
