# A/B of library builds kept under gpurun_exp/<name>/libflr.so (developer builds, e.g.
# FLR_QS=8 FLR_DEFS=...): each is swapped in and timed by bench.py with the given arguments.
#   bash tools/exp_bench.sh "<bench args>" name1 name2 ...
ARGS="$1"; shift
mkdir -p gpurun_out
for N in "$@"; do
  cp gpurun_exp/$N/libflr.so paper_2410_11625_b200/libflr.so
  for rep in 1 2; do
    timeout -s KILL 300 python bench.py $ARGS --no-cpu-baseline > gpurun_out/exp_$N.json 2> gpurun_out/exp_$N.err
    echo -n "$N rc=$? "; tail -1 gpurun_out/exp_$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_frame']*1e3,2), 'us/frame', {k: round(v,2) for k,v in d['kernel_us'].items()}, 'parity', d.get('parity',{}).get('violations'))" 2>&1 | tail -1
  done
done
