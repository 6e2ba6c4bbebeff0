mkdir -p gpurun_out
for V in 1; do
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph --variant $V"
timeout -s KILL 300 $CMD > gpurun_out/plain_v$V.log 2>&1 && timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"k_blur|k_solve" -s 2 -c 2 -o gpurun_out/prof_v$V $CMD > gpurun_out/ncu_v$V.log 2>&1; echo "ncu v$V rc=$?"
done
