mkdir -p gpurun_out
for F in 1 8; do
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k 'regex:^k_' -c 40 --csv --log-file gpurun_out/warm$F.csv python bench.py --no-cpu-baseline --e2e-steps 1 --variant 1 --frames-per-step $F --steps 4 --warmup 4 --no-graph > gpurun_out/ncu_w$F.log 2>&1; tail -1 gpurun_out/ncu_w$F.log | cut -c1-100
done
