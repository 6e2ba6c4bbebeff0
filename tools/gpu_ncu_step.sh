# whole-step DRAM traffic of one C2 call (ncu range replay over a cudaProfilerStart/Stop range)
mkdir -p gpurun_out
for V in staged fused; do
timeout -s KILL 600 ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r02_step_traffic_$V.csv python tools/step_traffic.py $V > gpurun_out/ncu_step_$V.log 2>&1; echo "ncu step $V rc=$?"; tail -3 gpurun_out/ncu_step_$V.log; cat gpurun_out/r02_step_traffic_$V.csv | tail -6
done
