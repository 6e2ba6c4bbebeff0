# round-2 evidence: gpu tests, smoke, C2 bench with parity, whole-step DRAM traffic (ncu range replay)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --check > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_c2.log
for V in staged fused; do
timeout -s KILL 300 python tools/step_traffic.py $V > /dev/null 2>&1 && \
timeout -s KILL 600 ncu --replay-mode range --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r02_step_traffic_$V.csv python tools/step_traffic.py $V > gpurun_out/ncu_step_$V.log 2>&1; echo "ncu step $V rc=$?"; cat gpurun_out/r02_step_traffic_$V.csv | tail -5
done
