mkdir -p gpurun_out
./tools/ubench_fma > gpurun_out/ubench_fma.log 2>&1; echo "ubench rc=$?"; cat gpurun_out/ubench_fma.log
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --check > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 20 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
