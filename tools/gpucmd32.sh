mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_modulated_gpu.py -q -x -rf > gpurun_out/pt_mod.log 2>&1; echo "mod rc=$?"; tail -15 gpurun_out/pt_mod.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
