set -x
mkdir -p gpurun_out
B="python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/exp_base.log 2>&1; echo base=$?
cp paper_2410_11625_b200/libflr.so gpurun_exp/libflr_base.so
cp gpurun_exp/libflr_ty4.so paper_2410_11625_b200/libflr.so
timeout 300 $B > gpurun_out/exp_ty4.log 2>&1; echo ty4=$?
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 --check > gpurun_out/exp_ty4_check.log 2>&1; echo check=$?
timeout 300 $B > gpurun_out/exp_ty4b.log 2>&1
cp gpurun_exp/libflr_base.so paper_2410_11625_b200/libflr.so
timeout 300 $B > gpurun_out/exp_base2.log 2>&1; echo base2=$?
for f in gpurun_out/exp_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_frame']*1000, d['kernel_us'], d.get('parity'))" ; done
