set -x
mkdir -p gpurun_out
B="python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/exp_base.log 2>&1; echo base=$?
cp paper_2410_11625_b200/libflr.so gpurun_exp/libflr_base.so
cp gpurun_exp/libflr_frsq.so paper_2410_11625_b200/libflr.so
timeout 300 $B > gpurun_out/exp_frsq.log 2>&1; echo frsq=$?
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 --check > gpurun_out/exp_frsq_check.log 2>&1; echo check=$?
timeout 300 $B > gpurun_out/exp_frsqb.log 2>&1
cp gpurun_exp/libflr_base.so paper_2410_11625_b200/libflr.so
timeout 300 $B > gpurun_out/exp_base2.log 2>&1; echo base2=$?
for f in gpurun_out/exp_base*.log gpurun_out/exp_frsq*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_frame']*1000, d['kernel_us'], d.get('parity'))" ; done
