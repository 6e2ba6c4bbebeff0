mkdir -p gpurun_out
timeout -s KILL 60 tools/ubench_stream
for n in 1 8; do timeout -s KILL 30 tools/t_k2 $n | grep tile; done; timeout -s KILL 30 tools/t_k2_ph 1 | grep -A1 tile
