for i in 1 2; do timeout -s KILL 30 tools/t_k2_ph 1 | grep -A2 tile; done
timeout -s KILL 30 tools/t_k2_ty4 1 | grep -A2 tile
