for v in base direct ldg ldgdir; do echo "== $v"; for i in 1 2; do timeout -s KILL 30 tools/t_k2_$v 1 | grep -A2 "tile " | grep -v rows; done; timeout -s KILL 30 tools/t_k2_$v 8 | grep "tile "; done
