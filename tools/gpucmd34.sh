for v in base noc s3 s5; do echo "== $v"; timeout -s KILL 60 tools/t_fitws_$v; done
