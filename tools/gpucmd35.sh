for v in fence nofence s3nf; do echo "== $v"; timeout -s KILL 60 tools/t_fitws_$v; done
