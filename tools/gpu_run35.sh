for m in 128 256 512; do python tools/lb_feasibility.py $m; done
