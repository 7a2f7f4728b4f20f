python tools/lb_feasibility.py 256
python tools/lb_feasibility.py 256 2e6 3
