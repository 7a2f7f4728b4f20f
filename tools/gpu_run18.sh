timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
MODES=keys python tools/len_times.py 64 256 512 2>&1 | tail -3 | sed 's/"profile_kernel_s.*//'
