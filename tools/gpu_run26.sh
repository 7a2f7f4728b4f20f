timeout 900 python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
MODES=keys python tools/len_times.py 64 256 512 2>&1 | tail -3 | sed 's/"profile_kernel_s.*//'
