timeout 600 python -m pytest tests/test_gpu_keys.py -x -q 2>&1 | tail -2
for v in 1 0; do MODES=keys PASTILA_V2=$v python tools/len_times.py 64 256 512 2>&1 | tail -3; done
