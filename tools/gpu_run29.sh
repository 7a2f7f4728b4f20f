timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
PASTILA_SCALE_C4=1 timeout 1200 python -m pytest tests/test_gpu_scale.py -q -k c4 > gpurun_out/r02_c4_parity.txt 2>&1; tail -2 gpurun_out/r02_c4_parity.txt
for g in 0 1 2 4; do echo GRP=$g; PASTILA_GRP=$g MODES=keys python tools/len_times.py 64 256 512 2>&1 | tail -3 | sed 's/"profile_kernel_s.*//'; done
