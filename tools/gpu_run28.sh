timeout 2400 python tools/c4_run.py > gpurun_out/r02_c4.txt 2>&1
PASTILA_SCALE_C4=1 timeout 1200 python -m pytest tests/test_gpu_scale.py -q -k c4 > gpurun_out/r02_c4_parity.txt 2>&1
tail -2 gpurun_out/r02_c4.txt; tail -2 gpurun_out/r02_c4_parity.txt
