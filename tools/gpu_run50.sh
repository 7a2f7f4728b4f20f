python -m pytest tests/test_gpu_keys.py -q -m gpu -x 2>&1 | tail -1
PASTILA_DEBUG=1 python tools/c4_run.py > gpurun_out/c4_b16.txt 2> gpurun_out/c4_b16_err.log; tail -4 gpurun_out/c4_b16_err.log; cat gpurun_out/c4_b16.txt
