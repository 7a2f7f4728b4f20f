PASTILA_DEBUG=1 python -m pytest tests/test_gpu_keys.py -q -m gpu -x -s -k "uncertain" 2>&1 | grep -v "^\." | tail -6
python -m pytest tests/test_gpu_keys.py -q -m gpu -x 2>&1 | tail -2 && PASTILA_DEBUG=1 python tools/c4_run.py > gpurun_out/r02_c4_pruned.txt 2> gpurun_out/c4_err.log; tail -4 gpurun_out/c4_err.log; cat gpurun_out/r02_c4_pruned.txt
