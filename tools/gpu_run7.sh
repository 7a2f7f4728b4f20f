timeout 900 python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
MODES=keys timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_rowsP|k_select_run' -s 40 -c 2 -o gpurun_out/full_v2_m256 -f python tools/len_times.py 256 > gpurun_out/full_v2_m256.log 2>&1
