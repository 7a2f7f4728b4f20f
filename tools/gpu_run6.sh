timeout 900 python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15
MODES=keys python tools/len_times.py 64 128 256 512 2>&1 | tail -4
for m in 64 256 512; do
 MODES=keys ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_v2_m$m.csv python tools/len_times.py $m > /dev/null 2>&1
done
