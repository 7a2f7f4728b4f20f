MODES=keys PASTILA_V2=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_v2b_m256.csv python tools/len_times.py 256 > /dev/null 2>&1
MODES=keys PASTILA_V2=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_rowsP' -s 20 -c 1 -o gpurun_out/full_v2b_m256 -f python tools/len_times.py 256 > /dev/null 2>&1
