# r02 evidence: launch list of one m=256 search, ncu --set full of one batch (row + selection), C5 sweep, C4 single-GPU run
MODES=keys ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_m256.csv python tools/len_times.py 256 > /dev/null 2>&1
MODES=keys timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_mpdist|k_select_run' -s 40 -c 2 -o gpurun_out/r02_full_m256 -f python tools/len_times.py 256 > /dev/null 2>&1
timeout 1500 python tools/c5_run.py > gpurun_out/r02_c5.txt 2>&1
