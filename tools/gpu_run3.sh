# ncu --set full of one key-path batch at m=256 (row kernel + selection)
MODES=keys timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_mpdist|k_select_run' -s 40 -c 2 -o gpurun_out/full_keys_m256 -f python tools/len_times.py 256 > gpurun_out/full_keys_m256.log 2>&1
ls -la gpurun_out/
