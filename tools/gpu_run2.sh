python tools/len_times.py 64 128 256 512 > gpurun_out/len_times.jsonl 2> gpurun_out/len_times.err
for m in 64 256 512; do
 MODES=keys ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_keys_m$m.csv python tools/len_times.py $m > /dev/null 2>&1
done
