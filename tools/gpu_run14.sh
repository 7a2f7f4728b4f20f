for nws in 1 4; do for m in 64 256 512; do
PASTILA_NWS=$nws MODES=keys ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:k_select_run --log-file gpurun_out/sel_nws${nws}_m$m.csv python tools/len_times.py $m > /dev/null 2>&1
done; done
