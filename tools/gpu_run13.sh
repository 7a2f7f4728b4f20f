for f in 0 1 4 5; do echo DBGF=$f; MODES=keys PASTILA_KTIME=1 PASTILA_DBGF=$f python tools/len_times.py 64 256 512 2>&1 | tail -3 | sed 's/"pairs_per_s.*//'; done
