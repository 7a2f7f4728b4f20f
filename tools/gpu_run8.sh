for v in 1 0; do MODES=keys PASTILA_V2=$v python tools/len_times.py 64 256 512 2>&1 | tail -3; done
for nws in 1 2; do MODES=keys PASTILA_V2=0 PASTILA_NWS=$nws python tools/len_times.py 64 256 512 2>&1 | tail -3; done
