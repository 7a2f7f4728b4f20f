for rep in 1 2; do for cfg in "X=1" "PASTILA_ROW_SMEM_KB=120" "PASTILA_ROW_SMEM_KB=120 PASTILA_NWS=4"; do echo "CFG $cfg"; env $cfg MODES=keys python tools/len_times.py 192 256 2>&1 | python -c "
import sys,json
t=0
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); t+=d['total_s']; print(d['m'], round(d['total_s'],3), end='; ')
print('sum', round(t,3))"; done; done
