for rep in 1 2; do for cfg in "X=1" "PASTILA_NWS=1" "PASTILA_NWS=2"; do echo "CFG $cfg"; env $cfg MODES=keys python tools/len_times.py 64 96 128 160 192 224 256 288 320 352 384 416 448 480 512 2>&1 | python -c "
import sys,json
t=0
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); t+=d['total_s']; print(d['m'], round(d['total_s'],3), end='; ')
print('sum', round(t,3))"; done; done
