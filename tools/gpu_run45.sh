for rep in 1 2; do for cfg in "PASTILA_SCRATCH_GB=20" "PASTILA_SCRATCH_GB=32" "PASTILA_SCRATCH_GB=48"; do echo "CFG $cfg"; env $cfg MODES=keys python tools/len_times.py 64 128 192 256 320 384 448 512 2>&1 | python -c "
import sys,json
t=0
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); t+=d['total_s']; print(d['m'], round(d['total_s'],3), end='; ')
print('sum', round(t,3))"; done; done
