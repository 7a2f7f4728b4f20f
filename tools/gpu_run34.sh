set -e
for rep in 1 2; do for v in base occ unr both; do echo V=$v; if [ $v = base ]; then unset PASTILA_LIB; else export PASTILA_LIB=tools/libpastila_$v.so; fi; MODES=keys python tools/len_times.py 64 128 192 256 384 512 2>&1 | tail -6 | python -c "
import sys,json
tot=0
for l in sys.stdin:
    d=json.loads(l); tot+=d['total_s']; print(d['m'], round(d['total_s'],3), end='; ')
print('sum', round(tot,3))"; done; done
