set -e
python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for v in new old new old; do echo V=$v; if [ $v = old ]; then export PASTILA_LIB=tools/libpastila_old.so; else unset PASTILA_LIB; fi; MODES=keys python tools/len_times.py 64 128 192 256 320 384 448 512 2>&1 | tail -8 | python -c "
import sys,json
tot=0
for l in sys.stdin:
    d=json.loads(l); tot+=d['total_s']; print(d['m'], round(d['total_s'],3), end='; ')
print('sum', round(tot,3))"; done
