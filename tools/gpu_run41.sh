for rep in 1 2; do for v in def nt256; do echo V=$v; if [ $v = def ]; then unset PASTILA_NT_W; else export PASTILA_NT_W=9999; fi; MODES=keys python tools/len_times.py 64 96 128 2>&1 | tail -3 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['m'], round(d['total_s'],3), d['snippets'], end='; ')
print()"; done; done
