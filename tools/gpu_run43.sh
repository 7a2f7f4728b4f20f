for cfg in "X=1" "PASTILA_P=5" "PASTILA_NT_W=99999" "PASTILA_NT_W=99999 PASTILA_P=5"; do echo "CFG $cfg"; env $cfg MODES=keys python tools/len_times.py 1024 2048 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['m'], round(d['total_s'],3), d['snippets'], end='; ')
print()"; done
