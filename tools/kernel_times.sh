#!/bin/bash
# per-kernel serialized times (ncu launch list) of tools/tune.py for one m; args: m [env assignments...]
m=$1; shift
env "$@" ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/kt.csv python tools/tune.py $m 1000000 24 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('/tmp/kt.csv'))); hdr=None; agg=collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            agg[d['Kernel Name'].split('(')[0][-28:]].append(float(d['Metric Value'])*{'ns':1e-6,'us':1e-3,'ms':1}[d['Metric Unit']])
print('  '.join(f"{k}: {sum(v):.1f} ms/{len(v)}" for k,v in sorted(agg.items(), key=lambda x:-sum(x[1])) if 'k_prefix' not in k and sum(v) > 1))
PY
