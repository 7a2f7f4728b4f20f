"""Configs C1 and C2 (BASELINE.json configs[0..1]) end to end through the public API,
host series in, results out; the reference's own CPU times on the same inputs are
in SURVEY.md §8(d) (C1: 10.6 s on 1 core, C2: 851.1 s on 8 cores).  One JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_13680_b200 as P
from paper_2401_13680_b200.datagen import planted_walk

x1, _ = planted_walk(20000, m_act=120, A=3, seed=0)
x2, _ = planted_walk(100000, m_act=120, A=3, seed=0)
P.select_snippets(P.TimeSeries(x1), P.MPdistParams(120), 3)  # context + library warm-up
out = {}
for rep in range(2):  # second repetition reported (first includes per-length allocations)
    t0 = time.perf_counter()
    r = P.select_snippets(P.TimeSeries(x1.copy()), P.MPdistParams(120), 3)
    lab = P.label_series(r)
    c1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep2, res2 = P.select_length(P.TimeSeries(x2.copy()), list(range(64, 513, 32)), 3, training_log=False)
    c2 = time.perf_counter() - t0
out = {"C1": {"seconds": c1, "reference_cpu_seconds": 10.6, "speedup_vs_1_core": 10.6 / c1,
              "snippets": [s.index for s in r.snippets]},
       "C2": {"seconds": c2, "reference_cpu_seconds_8_cores": 851.1, "speedup_vs_8_cores": 851.1 / c2,
              "m_best": rep2.m_best}}
print(json.dumps(out), flush=True)
