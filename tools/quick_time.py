import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_13680_b200 as P
from paper_2401_13680_b200.datagen import planted_walk
def pairs(n, m):
    l = P.default_window_size(m); return (m - l + 1) * (n - l + 1) * (n // m)
x, _ = planted_walk(100000, m_act=120, A=3, seed=0)
s = P.TimeSeries(x)
P.select_snippets(s, P.MPdistParams(64), 3)
t0 = time.perf_counter(); P.select_length(s, list(range(64, 513, 32)), 3, training_log=False); t = time.perf_counter() - t0
tot = sum(pairs(100000, m) for m in range(64, 513, 32))
print(f"C2 sweep: {t:.2f} s, {tot/t:.3e} pairs/s")
for m in (64, 256, 512):
    t0 = time.perf_counter(); P.select_snippets(s, P.MPdistParams(m), 3); t = time.perf_counter() - t0
    print(f"n=1e5 m={m}: {t:.3f} s {pairs(100000, m)/t:.3e} pairs/s")
x, _ = planted_walk(1000000, m_act=256, A=4, seed=0)
s = P.TimeSeries(x)
for m in (256,):
    t0 = time.perf_counter(); P.select_snippets(s, P.MPdistParams(m), 4); t = time.perf_counter() - t0
    print(f"n=1e6 m={m}: {t:.3f} s {pairs(1000000, m)/t:.3e} pairs/s")
