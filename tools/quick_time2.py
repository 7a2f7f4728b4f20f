import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_13680_b200 as P
from paper_2401_13680_b200.datagen import planted_walk
def pairs(n, m):
    l = P.default_window_size(m); return (m - l + 1) * (n - l + 1) * (n // m)
x, _ = planted_walk(1000000, m_act=256, A=4, seed=0)
s = P.TimeSeries(x)
P.select_snippets(s, P.MPdistParams(512), 4)
for m in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64,256,512").split(",")]:
    t0 = time.perf_counter(); P.select_snippets(s, P.MPdistParams(m), 4); t = time.perf_counter() - t0
    print(f"n=1e6 m={m}: {t:.3f} s {pairs(1000000, m)/t:.3e} pairs/s", flush=True)
