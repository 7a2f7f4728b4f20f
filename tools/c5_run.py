"""Config C5 (BASELINE.json configs[4]): n = 2,000,000 planted walk (A=5, m_act=2048),
long windows m in {1024, 2048, 4096}, K = 5.  Prints per-length time and pairs/s."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_13680_b200 as P
from paper_2401_13680_b200.datagen import planted_walk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
x, _ = planted_walk(n, m_act=2048, A=5, seed=0)
s = P.TimeSeries(x)
P.select_snippets(s, P.MPdistParams(1024), 5)  # warm-up
for m in (1024, 2048, 4096):
    l = P.default_window_size(m)
    pairs = (m - l + 1) * (n - l + 1) * (n // m)
    t0 = time.perf_counter()
    r = P.select_snippets(s, P.MPdistParams(m), 5)
    t = time.perf_counter() - t0
    print(f"C5 m={m}: {t:.2f} s {pairs / t:.3e} pairs/s snippets={[q.index for q in r.snippets]}", flush=True)
