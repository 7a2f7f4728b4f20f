"""One select_snippets at n=1e5 (planted walk), m given on argv -- profiling target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_13680_b200 as P
from paper_2401_13680_b200.datagen import planted_walk
m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
x, _ = planted_walk(n, m_act=120, A=3, seed=0)
r = P.select_snippets(P.TimeSeries(x), P.MPdistParams(m), 3)
print([s.index for s in r.snippets])
