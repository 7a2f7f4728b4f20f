"""Decision margins of the C3 workload (planted walk, m_act=256, A=4) at reduced n:
attribution (best vs second-best segment per window) and greedy area gaps,
from exact device profiles.  Sizes how many decisions a coarser profile key
would leave uncertain.  usage: python tools/gap_stats.py [n] [m ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
ms = [int(a) for a in sys.argv[2:]] or [64, 256, 512]
x, _ = planted_walk(n, m_act=256, A=4, seed=0)
for m in ms:
    pr = P.MPdistParams(m)
    S, N = n // m, n - m + 1
    D = np.empty((S, N))
    with _native.context().using(x) as ctx:
        ctx.call("pst_mpdist_profiles", m, pr.window_size, pr.k, 0, S, _native.ptr(D))
    part = np.partition(D, 1, axis=0)
    b1, b2 = part[0], part[1]
    rel = (b2 - b1) / np.maximum(b1, 1e-300)
    # greedy
    curve = np.full(N, np.inf)
    taken = np.zeros(S, bool)
    ggaps = []
    for step in range(4):
        areas = np.minimum(D, curve).sum(axis=1)
        areas[taken] = np.inf
        o = np.argsort(areas)
        ggaps.append(float((areas[o[1]] - areas[o[0]]) / areas[o[0]]))
        taken[o[0]] = True
        curve = np.minimum(curve, D[o[0]])
    rec = {"n": n, "m": m, "S": S, "N": N,
           "profile_value_quantiles": np.quantile(D, [0, 0.001, 0.01, 0.5, 0.99, 1]).tolist(),
           "attrib_rel_gap_lt": {t: int((rel < float(t)).sum()) for t in ["1e-2", "3e-3", "1e-3", "5e-4", "1e-4", "1e-6"]},
           "attrib_exact_ties": int((b2 == b1).sum()),
           "greedy_rel_gaps": ggaps,
           "max_top2_rel": float((np.sort(D.ravel())[-1] - np.sort(D.ravel())[-2]) / np.max(D))}
    rec["attrib_rel_gap_lt"] = {k: v for k, v in rec["attrib_rel_gap_lt"].items()}
    print(json.dumps(rec), flush=True)
