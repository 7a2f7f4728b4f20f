"""Config C4 (BASELINE.json configs[3]) on the GPUs of this process group, or one GPU:
n = 10,000,000 planted walk (A=3, m_act=256, seed 0), fixed m = 256 (l=128, k=26), K = 3.
The 39,062 x 9,999,745 profile matrix (1.6 TB of keys) does not fit, so selection
streams: the streamed key path (pastila.cu run_select_keys_streamed; greedy passes
after the second pruned to the rows that can still win).  Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native, parallel
from paper_2401_13680_b200.datagen import planted_walk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
m, K = 256, 3
x, _ = planted_walk(n, m_act=256, A=3, seed=0)
s, p = P.TimeSeries(x), P.MPdistParams(m)
t0 = time.perf_counter()
if parallel.world_size() > 1:
    r = parallel.select_snippets_sharded(s, p, K)
else:
    r = P.select_snippets(s, p, K)
t = time.perf_counter() - t0
pairs = (m - p.window_size + 1) * (n - p.window_size + 1) * (n // m)
labels = P.label_series(r)
ps = np.zeros(4, dtype=np.int64)
_native.context().call("pst_prune_stats", _native.ptr(ps, C.c_int64), 0)
if parallel.rank() == 0:
    print(json.dumps({"config": "C4", "n": n, "m": m, "K": K, "gpus": parallel.world_size(), "seconds": t,
                      "pairs": pairs, "pairs_per_s": pairs / t, "greedy_profile_passes": K,
                      "snippets": [q.index for q in r.snippets], "fracs": [q.frac for q in r.snippets],
                      "profile_area": r.profile_area, "profile_max": r.profile_max,
                      "label_counts": np.bincount(labels.labels).tolist(),
                      "pruned_passes": int(ps[0]), "pruned_rows": int(ps[1]), "segments": n // m,
                      "prune_fallbacks": int(ps[2])}), flush=True)
