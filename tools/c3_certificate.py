"""Near-tie certificate for the C3 sweep (n = 1e6, 15 lengths, K = 4): every length
on the key path (certified decisions, exact recomputation of the uncertain ones) and on
the exact fp64 path (PASTILA_EXACT=1); all outputs must be identical.  Writes JSON.
usage: python tools/c3_certificate.py out.json"""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk

x, _ = planted_walk(1_000_000, m_act=256, A=4, seed=0)
s = P.TimeSeries(x)
ctx = _native.context()
names = ["lengths", "greedy_exact_candidates", "greedy_steps_multi", "attribution_uncertain_windows",
         "exact_window_evals", "max_candidates", "fallbacks_to_exact", "windows"]
out = {"workload": "C3: planted walk n=1e6 (A=4, m_act=256, seed 0), m=64..512 step 32, K=4",
       "lengths": []}
allsame = True
for m in range(64, 513, 32):
    p = P.MPdistParams(m)
    st = np.zeros(8, dtype=np.int64)
    ctx.call("pst_cert_stats", _native.ptr(st, C.c_int64), 1)
    os.environ["PASTILA_EXACT"] = "0"
    t0 = time.perf_counter(); a = P.select_snippets(s, p, 4); ta = time.perf_counter() - t0
    ctx.call("pst_cert_stats", _native.ptr(st, C.c_int64), 1)
    os.environ["PASTILA_EXACT"] = "1"
    t0 = time.perf_counter(); b = P.select_snippets(s, p, 4); tb = time.perf_counter() - t0
    same = ([q.index for q in a.snippets] == [q.index for q in b.snippets]
            and [q.frac for q in a.snippets] == [q.frac for q in b.snippets]
            and np.array_equal(a.segment_window_counts, b.segment_window_counts)
            and all(np.array_equal(u.neighbors, v.neighbors) for u, v in zip(a.snippets, b.snippets))
            and a.profile_area == b.profile_area and a.profile_max == b.profile_max
            and a.criterion_ == b.criterion_ and np.array_equal(a.labels_, b.labels_)
            and all(np.array_equal(u.values, v.values) for u, v in zip(a.profiles, b.profiles)))
    allsame &= same
    rec = {"m": m, "key_path_s": ta, "exact_path_s": tb, "identical_outputs": bool(same),
           "snippets": [q.index for q in a.snippets], "fracs": [q.frac for q in a.snippets],
           "criterion": a.criterion_, "profile_max": a.profile_max,
           "certification": dict(zip(names, st.tolist()))}
    out["lengths"].append(rec)
    print(json.dumps(rec), flush=True)
del os.environ["PASTILA_EXACT"]
out["all_identical"] = bool(allsame)
out["meaning"] = ("key path: every greedy argmin, nearest-segment argmin and profile_max is decided from "
                  "monotone interval bounds of the 32-bit e-keys; decisions the bounds cannot separate "
                  "(counts above) are recomputed with exact fp64 values; identical_outputs compares the "
                  "result with the all-exact path bit for bit")
json.dump(out, open(sys.argv[1], "w"), indent=1)
