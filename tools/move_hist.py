"""Rank-move histogram of the selection (previous answer vs this window's rank), C3 series.
usage: PASTILA_DBGF=16 python tools/move_hist.py m nseg"""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk
m, nseg = int(sys.argv[1]), int(sys.argv[2])
x, _ = planted_walk(1_000_000, m_act=256, A=4, seed=0)
pr = P.MPdistParams(m)
out = np.empty((nseg, x.size - m + 1), dtype=np.int32)
ctx = _native.context()
with ctx.using(x):
    ctx.call("pst_profile_keys", m, pr.window_size, pr.k, 0, nseg, _native.ptr(out, C.c_int32))
    h = np.zeros(8, dtype=np.int64)
    ctx.call("pst_debug_hist", _native.ptr(h, C.c_int64))
tot = h.sum()
print(json.dumps({"m": m, "hist": dict(zip(["0", "1", "2", "3-4", "5-8", "9-16", ">16"], (h[:7] / tot).round(4).tolist()))}))
