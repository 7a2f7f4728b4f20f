"""Per-length timing on the C3 series: total select_snippets time and profile-kernel
time (pst_timing, CUDA events on the library stream), key path vs exact path.
usage: python tools/len_times.py [m ...]   (env PASTILA_* knobs apply)"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk

ms = [int(a) for a in sys.argv[1:]] or [64, 256, 512]
modes = os.environ.get("MODES", "keys,exact").split(",")
x, _ = planted_walk(1_000_000, m_act=256, A=4, seed=0)
s = P.TimeSeries(x)
ctx = _native.context()
out = []
for m in ms:
    for mode in modes:
        os.environ["PASTILA_EXACT"] = "1" if mode == "exact" else "0"
        P.select_snippets(s, P.MPdistParams(m), 4)  # warm
        ctx.call("pst_timing", 1)
        st = np.zeros(8, dtype=np.int64)
        ctx.call("pst_cert_stats", _native.ptr(st, C.c_int64), 1)
        t0 = time.perf_counter()
        r = P.select_snippets(s, P.MPdistParams(m), 4)
        ctx.call("pst_sync")
        dt = time.perf_counter() - t0
        kms, kl = C.c_double(0), C.c_int64(0)
        ctx.call("pst_timing_read", C.byref(kms), C.byref(kl))
        kt = np.zeros(2)
        ctx.call("pst_kernel_times", _native.ptr(kt))
        ctx.call("pst_timing", 0)
        ctx.call("pst_cert_stats", _native.ptr(st, C.c_int64), 0)
        l = P.MPdistParams(m).window_size
        pairs = (m - l + 1) * (x.size - l + 1) * (x.size // m)
        rec = {"m": m, "mode": mode, "total_s": dt, "profile_kernel_s": kms.value / 1e3, "row_s": kt[0] / 1e3, "sel_s": kt[1] / 1e3,
               "pairs_per_s": pairs / dt, "snippets": [sn.index for sn in r.snippets],
               "cert": st.tolist()}
        out.append(rec)
        print(json.dumps(rec), flush=True)
