"""Key-path profile kernel timing over geometry knobs (PASTILA_* env), C3 series.
usage: python tools/tune_keys.py m nseg  (reads configs from TUNE env: 'CHM=5,ROWS2=0;CHM=9,ROWS2=1;...')"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk

m, nseg = int(sys.argv[1]), int(sys.argv[2])
x, _ = planted_walk(1_000_000, m_act=256, A=4, seed=0)
pr = P.MPdistParams(m)
N = x.size - m + 1
out = np.empty((nseg, N), dtype=np.int32)
ctx = _native.context()
cfgs = [c for c in os.environ.get("TUNE", "").split(";") if c] or [""]
for cfg in cfgs:
    kv = dict(t.split("=") for t in cfg.split(",") if t)
    saved = {k: os.environ.get(k) for k in kv}
    for k, v in kv.items():
        os.environ["PASTILA_" + k] = v
    try:
        with ctx.using(x):
            ctx.call("pst_profile_keys", m, pr.window_size, pr.k, 0, nseg, _native.ptr(out, C.c_int32))
            best = None
            for _ in range(int(os.environ.get("TUNE_REPS", "2"))):
                ctx.call("pst_timing", 1)
                ctx.call("pst_profile_keys", m, pr.window_size, pr.k, 0, nseg, _native.ptr(out, C.c_int32))
                kms, kl = C.c_double(0), C.c_int64(0)
                ctx.call("pst_timing_read", C.byref(kms), C.byref(kl))
                ctx.call("pst_timing", 0)
                best = kms.value if best is None else min(best, kms.value)
            kms = C.c_double(best)
        l = pr.window_size
        pairs = (m - l + 1) * (x.size - l + 1) * nseg
        print(json.dumps({"m": m, "cfg": cfg, "ms": kms.value, "pairs_per_s": pairs / (kms.value / 1e3)}), flush=True)
    except Exception as e:
        print(json.dumps({"m": m, "cfg": cfg, "error": str(e)[:200]}), flush=True)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop("PASTILA_" + k, None)
            else:
                os.environ["PASTILA_" + k] = v
