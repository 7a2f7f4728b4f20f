import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk
from oracle import pastila_oracle as O
n, m = 3000, 64
x, _ = planted_walk(n, m_act=50, A=3, seed=3)
pr = P.MPdistParams(m); l, k = pr.window_size, pr.k
S, N = n // m, n - m + 1
D = np.empty((S, N))
with _native.context().using(x) as ctx:
    ctx.call("pst_mpdist_profiles", m, l, k, 0, S, _native.ptr(D))
seg, win = np.meshgrid(np.arange(S), np.arange(N), indexing="ij")
seg = np.ascontiguousarray(seg.ravel()); win = np.ascontiguousarray(win.ravel())
out = np.empty(seg.size)
with _native.context().using(x) as ctx:
    ctx.call("pst_window_exact", m, l, k, _native.ptr(seg, C.c_int64), _native.ptr(win, C.c_int64), seg.size, _native.ptr(out))
out = out.reshape(S, N)
bad = np.argwhere(out != D)
print("mismatches", len(bad), "of", D.size)
st = O.sliding_stats(x, l)
for s in sorted(set(bad[:, 0].tolist()))[:4]:
    ref = O.mpdist_profile(x, s, m, l, k, st)
    js = bad[bad[:, 0] == s][:, 1]
    print("seg", s, "windows", js[:10], "kernel-oracle", np.abs(D[s] - ref).max(), "eval-oracle", np.abs(out[s] - ref).max())
    for j in js[:5]:
        print("  j", j, D[s, j], out[s, j], ref[j])
