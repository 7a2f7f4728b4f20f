import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from oracle import pastila_oracle as O
m = 4096
rng = np.random.default_rng(11)
x = np.cumsum(rng.standard_normal(12 * m))
x[5 * m:6 * m] = x[1 * m:2 * m]
x[8 * m:9 * m] = x[1 * m:2 * m] + 1e-12 * rng.standard_normal(m)
pr = P.MPdistParams(m); l = pr.window_size
st = O.sliding_stats(x, l)
seg = 1
ref = O.mpdist_profile(x, seg, m, l, pr.k, st, col_chunk=20_000)
out = np.empty((1, x.size - m + 1))
with _native.context().using(x) as ctx:
    ctx.call("pst_mpdist_profiles", m, l, pr.k, seg, seg + 1, _native.ptr(out))
got = out[0]
d = np.abs(got - ref)
j = int(np.argmax(d))
print("worst j", j, "got", got[j], "ref", ref[j], "diff", d[j], "p99 diff", np.quantile(d, 0.99))
# exact distance rows for this window via direct z-normalization, then P_ABBA k-th
w = m - l + 1
rows = np.stack([O.znorm_direct_row(x, seg * m + i, l) for i in range(w)])
ab = rows[:, j:j + w].min(axis=1)
ba = rows.min(axis=0)[j:j + w]
ba[(np.arange(j, j + w) >= seg*m) & (np.arange(j, j + w) < seg*m + w)] = 0.0
allv = np.concatenate([ab, ba])
exact = np.partition(allv, pr.k - 1)[pr.k - 1]
print("direct z-norm value", exact, "|got-direct|", abs(got[j] - exact), "|ref-direct|", abs(ref[j] - exact))
