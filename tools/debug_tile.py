"""Debug: compare the first tile's AB matrix / column minima with a numpy emulation."""
import os, sys, json, ctypes as C
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PASTILA_DEBUG"] = "1"
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from oracle import pastila_oracle as O
g = np.load('tests/golden/golden.npz'); meta = json.load(open('tests/golden/golden.json'))
case = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cs = meta['prof'][case]; x = g[f'prof{case}_x']
m, l, k = cs['m'], cs['l'], cs['k']; n = len(x); w = m-l+1; Nl = n-l+1; N = n-m+1
seg = cs["segs"][int(sys.argv[2]) if len(sys.argv) > 2 else 0]
prof = P.mpdist_profile(P.TimeSeries(x), seg, P.MPdistParams(m, l, k)).values
lib = _native.load_library()
lib.pst_debug_last_tile.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
dims = np.zeros(3, dtype=np.int64)
lib.pst_debug_last_tile(_native.context().h, None, None, dims.ctypes.data_as(C.POINTER(C.c_int64)))
W, T, NC = dims
ab = np.zeros(W*T); ba = np.zeros(NC)
lib.pst_debug_last_tile(_native.context().h, ab.ctypes.data_as(C.POINTER(C.c_double)), ba.ctypes.data_as(C.POINTER(C.c_double)), dims.ctypes.data_as(C.POINTER(C.c_int64)))
ab = ab.reshape(W, T)
mu, sd, var = O.sliding_stats(x, l)
rows = O.distance_block(x, mu, var, seg*m, w, l)   # distances
E = rows**2/(2*l)
ba_ref = E.min(0)[:NC]
ab_ref = np.stack([E[:, j:j+w].min(1) for j in range(min(T, N))], 1)
print('dims', dims, 'N', N)
print('BA maxdiff', np.abs(ba-ba_ref).max(), 'first bad', np.flatnonzero(np.abs(ba-ba_ref)>1e-9)[:10])
d = np.abs(ab[:, :ab_ref.shape[1]]-ab_ref)
print('AB maxdiff', d.max(), 'bad (row,col)', np.argwhere(d>1e-9)[:10])
ref = O.mpdist_profile(x, seg, m, l, k)
print('prof maxdiff', np.abs(prof-ref).max(), np.flatnonzero(np.abs(prof-ref)>1e-7)[:20])
