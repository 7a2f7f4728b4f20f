"""Rank-move statistics of the selection pivot (previous window's answer) on planted-walk data,
from the oracle's AB/BA multisets: fraction of windows whose answer keeps / moves its rank.
usage: python tools/rankmove.py 64,96,128,256,512"""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle.pastila_oracle import sliding_stats, distance_block, window_default, order_default
from paper_2401_13680_b200.datagen import planted_walk
from scipy.ndimage import minimum_filter1d
from numpy.lib.stride_tricks import sliding_window_view
x,_ = planted_walk(100000, m_act=120, A=3, seed=0)
for m in [int(a) for a in sys.argv[1].split(',')]:
    l = window_default(m); k = order_default(m); w = m-l+1
    st = sliding_stats(x, l); mu,_,var = st
    N = x.size-m+1
    moves=[]
    for seg in [3, 100, 150]:
        rows = distance_block(x, mu, var, seg*m, w, l)[:, :20000+w]
        colmin = rows.min(axis=0)
        NN=20000
        ab = minimum_filter1d(rows, size=w, axis=-1, mode="nearest")[:, w//2: w//2+NN]
        ba = sliding_window_view(colmin[:NN+w-1], w).T
        M = np.concatenate([ab, ba], axis=0)
        ans = np.partition(M, k-1, axis=0)[k-1]
        p = ans[:-1]; Mn = M[:,1:]
        lt = (Mn < p).sum(0); le = (Mn <= p).sum(0)
        mv = np.where(k <= lt, k-lt-1, np.where(k > le, k-le, 0))
        moves.append(mv)
    mv = np.concatenate(moves)
    a = np.abs(mv)
    print(f"m={m} w={w} k={k}: " + " ".join(f"<={t}:{(a<=t).mean():.3f}" for t in (0,1,2,3,4,6,8,12,16)) + f" max {a.max()}")
