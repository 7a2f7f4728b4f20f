"""How many rows' sliding minima (AB) change between adjacent windows, on planted-walk
data (oracle AB matrices): the cost driver of any change-list selection design.
usage: python tools/ab_changes.py"""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle.pastila_oracle import sliding_stats, distance_block, window_default, order_default
from paper_2401_13680_b200.datagen import planted_walk
from scipy.ndimage import minimum_filter1d
x,_ = planted_walk(200000, m_act=256, A=4, seed=0)
for m in [64, 128, 256, 512]:
    l = window_default(m); w = m-l+1
    mu,_,var = sliding_stats(x, l)
    tot=[]
    for seg in [3, 50, 200]:
        rows = distance_block(x, mu, var, seg*m, w, l)[:, :30000+w]
        ab = minimum_filter1d(rows, size=w, axis=-1, mode="nearest")[:, w//2: w//2+30000]
        ch = (ab[:,1:] != ab[:,:-1]).sum(axis=0)
        tot.append(ch)
    ch=np.concatenate(tot)
    print(f"m={m} w={w}: changes/window mean {ch.mean():.2f} median {np.median(ch):.0f} p90 {np.percentile(ch,90):.0f} p99 {np.percentile(ch,99):.0f} max {ch.max()}  frac>16: {(ch>16).mean():.3f}")
