"""Feasibility of block-minimum lower bounds for pruned greedy passes (C4 idea).
C3 series, one length: step-1 areas sum_j min(curve_j, d(s, j)) vs the lower
bound sum_j min(curve_j, min_{j' in block(j)} d(s, j')); prints how many
segments the bound cannot exclude, per block size.
usage: python tools/lb_feasibility.py m [n] [A]   (default: the C3 series, n = 1e6, A = 4)"""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk
m = int(sys.argv[1])
n_ = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
A_ = int(sys.argv[3]) if len(sys.argv) > 3 else 4
x, _ = planted_walk(n_, m_act=256, A=A_, seed=0)
pr = P.MPdistParams(m)
l = pr.window_size
N = x.size - m + 1
S = x.size // m
ctx = _native.context()
CH = 256
BS = (16, 32, 64, 128, 256)
def keys_to_d(kk):
    hi = kk.to(torch.int64) << 32
    e = hi.view(torch.float64)
    e = torch.where(kk < 0, torch.zeros_like(e), e).clamp(max=2.0)
    return torch.sqrt(2.0 * l * e)
def chunks():
    out = np.empty((CH, N), dtype=np.int32)
    for s0 in range(0, S, CH):
        s1 = min(S, s0 + CH)
        ctx.call("pst_profile_keys", m, l, pr.k, s0, s1, _native.ptr(out, C.c_int32))
        yield s0, keys_to_d(torch.from_numpy(out[: s1 - s0]).cuda())
with ctx.using(x):
    a0 = []
    for s0, d in chunks():
        a0.append(d.sum(1).cpu())
    a0 = torch.cat(a0)
    best = int(a0.argmin())
    _, dbest = next((s0, d) for s0, d in chunks() if s0 <= best < s0 + CH)
    curve = dbest[best % CH].clone()
    area, lb = [], {B: [] for B in BS}
    for s0, d in chunks():
        area.append(torch.minimum(d, curve).sum(1).cpu())
        for B in BS:
            nb = (N + B - 1) // B
            pad = torch.nn.functional.pad(d, (0, nb * B - N), value=float("inf"))
            bm = pad.view(d.shape[0], nb, B).amin(2)
            lbv = torch.minimum(bm.repeat_interleave(B, 1)[:, :N], curve).sum(1)
            lb[B].append(lbv.cpu())
    area = torch.cat(area)
    area[best] = float("inf")
    amin = float(area.min())
    res = {"m": m, "S": S, "step": 1, "best0": best, "amin1": amin}
    for B in BS:
        v = torch.cat(lb[B]); v[best] = float("inf")
        res[f"cand_B{B}"] = int((v <= amin).sum())
        res[f"lb_gap_B{B}"] = float(((area - v) / area)[torch.isfinite(area)].mean())
    print(json.dumps(res), flush=True)
    # step 2: curve = min(curve, profile of the step-1 winner)
    best1 = int(area.argmin())
    _, d1 = next((s0, d) for s0, d in chunks() if s0 <= best1 < s0 + CH)
    curve = torch.minimum(curve, d1[best1 % CH])
    area, lb = [], {B: [] for B in BS}
    for s0, d in chunks():
        area.append(torch.minimum(d, curve).sum(1).cpu())
        for B in BS:
            nb = (N + B - 1) // B
            pad = torch.nn.functional.pad(d, (0, nb * B - N), value=float("inf"))
            bm = pad.view(d.shape[0], nb, B).amin(2)
            lb[B].append(torch.minimum(bm.repeat_interleave(B, 1)[:, :N], curve).sum(1).cpu())
    area = torch.cat(area)
    area[[best, best1]] = float("inf")
    amin = float(area.min())
    res = {"m": m, "S": S, "step": 2, "best1": best1, "amin2": amin}
    for B in BS:
        v = torch.cat(lb[B]); v[[best, best1]] = float("inf")
        res[f"cand_B{B}"] = int((v <= amin).sum())
    print(json.dumps(res), flush=True)
