"""CPU oracle for the PaSTiLa hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the reference algorithm of
sniplab (arXiv 2401.13680 reference, /root/reference/pkg/src/sniplab).  It is
the checker for the CUDA path and the CPU baseline leg of ``bench.py``; the
product package (``paper_2401_13680_b200``) never imports it.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may use it.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function below
against golden vectors produced by the real reference
(``tests/golden/make_golden.py``); the restatement uses the same floating-point
operation order as the reference, so stats, distance rows and profiles agree
bit-for-bit on this machine (BLAS dot order aside).

Each function cites the reference lines it follows.
"""

from __future__ import annotations

import math
from itertools import combinations

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view
from scipy.ndimage import maximum_filter1d, minimum_filter1d


# ----------------------------------------------------------------- parameters
def window_default(m: int) -> int:
    """l = max(1, ceil(m/2))  -- mpdist.py:26-28."""
    return max(1, math.ceil(m / 2))


def order_default(m: int) -> int:
    """k = max(1, ceil(0.05*2*m))  -- mpdist.py:31-33."""
    return max(1, math.ceil(0.05 * 2 * m))


# ------------------------------------------------------------------ statistics
def sliding_stats(x: np.ndarray, l: int):
    """(means, stds, variances) of every length-l window -- series.py:152-190.

    Sequential prefix sums of x and x*x, variance clamped at 0, exact 0 for
    windows whose sliding max equals their sliding min.
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.size
    if not 1 <= l <= n:
        raise ValueError(f"window length {l} out of range [1, {n}]")
    s1 = np.zeros(n + 1)
    s2 = np.zeros(n + 1)
    np.cumsum(x, out=s1[1:])
    np.cumsum(x * x, out=s2[1:])
    mu = (s1[l:] - s1[:-l]) / l
    var = (s2[l:] - s2[:-l]) / l - mu * mu
    np.maximum(var, 0.0, out=var)
    cnt = n - l + 1
    half = l // 2
    flat = (minimum_filter1d(x, l, mode="nearest")[half:half + cnt]
            == maximum_filter1d(x, l, mode="nearest")[half:half + cnt])
    var[flat] = 0.0
    return mu, np.sqrt(var), var


# ------------------------------------------------------------ distance rows
def _row_from_dots(qt, mu, var, q, l):
    """Correlation-identity distances for one query -- zdist.py:98-123."""
    flat = var == 0.0
    if var[q] == 0.0:
        row = np.where(flat, 0.0, np.sqrt(l))
    else:
        cov = qt / l - mu[q] * mu
        with np.errstate(divide="ignore", invalid="ignore"):
            rho = cov / np.sqrt(var[q] * var)
        rho = np.clip(rho, -1.0, 1.0)
        row = np.sqrt(2.0 * l * (1.0 - rho))
        if flat.any():
            row[flat] = np.sqrt(l)
    row[q] = 0.0
    return row


def distance_block(x, mu, var, q0, rows, l):
    """ED_matr rows q0..q0+rows-1 against every window -- zdist.py:74-95, 191-225.

    Row 0 is a full sliding dot product; later rows use the diagonal update
    QT_i[c] = QT_{i-1}[c-1] - x[q-1]x[c-1] + x[q+l-1]x[c+l-1] with a fresh dot
    product in column 0.
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.size
    win = sliding_window_view(x, l)
    out = np.empty((rows, n - l + 1))
    qt = win @ x[q0:q0 + l]
    out[0] = _row_from_dots(qt, mu, var, q0, l)
    for i in range(1, rows):
        q = q0 + i
        nxt = np.empty_like(qt)
        nxt[0] = x[q:q + l] @ x[:l]
        nxt[1:] = qt[:-1] - x[q - 1] * x[:n - l] + x[q + l - 1] * x[l:]
        qt = nxt
        out[i] = _row_from_dots(qt, mu, var, q, l)
    return out


def znorm_direct_row(x, q, l):
    """Distance row by explicit z-normalization (oracles.py-style brute force)."""
    x = np.asarray(x, dtype=np.float64)
    win = sliding_window_view(x, l)
    mean = win.mean(axis=1, keepdims=True)
    std = win.std(axis=1, keepdims=True)
    flat = win.max(axis=1, keepdims=True) == win.min(axis=1, keepdims=True)
    z = np.where(flat, 0.0, (win - mean) / np.where(flat, 1.0, std))
    return np.linalg.norm(z - z[q], axis=1)


# ------------------------------------------------------------------ MPdist
def mpdist_profile(x, seg, m, l, k, stats=None, col_chunk: int | None = None):
    """MPdist profile of segment ``seg`` -- mpdist.py:179-232.

    P_ABBA per window j: w row minima over [j, j+w) and the column minima of
    columns j..j+w-1; the k-th smallest (1-based) if 2w > k else the max.
    ``col_chunk`` bounds memory by processing windows in chunks (identical
    values: each chunk carries its w-1 column halo).
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.size
    if stats is None:
        stats = sliding_stats(x, l)
    mu, _, var = stats
    w = m - l + 1
    N = n - m + 1
    rows = distance_block(x, mu, var, seg * m, w, l)          # w x N_l
    colmin = rows.min(axis=0)                                 # allP_BA  (mpdist.py:224)
    chunk = N if col_chunk is None else col_chunk
    out = np.empty(N)
    for j0 in range(0, N, chunk):
        j1 = min(N, j0 + chunk)
        sub = rows[:, j0:j1 + w - 1]
        ab = minimum_filter1d(sub, size=w, axis=-1, mode="nearest")[:, w // 2: w // 2 + (j1 - j0)]
        ba = sliding_window_view(colmin[j0:j1 + w - 1], w).T     # w x (j1-j0)
        merged = np.concatenate([ab, ba], axis=0)
        if merged.shape[0] > k:
            out[j0:j1] = np.partition(merged, k - 1, axis=0)[k - 1]
        else:
            out[j0:j1] = merged.max(axis=0)
    return out


def all_profiles(x, m, l, k):
    """Profiles of all S = n//m segments stacked (snippets.py:119-128, 198)."""
    st = sliding_stats(x, l)
    S = len(x) // m
    return np.vstack([mpdist_profile(x, s, m, l, k, st) for s in range(S)])


# ------------------------------------------------------------------ snippets
def greedy_pick(D, K):
    """K rounds of argmin_s sum_j min(D[s], curve) -- snippets.py:201-210."""
    S, N = D.shape
    taken = np.zeros(S, dtype=bool)
    curve = np.full(N, np.inf)
    chosen = []
    for _ in range(K):
        areas = np.minimum(D, curve).sum(axis=1)
        areas[taken] = np.inf
        b = int(np.argmin(areas))
        chosen.append(b)
        taken[b] = True
        curve = np.minimum(curve, D[b])
    return chosen, curve


def select_snippets(x, m, K, l=None, k=None, D=None):
    """Greedy snippets + nearest-segment attribution -- snippets.py:154-244."""
    x = np.asarray(x, dtype=np.float64)
    l = window_default(m) if l is None else l
    k = order_default(m) if k is None else k
    if D is None:
        D = all_profiles(x, m, l, k)
    S, N = D.shape
    chosen, curve = greedy_pick(D, K)
    nearest = np.argmin(D, axis=0)
    counts = np.bincount(nearest, minlength=S)
    snips = [(c, c * m, counts[c] / N, np.flatnonzero(nearest == c)) for c in chosen]
    snips.sort(key=lambda s: (-s[2], s[0]))
    return {
        "indices": [s[0] for s in snips],
        "starts": [s[1] for s in snips],
        "fracs": [s[2] for s in snips],
        "neighbors": [s[3] for s in snips],
        "curve": curve,
        "profile_area": float(curve.sum()),
        "profiles": D[[s[0] for s in snips]],
        "profile_max": float(D.max()),
        "counts": counts,
        "unassigned_windows": int(N - counts[chosen].sum()),
        "nearest": nearest,
    }


def criterion(profiles, profile_max):
    """Eq. 18: pairwise L1 separation over profile_max -- length_select.py:56-87."""
    if len(profiles) < 2:
        raise ValueError("separation needs at least 2 snippets")
    if profile_max == 0.0:
        return 0.0
    tot = 0.0
    for a, b in combinations(range(len(profiles)), 2):
        tot += float(np.abs(profiles[a] - profiles[b]).sum())
    return tot / profile_max


def labels(profiles, n):
    """Window argmin over the ordered profiles, tail copies the last -- labeling.py:114-118."""
    lab = np.argmin(np.vstack(profiles), axis=0)
    out = np.empty(n, dtype=np.int64)
    out[:lab.size] = lab
    out[lab.size:] = lab[-1]
    return out


def select_length(x, grid, K, window_rule=window_default):
    """One search per m, argmax of (score, -m) -- length_select.py:116-182."""
    cands = []
    results = {}
    for m in grid:
        r = select_snippets(x, m, K, l=window_rule(m))
        results[m] = r
        cands.append((m, criterion(r["profiles"], r["profile_max"]), r["profile_area"]))
    best = max(cands, key=lambda c: (c[1], -c[0]))
    return best[0], cands, results
