"""Key path (csrc/mpdist.cu V = int, csrc/pastila.cu run_select_keys) on the GPU.

The fast profile pass stores the 32-bit key (high word of e = d^2/2l) of every
window's k-th smallest P_ABBA element; the selection certifies every decision
from the key buckets and resolves the rest with exact values.  These tests pin
the three properties that make its outputs identical to the exact path:
  1. every exact profile value lies in its key's bucket image [f(lo), f(hi)];
  2. the single-window evaluator is bit-identical to the full exact profiles;
  3. select_snippets on the key path == select_snippets on the exact path
     (PASTILA_EXACT=1), field by field, on data with and without exact ties.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk, two_regime_series

pytestmark = pytest.mark.gpu


def _keys(x, m, lo, hi):
    l, k = P.MPdistParams(m).window_size, P.MPdistParams(m).k
    n = x.size
    out = np.empty((hi - lo, n - m + 1), dtype=np.int32)
    with _native.context().using(x) as ctx:
        ctx.call("pst_profile_keys", m, l, k, lo, hi, _native.ptr(out, C.c_int32))
    return out


def _exact(x, m, lo, hi):
    l, k = P.MPdistParams(m).window_size, P.MPdistParams(m).k
    out = np.empty((hi - lo, x.size - m + 1))
    with _native.context().using(x) as ctx:
        ctx.call("pst_mpdist_profiles", m, l, k, lo, hi, _native.ptr(out))
    return out


def _window_exact(x, m, seg, win):
    l, k = P.MPdistParams(m).window_size, P.MPdistParams(m).k
    seg = np.ascontiguousarray(seg, dtype=np.int64)
    win = np.ascontiguousarray(win, dtype=np.int64)
    out = np.empty(seg.size)
    with _native.context().using(x) as ctx:
        ctx.call("pst_window_exact", m, l, k, _native.ptr(seg, C.c_int64), _native.ptr(win, C.c_int64),
                 seg.size, _native.ptr(out))
    return out


def _f(e, l):
    """e_to_dist (mpdist.cu) in numpy: same IEEE operations."""
    e = np.where(e < 1e-15, 0.0, e)
    e = np.where(e > 2.0, 2.0, e)
    return np.sqrt((2.0 * l) * e)


def _bucket(keys, l):
    k64 = keys.astype(np.int64)
    lo_bits = (k64 & 0xFFFFFFFF) << 32
    hi_bits = lo_bits | 0xFFFFFFFF
    lo = _f(lo_bits.astype(np.uint64).view(np.float64), l)
    hi = _f(hi_bits.astype(np.uint64).view(np.float64), l)
    neg = keys < 0
    return np.where(neg, 0.0, lo), np.where(neg, 0.0, hi)


@pytest.mark.parametrize("m", [16, 64, 120, 256, 512, 700])
def test_exact_profiles_lie_in_key_buckets(m):
    x, _ = planted_walk(24_000, m_act=120, A=3, seed=2)
    S = x.size // m
    lo, hi = 0, min(S, 12)
    K = _keys(x, m, lo, hi)
    D = _exact(x, m, lo, hi)
    blo, bhi = _bucket(K, P.MPdistParams(m).window_size)
    assert np.all(blo <= D) and np.all(D <= bhi)
    # the bucket is tight: 2^-20 relative in e, 2^-21 in d
    pos = D > 1e-3
    assert np.all((bhi[pos] - blo[pos]) <= 1e-6 * D[pos])


@pytest.mark.parametrize("m,n", [(64, 3000), (40, 2500), (300, 4000)])
def test_window_evaluator_bit_identical_everywhere(m, n):
    """Every (segment, window) of a small series, so every tile boundary is covered."""
    x, _ = planted_walk(n, m_act=50, A=3, seed=3)
    S, N = n // m, n - m + 1
    D = _exact(x, m, 0, S)
    seg, win = np.meshgrid(np.arange(S), np.arange(N), indexing="ij")
    got = _window_exact(x, m, seg.ravel(), win.ravel()).reshape(S, N)
    assert np.array_equal(got, D)


@pytest.mark.parametrize("m", [64, 256, 1024])
def test_window_evaluator_bit_identical_sampled(m):
    x, _ = planted_walk(60_000, m_act=256, A=4, seed=0)
    S, N = x.size // m, x.size - m + 1
    rng = np.random.default_rng(m)
    segs = rng.choice(S, size=min(S, 6), replace=False)
    D = _exact(x, m, 0, S)[segs]
    win = np.unique(np.concatenate([rng.integers(0, N, 400), [0, 1, N - 2, N - 1]]))
    for r, s in enumerate(segs):
        got = _window_exact(x, m, np.full(win.size, s), win)
        assert np.array_equal(got, D[r, win]), s


def _run(series, m, K, exact):
    old = os.environ.get("PASTILA_EXACT")
    os.environ["PASTILA_EXACT"] = "1" if exact else "0"
    try:
        return P.select_snippets(series, P.MPdistParams(m), K)
    finally:
        if old is None:
            del os.environ["PASTILA_EXACT"]
        else:
            os.environ["PASTILA_EXACT"] = old


def _same(a, b):
    assert [s.index for s in a.snippets] == [s.index for s in b.snippets]
    assert [s.frac for s in a.snippets] == [s.frac for s in b.snippets]
    for sa, sb in zip(a.snippets, b.snippets):
        assert np.array_equal(sa.neighbors, sb.neighbors)
    assert np.array_equal(a.segment_window_counts, b.segment_window_counts)
    assert a.unassigned_windows == b.unassigned_windows
    assert np.array_equal(a.curve, b.curve)
    for pa, pb in zip(a.profiles, b.profiles):
        assert np.array_equal(pa.values, pb.values)
    assert a.profile_area == b.profile_area
    assert a.profile_max == b.profile_max
    assert a.criterion_ == b.criterion_
    assert np.array_equal(a.labels_, b.labels_)


def _stats(reset=False):
    out = np.zeros(8, dtype=np.int64)
    _native.context().call("pst_cert_stats", _native.ptr(out, C.c_int64), 1 if reset else 0)
    return out


@pytest.mark.parametrize("case", ["planted", "random_walk", "two_regime_exact", "two_regime_noisy", "constant_tail"])
@pytest.mark.parametrize("m", [32, 96, 256])
def test_key_path_equals_exact_path(case, m):
    n = 30_000
    if case == "planted":
        x, _ = planted_walk(n, m_act=120, A=3, seed=5)
    elif case == "random_walk":
        x = np.cumsum(np.random.default_rng(7).standard_normal(n))
    elif case == "two_regime_exact":  # bit-identical repeats: exact ties everywhere
        x, _ = two_regime_series(n, period=32, block_len=64, noise=0.0)
    elif case == "two_regime_noisy":
        x, _ = two_regime_series(n, period=32, block_len=64, noise=0.1, seed=1)
    else:  # constant stretches: constant-window conventions and many equal values
        x, _ = planted_walk(n, m_act=120, A=3, seed=6)
        x[5000:9000] = 1.25
        x[20000:21000] = -3.0
    s = P.TimeSeries(x)
    _stats(reset=True)
    a = _run(s, m, 4, exact=False)
    st = _stats()
    b = _run(s, m, 4, exact=True)
    _same(a, b)
    assert st[0] == 1  # the key path ran (one length)
    if case in ("planted", "random_walk"):
        assert st[6] == 0  # no fallback to the exact path


def test_select_length_key_path_equals_exact_path():
    x, _ = planted_walk(40_000, m_act=120, A=3, seed=0)
    s = P.TimeSeries(x)
    grid = [64, 96, 128, 160]
    os.environ["PASTILA_EXACT"] = "1"
    try:
        rb, resb = P.select_length(s, grid, 3, training_log=False)
    finally:
        del os.environ["PASTILA_EXACT"]
    ra, resa = P.select_length(s, grid, 3, training_log=False)
    assert ra.m_best == rb.m_best
    assert [c.score for c in ra.candidates] == [c.score for c in rb.candidates]
    for m in grid:
        _same(resa[m], resb[m])


@pytest.mark.parametrize("chunk", ["1", "7", "64"])
@pytest.mark.parametrize("case", ["planted", "two_regime_exact"])
def test_streamed_key_path_equals_exact_path(monkeypatch, case, chunk):
    """Key matrix streamed in chunks of segments (C4 mode: max(K, 2) profile passes,
    attribution state accumulated across chunks, candidate pairs collected in pass 1)
    == the exact path, field by field."""
    n = 20_000
    if case == "planted":
        x, _ = planted_walk(n, m_act=120, A=3, seed=8)
    else:
        x, _ = two_regime_series(n, period=32, block_len=64, noise=0.0)
    s = P.TimeSeries(x)
    b = _run(s, 96, 3, exact=True)
    monkeypatch.setenv("PASTILA_STREAM_KEYS", chunk)
    _stats(reset=True)
    a = _run(s, 96, 3, exact=False)
    st = _stats()
    _same(a, b)
    assert st[0] == 1
    if case == "planted":
        assert st[6] == 0


def _prune_stats(reset=False):
    out = np.zeros(4, dtype=np.int64)
    _native.context().call("pst_prune_stats", _native.ptr(out, C.c_int64), 1 if reset else 0)
    return out


@pytest.mark.parametrize("chunk", ["1", "16"])
@pytest.mark.parametrize("case", ["planted", "random_walk", "two_regime_exact"])
def test_pruned_greedy_passes_equal_exact_path(monkeypatch, case, chunk):
    """Streamed key path with K = 5: passes 1..4 recompute only the rows whose
    block-minimum area bound can still win, pass 1 takes its candidate pairs
    from the block summaries (or a pass falls back to a full one); the result
    == the exact path, field by field, and == the unpruned run."""
    n = 40_000
    if case == "planted":
        x, _ = planted_walk(n, m_act=120, A=3, seed=11)
    elif case == "random_walk":
        x = np.cumsum(np.random.default_rng(12).standard_normal(n))
    else:
        x, _ = two_regime_series(n, period=32, block_len=64, noise=0.0)
    s = P.TimeSeries(x)
    m, K = 128, 5
    b = _run(s, m, K, exact=True)
    monkeypatch.setenv("PASTILA_STREAM_KEYS", chunk)
    _prune_stats(reset=True)
    _stats(reset=True)
    a = _run(s, m, K, exact=False)
    ps, st = _prune_stats(), _stats()
    _same(a, b)
    S = n // m
    if st[6] == 0:  # no certification cap exceeded (exact ties everywhere can exceed one)
        assert ps[0] + ps[2] == K - 1  # every pass >= 1 was pruned or fell back to a full pass
    if case != "two_regime_exact":
        assert st[6] == 0 and ps[0] == K - 1 and ps[1] < (K - 1) * S // 4
    print(case, chunk, "pruned passes", int(ps[0]), "rows", int(ps[1]), "of", (K - 1) * S, "fallbacks", int(ps[2]))
    monkeypatch.setenv("PASTILA_PRUNE", "0")
    _prune_stats(reset=True)
    c = _run(s, m, K, exact=False)
    assert _prune_stats()[0] == 0
    _same(a, c)


@pytest.mark.parametrize("K", [1, 2])
def test_pruned_pass1_small_K(monkeypatch, K):
    """K = 1 (pass 1 only collects pairs) and K = 2 (pass 1 = last greedy step)."""
    x, _ = planted_walk(30_000, m_act=120, A=3, seed=13)
    s = P.TimeSeries(x)
    b = _run(s, 96, K, exact=True)
    monkeypatch.setenv("PASTILA_STREAM_KEYS", "8")
    _prune_stats(reset=True)
    a = _run(s, 96, K, exact=False)
    ps = _prune_stats()
    _same(a, b)
    assert ps[0] + ps[2] == 1


def test_pruned_streamed_c3_length_with_uncertain_windows(monkeypatch):
    """The C3 series at m = 128 (17 attribution windows the key buckets leave
    uncertain, profiles/r02_c3_certificate.json): streamed with pruned passes
    1..3, pass 1's pairs taken from the block summaries == the resident key path."""
    x, _ = planted_walk(1_000_000, m_act=256, A=4, seed=0)
    s = P.TimeSeries(x)
    a = _run(s, 128, 4, exact=False)
    monkeypatch.setenv("PASTILA_STREAM_KEYS", "3000")
    _prune_stats(reset=True)
    _stats(reset=True)
    b = _run(s, 128, 4, exact=False)
    ps, st = _prune_stats(), _stats()
    _same(a, b)
    assert st[6] == 0 and st[3] > 0  # uncertain windows were resolved through the summary pairs
    assert ps[0] == 3 and ps[2] == 0
