"""MPdist parameters, profile type and GPU profile computation (reference mpdist.py).

``mpdist_profile`` runs the fused tile kernel of csrc/mpdist.cu (distances,
column minima, row sliding minima and the exact k-th smallest of P_ABBA).
``column_minima``, ``row_sliding_minima`` and ``mpdist_at`` are the
reference's per-window contract helpers on caller-supplied arrays; they are
host utilities, not hot-path kernels (mpdist contract helpers).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .series import SlidingStats, TimeSeries


def default_window_size(snippet_size: int) -> int:
    """ceil(m/2), at least 1 (mpdist.py:26-28)."""
    return max(1, math.ceil(snippet_size / 2))


def default_order_stat(snippet_size: int) -> int:
    """ceil(0.05 * 2m), at least 1 (mpdist.py:31-33)."""
    return max(1, math.ceil(0.05 * 2 * snippet_size))


@dataclass(frozen=True)
class MPdistParams:
    """Snippet size m, inner window l, order statistic k (mpdist.py:36-72)."""

    snippet_size: int
    window_size: int | None = None
    k: int | None = None

    def __post_init__(self):
        m = self.snippet_size
        if m < 2:
            raise ValueError(f"snippet size must be at least 2, got {m}")
        if self.window_size is None:
            object.__setattr__(self, "window_size", default_window_size(m))
        if self.k is None:
            object.__setattr__(self, "k", default_order_stat(m))
        if not 1 <= self.window_size <= m:
            raise ValueError(f"window size {self.window_size} out of range [1, {m}]")
        if self.k < 1:
            raise ValueError(f"order statistic must be at least 1, got {self.k}")

    @property
    def profile_width(self) -> int:
        return self.snippet_size - self.window_size + 1


@dataclass(frozen=True)
class MPdistProfile:
    """MPdist of one segment against every window (mpdist.py:75-93)."""

    segment_index: int
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.float64)
        if v.ndim != 1 or v.size == 0:
            raise ValueError(f"profile must be a non-empty vector, got shape {v.shape}")
        if v.min() < 0:
            raise ValueError(f"profile entries must be non-negative, min is {v.min()}")
        v = v.copy()
        v.flags.writeable = False
        object.__setattr__(self, "values", v)

    def __len__(self) -> int:
        return int(self.values.size)


def _stack_rows(rows) -> np.ndarray:
    if isinstance(rows, np.ndarray) and rows.ndim == 2:
        return rows
    arrs = [np.asarray(getattr(r, "entries", r), dtype=np.float64) for r in rows]
    if not arrs:
        raise ValueError("no distance rows given")
    width = arrs[0].size
    for i, a in enumerate(arrs):
        if a.ndim != 1 or a.size != width:
            raise ValueError(f"row {i} has length {a.size}, expected {width}")
    return np.vstack(arrs)


def column_minima(rows) -> np.ndarray:
    """Column-wise minimum of distance rows (mpdist.py:112-118)."""
    return _stack_rows(rows).min(axis=0)


def row_sliding_minima(row, window: int) -> np.ndarray:
    """Minimum of every length-``window`` span (mpdist.py:121-143), van Herk blocks."""
    r = np.asarray(getattr(row, "entries", row), dtype=np.float64)
    if window < 1:
        raise ValueError(f"window must be at least 1, got {window}")
    if r.size < window:
        raise ValueError(f"window {window} larger than row of length {r.size}")
    nb = -(-r.size // window)
    pad = np.full(nb * window, np.inf)
    pad[:r.size] = r
    blocks = pad.reshape(nb, window)
    pre = np.minimum.accumulate(blocks, axis=1).ravel()
    suf = np.minimum.accumulate(blocks[:, ::-1], axis=1)[:, ::-1].ravel()
    cnt = r.size - window + 1
    j = np.arange(cnt)
    return np.minimum(suf[j], pre[j + window - 1])


def mpdist_at(ab_part, ba_part, params: MPdistParams) -> float:
    """k-th smallest of one window's concatenated profile halves (mpdist.py:154-176)."""
    ab = np.asarray(getattr(ab_part, "entries", ab_part), dtype=np.float64)
    ba = np.asarray(ba_part, dtype=np.float64)
    if ab.size != ba.size:
        raise ValueError(f"profile halves differ in length: {ab.size} vs {ba.size}")
    if ab.size != params.profile_width:
        raise ValueError(f"profile halves have {ab.size} entries, expected {params.profile_width}")
    both = np.concatenate([ab, ba])
    if both.size > params.k:
        return float(np.partition(both, params.k - 1)[params.k - 1])
    return float(both.max())


def _check_profile_args(series: TimeSeries, params: MPdistParams, stats) -> None:
    if params.snippet_size > series.n:
        raise ValueError(f"snippet size {params.snippet_size} exceeds series length {series.n}")
    if stats is not None and stats.window_len != params.window_size:
        raise ValueError(
            f"stats were built for window length {stats.window_len}, not {params.window_size}"
        )


def profiles_host(series: TimeSeries, params: MPdistParams, seg_lo: int, seg_hi: int) -> np.ndarray:
    """Profiles of segments [seg_lo, seg_hi) computed on the GPU, copied to host."""
    N = series.n - params.snippet_size + 1
    out = np.empty((seg_hi - seg_lo, N))
    with _native.context().using(series.values) as ctx:
        ctx.call("pst_mpdist_profiles", int(params.snippet_size), int(params.window_size), int(params.k),
                 int(seg_lo), int(seg_hi), _native.ptr(out))
    return out


def mpdist_profile(series: TimeSeries, segment_index: int, params: MPdistParams,
                   stats: SlidingStats | None = None) -> MPdistProfile:
    """MPdist profile of segment ``segment_index`` against every window (mpdist.py:179-232)."""
    _check_profile_args(series, params, stats)
    S = series.n // params.snippet_size
    if not 0 <= segment_index < S:
        raise ValueError(f"segment index {segment_index} out of range [0, {S})")
    vals = profiles_host(series, params, segment_index, segment_index + 1)[0]
    return MPdistProfile(segment_index=segment_index, values=vals)
