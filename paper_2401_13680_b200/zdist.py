"""Z-normalized distance rows (reference zdist.py), computed on the GPU.

``distance_row`` / ``segment_distance_matrix`` call libpastila
``pst_distance_rows``: method "sliding" uses the centered diagonal recurrence
of the correlation identity, "direct" z-normalizes every window explicitly.
``znorm_distance`` compares two user-supplied windows and is a host helper
(not on the hot path; reference zdist.py:43-71).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .series import SlidingStats, TimeSeries


@dataclass(frozen=True)
class DistanceRow:
    """Distances from one segment window to every series window (zdist.py:30-40)."""

    row_index: int
    entries: np.ndarray


def _zn(v: np.ndarray) -> np.ndarray:
    sd = v.std()
    if sd == 0.0 or v.max() == v.min():
        return np.zeros_like(v)
    return (v - v.mean()) / sd


def znorm_distance(a, b) -> float:
    """Euclidean distance of population-z-normalized copies; constant -> zeros."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 1 or b.ndim != 1:
        raise ValueError("windows must be one-dimensional")
    if a.size != b.size:
        raise ValueError(f"window length mismatch: {a.size} vs {b.size}")
    if a.size == 0:
        raise ValueError("windows must be non-empty")
    return float(np.linalg.norm(_zn(a) - _zn(b)))


def _check_stats(stats: SlidingStats, l: int) -> None:
    if stats.window_len != l:
        raise ValueError(f"stats were built for window length {stats.window_len}, not {l}")


def _rows(series: TimeSeries, l: int, q0: int, rows: int, method: int) -> np.ndarray:
    out = np.empty((rows, series.n - l + 1))
    with _native.context().using(series.values) as ctx:
        ctx.call("pst_distance_rows", int(l), int(q0), int(rows), int(method), _native.ptr(out))
    return out


def distance_row(series: TimeSeries, stats: SlidingStats, seg_start: int, row_offset: int,
                 subseq_len: int, method: str = "sliding") -> DistanceRow:
    """Row ``row_offset`` of the segment starting at ``seg_start`` (zdist.py:138-188)."""
    _check_stats(stats, subseq_len)
    n = series.n
    q = seg_start + row_offset
    if seg_start < 0 or row_offset < 0 or q + subseq_len > n:
        raise ValueError(f"query window [{q}, {q + subseq_len}) is outside a series of length {n}")
    if method not in ("sliding", "direct"):
        raise ValueError(f"unknown method {method!r}, expected 'sliding' or 'direct'")
    row = _rows(series, subseq_len, q, 1, 0 if method == "sliding" else 1)[0]
    return DistanceRow(row_index=row_offset, entries=row)


def segment_distance_matrix(series: TimeSeries, stats: SlidingStats, seg_start: int,
                            snippet_size: int) -> np.ndarray:
    """ED_matr of one segment: (m-l+1) x (n-l+1) distances (zdist.py:191-225)."""
    l = stats.window_len
    n = series.n
    if snippet_size < l:
        raise ValueError(f"snippet size {snippet_size} is smaller than window length {l}")
    if seg_start < 0 or seg_start + snippet_size > n:
        raise ValueError(f"segment [{seg_start}, {seg_start + snippet_size}) is outside a series of length {n}")
    return _rows(series, l, seg_start, snippet_size - l + 1, 0)
