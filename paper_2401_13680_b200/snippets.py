"""Greedy snippet selection on the GPU (reference snippets.py).

``select_snippets`` computes all S = n//m MPdist profiles on the device
(csrc/mpdist.cu), runs the K greedy ProfileArea rounds, the nearest-segment
attribution and the per-point labels there (csrc/pastila.cu), and copies back
only the K chosen profiles, the curve, the per-segment counts and the window
attribution.  The S x N profile matrix never leaves the GPU.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .mpdist import MPdistParams, MPdistProfile, profiles_host
from .series import SlidingStats, TimeSeries


@dataclass(frozen=True)
class SegmentSet:
    """Non-overlapping length-m segments; the remainder n % m is not segmented."""

    snippet_size: int
    starts: np.ndarray

    @property
    def count(self) -> int:
        return int(self.starts.size)


@dataclass(frozen=True)
class Snippet:
    """A chosen segment, the windows it is nearest to, and their share (frac)."""

    index: int
    start: int
    length: int
    frac: float
    neighbors: np.ndarray


@dataclass(frozen=True)
class SnippetResult:
    """One snippet search (reference snippets.py:55-98), snippets in (-frac, index) order."""

    snippet_size: int
    window_size: int
    k: int
    series_length: int
    snippets: tuple[Snippet, ...]
    curve: np.ndarray
    profile_area: float
    profiles: tuple[MPdistProfile, ...]
    profile_max: float
    segment_window_counts: np.ndarray
    unassigned_windows: int
    # device-computed extras (not part of the reference field set's semantics)
    labels_: np.ndarray | None = field(default=None, repr=False, compare=False)
    criterion_: float | None = field(default=None, repr=False, compare=False)

    def to_dict(self) -> dict:
        return {
            "schema": 1,
            "m": self.snippet_size,
            "l": self.window_size,
            "k": self.k,
            "snippets": [
                {"index": s.index, "start": s.start, "frac": s.frac, "neighbor_count": int(s.neighbors.size)}
                for s in self.snippets
            ],
            "profile_area": self.profile_area,
        }


def segment(series: TimeSeries, snippet_size: int) -> SegmentSet:
    """Segments at i*m for i < n//m; at least two are required (snippets.py:101-116)."""
    if snippet_size < 2:
        raise ValueError(f"snippet size must be at least 2, got {snippet_size}")
    S = series.n // snippet_size
    if S < 2:
        raise ValueError(
            f"snippet size {snippet_size} leaves only {S} segment(s) of a series of length "
            f"{series.n}; need at least 2"
        )
    return SegmentSet(snippet_size=snippet_size, starts=np.arange(S, dtype=np.int64) * snippet_size)


def segment_profiles(series: TimeSeries, params: MPdistParams, stats: SlidingStats | None = None
                     ) -> list[MPdistProfile]:
    """All S segment profiles, computed in one device pass (snippets.py:119-128)."""
    segs = segment(series, params.snippet_size)
    if stats is not None and stats.window_len != params.window_size:
        raise ValueError(f"stats were built for window length {stats.window_len}, not {params.window_size}")
    D = profiles_host(series, params, 0, segs.count)
    return [MPdistProfile(segment_index=i, values=D[i]) for i in range(segs.count)]


def representativeness_curve(profiles) -> np.ndarray:
    """Pointwise minimum of a non-empty set of equal-length profiles (Eq. 16)."""
    arrs = [np.asarray(getattr(p, "values", p), dtype=np.float64) for p in profiles]
    if not arrs:
        raise ValueError("profile subset must be non-empty")
    width = arrs[0].size
    for i, a in enumerate(arrs):
        if a.size != width:
            raise ValueError(f"profile {i} has length {a.size}, expected {width}")
    return np.minimum.reduce(arrs)


def profile_area(curve) -> float:
    """Sum of a curve, the greedy objective (Eq. 17)."""
    c = np.asarray(curve, dtype=np.float64)
    if c.size == 0:
        raise ValueError("curve must be non-empty")
    return float(c.sum())


def _run(series: TimeSeries, params: MPdistParams, K: int, D: np.ndarray | None) -> SnippetResult:
    n, m = series.n, params.snippet_size
    S, N = n // m, n - m + 1
    idx = np.empty(K, dtype=np.int64)
    fracs = np.empty(K)
    curve = np.empty(N)
    prof = np.empty((K, N))
    counts = np.empty(S, dtype=np.int64)
    nearest = np.empty(N, dtype=np.int32)
    labels = np.empty(n, dtype=np.int64)
    out = _native.Snippets(
        _native.ptr(idx, _native.C.c_int64), _native.ptr(fracs), _native.ptr(curve), _native.ptr(prof),
        _native.ptr(counts, _native.C.c_int64), _native.ptr(nearest, _native.C.c_int32),
        _native.ptr(labels, _native.C.c_int64), 0.0, 0.0, 0.0, 0)
    with _native.context().using(series.values) as ctx:
        if D is None:
            ctx.call("pst_select_snippets", int(m), int(params.window_size), int(params.k), int(K),
                     _native.C.byref(out))
        else:
            ctx.call("pst_select_from_profiles", _native.ptr(D), int(S), int(N), int(n), int(K),
                     _native.C.byref(out))
    snippets = tuple(
        Snippet(index=int(i), start=int(i) * m, length=m, frac=float(f),
                neighbors=np.flatnonzero(nearest == i).astype(np.int64))
        for i, f in zip(idx, fracs)
    )
    return SnippetResult(
        snippet_size=m, window_size=params.window_size, k=params.k, series_length=n,
        snippets=snippets, curve=curve, profile_area=float(out.profile_area),
        profiles=tuple(MPdistProfile(segment_index=int(i), values=prof[r]) for r, i in enumerate(idx)),
        profile_max=float(out.profile_max), segment_window_counts=counts,
        unassigned_windows=int(out.unassigned), labels_=labels,
        criterion_=float(out.criterion) if K >= 2 else None,
    )


def select_snippets(series: TimeSeries, params: MPdistParams, num_snippets: int, *,
                    profiles: list[MPdistProfile] | None = None, stats: SlidingStats | None = None
                    ) -> SnippetResult:
    """The ``num_snippets`` segments that greedily minimize ProfileArea (snippets.py:154-244)."""
    segs = segment(series, params.snippet_size)
    if not 1 <= num_snippets <= segs.count:
        raise ValueError(f"snippet count {num_snippets} out of range [1, {segs.count}]")
    if stats is not None and stats.window_len != params.window_size:
        raise ValueError(f"stats were built for window length {stats.window_len}, not {params.window_size}")
    D = None
    if profiles is not None:
        if len(profiles) != segs.count:
            raise ValueError(f"got {len(profiles)} profiles for {segs.count} segments")
        D = np.ascontiguousarray(np.vstack([p.values for p in profiles]), dtype=np.float64)
    return _run(series, params, num_snippets, D)


def export_curve_csv(result: SnippetResult, path) -> None:
    np.savetxt(path, result.curve, fmt="%.17g")


def export_profiles_csv(result: SnippetResult, path) -> None:
    with open(path, "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow([f"segment_{p.segment_index}" for p in result.profiles])
        for row in np.column_stack([p.values for p in result.profiles]):
            wr.writerow([f"{v:.17g}" for v in row])
