"""Multi-GPU sharding: one process per GPU over torch.distributed (NCCL on GPUs, gloo in CPU tests).

Two partitions of the pair work:

* length sharding (``run_sharded``): the Karmarkar-Karp partition of the
  per-length jobs (weights = subsequence-pair counts) assigns rank r the
  lengths of part r; every rank runs its searches on its own GPU and the
  finished results are all-gathered.  No data-path collective is needed --
  lengths are independent (scheduler.py:383-397).
* segment-row sharding of ONE length (``ShardedSearch``): rank r owns a
  contiguous range of segments (their MPdist profiles stay in its HBM); the
  greedy rounds exchange one (area, index) pair per rank plus a broadcast of
  the chosen profile, and the nearest-segment attribution is two all-reduce
  MIN passes (value, then lowest index among value ties).  The combine logic
  is backend-agnostic so the CPU tests can drive it with gloo.

Everything is keyed by snippet length / segment index, so outputs are
identical for any number of GPUs.
"""

from __future__ import annotations

import time

import numpy as np


def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch always present in this image
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def world_size() -> int:
    d = _dist()
    return d.get_world_size() if d else 1


def rank() -> int:
    d = _dist()
    return d.get_rank() if d else 0


def length_partition(weights, parts: int):
    """KK partition of job weights into ``parts`` rank lists (empty lists allowed)."""
    from .scheduler import kk_partition

    parts_eff = max(1, min(parts, len(weights)))
    sched = kk_partition(weights, parts_eff)
    out = [list(a) for a in sched.assignments]
    out += [[] for _ in range(parts - len(out))]
    return out


def run_sharded(series, jobs, num_snippets, weights, runner=None):
    """Length sharding across the ranks of the default process group."""
    from .scheduler import run_jobs

    dist = _dist()
    ws, rk = world_size(), rank()
    parts = length_partition(weights, ws)
    mine = [jobs[i] for i in parts[rk]]
    run = runner or run_jobs
    local = run(series, mine, num_snippets) if mine else []
    gathered = [None] * ws
    dist.all_gather_object(gathered, local)
    out = []
    for g in gathered:
        out.extend(g)
    return out


def segment_ranges(S: int, parts: int):
    """Contiguous, balanced segment ranges (equal pair cost per segment)."""
    base, extra = divmod(S, parts)
    out, s0 = [], 0
    for r in range(parts):
        cnt = base + (1 if r < extra else 0)
        out.append((s0, s0 + cnt))
        s0 += cnt
    return out


class ShardedSearch:
    """Greedy snippet selection over segment rows split across ranks.

    ``backend`` provides the local (per-rank) device work:
      areas(curve|None) -> float64[n_local]   row sums of min(D, curve)
      row(i_local) -> float64[N]              one profile row
      colmin() -> (float64[N], int64[N])      per-window min and local first argmin
      rowmax() -> float                       max of the local rows
    and ``to_tensor`` / ``from_tensor`` move arrays to the collective device.
    """

    def __init__(self, backend, seg_lo: int, seg_hi: int, N: int, to_tensor, from_tensor):
        self.b = backend
        self.lo, self.hi, self.N = seg_lo, seg_hi, N
        self.T = to_tensor
        self.F = from_tensor

    def run(self, K: int):
        import torch

        dist = _dist()
        ws = world_size()
        chosen: list[int] = []
        taken = set()
        curve = None
        for _ in range(K):
            areas = self.b.areas(curve)
            best_a, best_i = np.inf, np.iinfo(np.int64).max
            for i, a in enumerate(areas):
                g = self.lo + i
                if g in taken:
                    continue
                if a < best_a or (a == best_a and g < best_i):
                    best_a, best_i = a, g
            cand = torch.tensor([best_a, float(best_i)], dtype=torch.float64)
            allc = [torch.zeros(2, dtype=torch.float64) for _ in range(ws)]
            dist.all_gather(allc, self.T(cand))
            pairs = [(float(self.F(c)[0]), int(self.F(c)[1])) for c in allc]
            ga, gi = min(pairs, key=lambda p: (p[0], p[1]))
            chosen.append(gi)
            taken.add(gi)
            owner = next(r for r in range(ws) if self._range(r)[0] <= gi < self._range(r)[1])
            row = self.b.row(gi - self.lo) if self.lo <= gi < self.hi else np.zeros(self.N)
            rt = self.T(torch.from_numpy(np.ascontiguousarray(row)))
            dist.broadcast(rt, src=owner)
            row = self.F(rt)
            curve = row.copy() if curve is None else np.minimum(curve, row)
        # nearest segment per window: MIN over values, then MIN over indices among ties
        mv, ma = self.b.colmin()
        mvt = self.T(torch.from_numpy(np.ascontiguousarray(mv)))
        dist.all_reduce(mvt, op=dist.ReduceOp.MIN)
        gmin = self.F(mvt)
        idx = np.where(mv == gmin, ma + self.lo, np.iinfo(np.int64).max).astype(np.int64)
        it = self.T(torch.from_numpy(idx))
        dist.all_reduce(it, op=dist.ReduceOp.MIN)
        nearest = self.F(it)
        pm = self.T(torch.tensor([self.b.rowmax()], dtype=torch.float64))
        dist.all_reduce(pm, op=dist.ReduceOp.MAX)
        return chosen, curve, nearest, float(self.F(pm)[0])

    def _range(self, r):
        return self.ranges[r]

    ranges: list = []


def timed(fn, *a, **kw):
    t0 = time.perf_counter()
    out = fn(*a, **kw)
    return out, time.perf_counter() - t0
