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
    """Greedy snippet selection over segment rows split across ranks (one length).

    ``backend`` provides the rank-local work on its rows [seg_lo, seg_hi):
      areas(curve | None) -> float64[n_local]   row sums of min(D, curve)
      row(i_local) -> float64[N]                one profile row
      colmin() -> (float64[N], int64[N])        per-window min, local first argmin
      rowmax() -> float                         max over the local rows
    ``to_dev`` / ``from_dev`` move numpy arrays to / from the collective's device
    (CUDA tensors under NCCL, CPU tensors under gloo).
    """

    def __init__(self, backend, ranges, N: int, to_dev, from_dev):
        self.b = backend
        self.ranges = list(ranges)
        self.lo, self.hi = self.ranges[rank()]
        self.N = N
        self.to_dev = to_dev
        self.from_dev = from_dev

    def run(self, K: int):
        import torch

        dist = _dist()
        ws = world_size()
        chosen: list[int] = []
        self.chosen_rows = []  # profiles of the chosen segments, in greedy order
        curve = None
        for _ in range(K):
            # local best (lowest index among equal areas), then global (area, index) minimum
            areas = np.asarray(self.b.areas(curve), dtype=np.float64)
            best_a, best_i = np.inf, np.iinfo(np.int64).max
            for i, a in enumerate(areas):
                g = self.lo + i
                if g in chosen:
                    continue
                if a < best_a or (a == best_a and g < best_i):
                    best_a, best_i = float(a), g
            cand = self.to_dev(np.array([best_a, float(best_i)]))
            allc = [self.to_dev(np.zeros(2)) for _ in range(ws)]
            dist.all_gather(allc, cand)
            pairs = [tuple(self.from_dev(c)) for c in allc]
            ga, gi = min(pairs, key=lambda t: (t[0], t[1]))
            gi = int(gi)
            chosen.append(gi)
            owner = next(r for r, (lo, hi) in enumerate(self.ranges) if lo <= gi < hi)
            row = self.b.row(gi - self.lo) if owner == rank() else np.zeros(self.N)
            rt = self.to_dev(np.ascontiguousarray(row, dtype=np.float64))
            dist.broadcast(rt, src=owner)
            row = self.from_dev(rt)
            self.chosen_rows.append(np.array(row, dtype=np.float64, copy=True))
            curve = row.copy() if curve is None else np.minimum(curve, row)
        # nearest segment per window: MIN over values, then MIN over indices among ties
        mv, ma = self.b.colmin()
        mv = np.array(mv, dtype=np.float64, copy=True)
        mvt = self.to_dev(mv.copy())  # reduced in place: keep the local minima
        dist.all_reduce(mvt, op=dist.ReduceOp.MIN)
        gmin = self.from_dev(mvt)
        idx = np.where(mv == gmin, np.asarray(ma, dtype=np.int64) + self.lo, np.iinfo(np.int64).max)
        it = self.to_dev(idx.astype(np.int64, copy=True))
        dist.all_reduce(it, op=dist.ReduceOp.MIN)
        nearest = self.from_dev(it).astype(np.int64)
        pm = self.to_dev(np.array([self.b.rowmax()], dtype=np.float64))
        dist.all_reduce(pm, op=dist.ReduceOp.MAX)
        return chosen, curve, nearest, float(self.from_dev(pm)[0])


class DeviceRows:
    """ShardedSearch backend on this rank's GPU: the rank's segment profiles live
    in a device matrix filled by the profile kernels (pst_profiles_dev); areas and
    per-window minima run on the device (pst_areas_dev / pst_colmin_dev)."""

    def __init__(self, series, params, seg_lo: int, seg_hi: int):
        import ctypes as C

        import torch

        from . import _native

        self.C = C
        self.ctx = _native.context()
        self.dev = torch.device("cuda", self.ctx.device)
        n, m = series.n, params.snippet_size
        self.N = n - m + 1
        self.rows = seg_hi - seg_lo
        self.D = torch.empty((self.rows, self.N), dtype=torch.float64, device=self.dev)
        if self.rows == 0:  # more ranks than segments: this rank owns none
            return
        torch.cuda.synchronize(self.dev)  # D allocated on torch's stream, written on the library's
        with self.ctx.using(series.values):
            self.ctx.call("pst_profiles_dev", int(m), int(params.window_size), int(params.k), int(seg_lo),
                          int(seg_hi), C.c_void_p(self.D.data_ptr()), C.c_int64(self.N))
            self.ctx.call("pst_sync")

    def areas(self, curve):
        import torch

        out = torch.empty(self.rows, dtype=torch.float64, device=self.dev)
        if self.rows == 0:
            return out.cpu().numpy()
        cptr = None
        if curve is not None:
            ct = torch.as_tensor(curve, dtype=torch.float64, device=self.dev)
            cptr = self.C.c_void_p(ct.data_ptr())
        torch.cuda.synchronize(self.dev)  # inputs written on torch's stream
        self.ctx.call("pst_areas_dev", self.C.c_void_p(self.D.data_ptr()), self.C.c_int64(self.rows),
                      self.C.c_int64(self.N), self.C.c_int64(self.N), cptr, self.C.c_void_p(out.data_ptr()))
        self.ctx.call("pst_sync")
        return out.cpu().numpy()

    def row(self, i):
        return self.D[i].cpu().numpy()

    # device-resident variants for the library NCCL path (DeviceShardedSearch)
    def areas_dev(self, curve_t):
        import torch

        out = torch.empty(self.rows, dtype=torch.float64, device=self.dev)
        if self.rows:
            cptr = self.C.c_void_p(curve_t.data_ptr()) if curve_t is not None else None
            self.ctx.call("pst_areas_dev", self.C.c_void_p(self.D.data_ptr()), self.C.c_int64(self.rows),
                          self.C.c_int64(self.N), self.C.c_int64(self.N), cptr, self.C.c_void_p(out.data_ptr()))
        return out

    def row_dev(self, i):
        return self.D[i]

    def colmin_dev(self):
        import torch

        mv = torch.full((self.N,), float("inf"), dtype=torch.float64, device=self.dev)
        ma = torch.zeros(self.N, dtype=torch.int32, device=self.dev)
        torch.cuda.synchronize(self.dev)
        if self.rows:
            self.ctx.call("pst_colmin_dev", self.C.c_void_p(self.D.data_ptr()), self.C.c_int64(self.rows),
                          self.C.c_int64(self.N), self.C.c_int64(self.N), self.C.c_int64(0),
                          self.C.c_void_p(mv.data_ptr()), self.C.c_void_p(ma.data_ptr()))
            self.ctx.call("pst_sync")  # the caller may touch them on torch's stream
        return mv, ma

    def colmin(self):
        import torch

        if self.rows == 0:
            return np.full(self.N, np.inf), np.zeros(self.N, dtype=np.int64)
        mv = torch.empty(self.N, dtype=torch.float64, device=self.dev)
        ma = torch.empty(self.N, dtype=torch.int32, device=self.dev)
        self.ctx.call("pst_colmin_dev", self.C.c_void_p(self.D.data_ptr()), self.C.c_int64(self.rows),
                      self.C.c_int64(self.N), self.C.c_int64(self.N), self.C.c_int64(0),
                      self.C.c_void_p(mv.data_ptr()), self.C.c_void_p(ma.data_ptr()))
        self.ctx.call("pst_sync")
        return mv.cpu().numpy(), ma.cpu().numpy().astype(np.int64)

    def rowmax(self):
        import torch

        if not self.rows:
            return 0.0
        out = torch.empty(1, dtype=torch.float64, device=self.dev)
        self.ctx.call("pst_max_dev", self.C.c_void_p(self.D.data_ptr()), self.C.c_int64(self.rows),
                      self.C.c_int64(self.N), self.C.c_int64(self.N), self.C.c_void_p(out.data_ptr()))
        self.ctx.call("pst_sync")
        return float(out.item())


class StreamedRows:
    """ShardedSearch backend for rank-local segment rows that do not fit HBM
    (C4: n = 1e7, 39,062 segments of 1e7 windows = 3.1 TB): every areas() call
    recomputes the rank's profiles in device-sized chunks and reduces them on
    the fly (pst_profile_reduce_dev); the first call also yields the
    per-window minima and the row max, row(i) recomputes one profile.  Same
    values as DeviceRows (profiles do not depend on the chunking)."""

    def __init__(self, series, params, seg_lo: int, seg_hi: int):
        import ctypes as C

        import torch

        from . import _native

        self.C, self.torch = C, torch
        self.ctx = _native.context()
        self.values = series.values
        self.dev = torch.device("cuda", self.ctx.device)
        self.p = params
        self.lo, self.hi = seg_lo, seg_hi
        self.N = series.n - params.snippet_size + 1
        self.rows = seg_hi - seg_lo
        self._colmin = None
        self._rowmax = None

    def _mkl(self):
        return int(self.p.snippet_size), int(self.p.window_size), int(self.p.k)

    def areas(self, curve):
        torch, C = self.torch, self.C
        out = torch.empty(self.rows, dtype=torch.float64, device=self.dev)
        if self.rows == 0:
            self._colmin = (np.full(self.N, np.inf), np.zeros(self.N, dtype=np.int64))
            self._rowmax = 0.0
            return out.cpu().numpy()
        cptr = mv = ma = mx = None
        if curve is not None:
            ct = torch.as_tensor(curve, dtype=torch.float64, device=self.dev)
            cptr = C.c_void_p(ct.data_ptr())
        first = self._colmin is None
        if first:
            mvt = torch.full((self.N,), float("inf"), dtype=torch.float64, device=self.dev)
            mat = torch.zeros(self.N, dtype=torch.int32, device=self.dev)
            mxt = torch.zeros(1, dtype=torch.float64, device=self.dev)
            mv, ma, mx = (C.c_void_p(t.data_ptr()) for t in (mvt, mat, mxt))
        torch.cuda.synchronize(self.dev)  # filled on torch's stream, reduced on the library's
        with self.ctx.using(self.values):
            self.ctx.call("pst_profile_reduce_dev", *self._mkl(), self.lo, self.hi, cptr,
                          C.c_void_p(out.data_ptr()), mv, ma, mx)
            self.ctx.call("pst_sync")
        if first:
            self._colmin = (mvt.cpu().numpy(), mat.cpu().numpy().astype(np.int64) - self.lo)
            self._rowmax = float(mxt.item())
        return out.cpu().numpy()

    def row(self, i):
        torch, C = self.torch, self.C
        r = torch.empty((1, self.N), dtype=torch.float64, device=self.dev)
        s = self.lo + int(i)
        with self.ctx.using(self.values):
            self.ctx.call("pst_profiles_dev", *self._mkl(), s, s + 1, C.c_void_p(r.data_ptr()),
                          C.c_int64(self.N))
            self.ctx.call("pst_sync")
        return r[0].cpu().numpy()

    def colmin(self):
        if self._colmin is None:
            self.areas(None)
        return self._colmin

    def rowmax(self):
        if self._rowmax is None:
            self.areas(None)
        return self._rowmax if self.rows else 0.0

    # device-resident variants for the library NCCL path (DeviceShardedSearch)
    def areas_dev(self, curve_t):
        torch = self.torch
        curve = None if curve_t is None else curve_t.cpu().numpy()
        return torch.as_tensor(self.areas(curve), device=self.dev)

    def row_dev(self, i):
        return self.torch.as_tensor(self.row(i), device=self.dev)

    def colmin_dev(self):
        mv, ma = self.colmin()
        torch = self.torch
        return (torch.as_tensor(mv, dtype=torch.float64, device=self.dev),
                torch.as_tensor(ma, dtype=torch.int32, device=self.dev))


class LibComm:
    """NCCL communicator owned by libpastila (csrc/comm.cu, pst_comm_*): the
    collectives of the sharded search run inside the library, on its stream,
    on device buffers.  Bootstrap only goes through torch.distributed: rank 0's
    128-byte ncclUniqueId is broadcast as an object.  One per context."""

    _by_ctx: dict = {}

    def __init__(self):
        import ctypes as C

        from . import _native

        self.C, self.ctx = C, _native.context()
        self.ws, self.rk = world_size(), rank()
        uid = C.create_string_buffer(128)
        if self.rk == 0:
            _native._check(_native.load_library().pst_comm_unique_id(uid), "pst_comm_unique_id")
        raw = uid.raw
        if self.ws > 1:
            obj = [raw]
            _dist().broadcast_object_list(obj, src=0)
            raw = obj[0]
        self.ctx.call("pst_comm_init", raw, self.ws, self.rk)

    @classmethod
    def get(cls):
        from . import _native

        key = (id(_native.context()), world_size(), rank())
        c = cls._by_ctx.get(key)
        if c is None:
            c = cls._by_ctx[key] = cls()
        return c

    def p(self, t):
        return self.C.c_void_p(t.data_ptr())

    def all_gather(self, send, recv):
        self.ctx.call("pst_comm_allgather", self.p(send), self.p(recv), send.numel() * send.element_size())

    def broadcast(self, t, root):
        self.ctx.call("pst_comm_broadcast", self.p(t), t.numel() * t.element_size(), int(root))

    def all_reduce(self, t, op):  # op: "min" | "max"
        import torch

        dtype = {torch.float64: 0, torch.int64: 1, torch.int32: 2}[t.dtype]
        self.ctx.call("pst_comm_allreduce", self.p(t), t.numel(), dtype, {"min": 0, "max": 1, "sum": 2}[op])


class DeviceShardedSearch:
    """ShardedSearch with every per-step and per-window quantity on the device:
    local best (pst_local_best_dev), all-gather of the (area, index) pairs and the
    global pick (pst_pick_global_dev), broadcast of the chosen profile from its
    owner, curve update (pst_curve_min_dev), attribution by all-reduce MIN of the
    minima then of the tie indices (pst_tie_index_dev), profile_max by all-reduce
    MAX -- all through LibComm.  Host traffic: one 16-byte pick per step and the
    final outputs."""

    def __init__(self, backend, ranges, N: int, comm: LibComm):
        self.b, self.ranges, self.N, self.comm = backend, list(ranges), N, comm
        self.lo, self.hi = self.ranges[comm.rk]

    def run(self, K: int):
        import torch

        C, ctx, comm = self.comm.C, self.comm.ctx, self.comm
        dev = torch.device("cuda", ctx.device)
        rows, N, ws = self.hi - self.lo, self.N, comm.ws
        taken = torch.zeros(max(rows, 1), dtype=torch.uint8, device=dev)
        pair = torch.tensor([float("inf"), 9.0e18], dtype=torch.float64, device=dev)
        pairs = torch.empty(2 * ws, dtype=torch.float64, device=dev)
        pick = torch.empty(2, dtype=torch.float64, device=dev)
        curve = torch.empty(N, dtype=torch.float64, device=dev)
        torch.cuda.synchronize(dev)  # torch-filled buffers, library stream from here on
        chosen, self.chosen_rows = [], []
        for step in range(K):
            areas = self.b.areas_dev(curve if step else None)
            if rows:
                ctx.call("pst_local_best_dev", comm.p(areas), comm.p(taken), rows, self.lo, comm.p(pair))
            comm.all_gather(pair, pairs)
            ctx.call("pst_pick_global_dev", comm.p(pairs), ws, self.lo, rows, comm.p(taken), comm.p(pick))
            ctx.call("pst_sync")
            gi = int(pick[1].item())
            chosen.append(gi)
            owner = next(r for r, (lo, hi) in enumerate(self.ranges) if lo <= gi < hi)
            if owner == comm.rk:
                row = self.b.row_dev(gi - self.lo).contiguous()
            else:
                row = torch.empty(N, dtype=torch.float64, device=dev)
            torch.cuda.synchronize(dev)
            comm.broadcast(row, owner)
            ctx.call("pst_curve_min_dev", comm.p(curve), comm.p(row), N, 1 if step == 0 else 0)
            self.chosen_rows.append(row)
        mv, ma = self.b.colmin_dev()
        gmin = mv.clone()
        torch.cuda.synchronize(dev)
        comm.all_reduce(gmin, "min")
        idx = torch.empty(N, dtype=torch.int64, device=dev)
        ctx.call("pst_tie_index_dev", comm.p(mv), comm.p(gmin), comm.p(ma), self.lo, N, comm.p(idx))
        comm.all_reduce(idx, "min")
        pm = torch.tensor([self.b.rowmax()], dtype=torch.float64, device=dev)
        torch.cuda.synchronize(dev)
        comm.all_reduce(pm, "max")
        ctx.call("pst_sync")
        self.chosen_rows = [r.cpu().numpy() for r in self.chosen_rows]
        return chosen, curve.cpu().numpy(), idx.cpu().numpy(), float(pm.item())


def select_snippets_sharded(series, params, num_snippets: int, *, backend=None, comm=None):
    """``select_snippets`` for ONE length with its segment rows sharded over the
    ranks of the default process group: rank r owns a
    contiguous segment range, keeps its profiles in HBM when they fit
    (DeviceRows) or recomputes them per greedy round (StreamedRows), and the
    ranks combine through ShardedSearch (NCCL on GPUs, gloo in CPU tests).
    Every rank returns the same SnippetResult as the single-GPU call."""
    import torch

    from .mpdist import MPdistProfile
    from .snippets import Snippet, SnippetResult, segment

    segs = segment(series, params.snippet_size)
    S, K, n, m = segs.count, int(num_snippets), series.n, params.snippet_size
    if not 1 <= K <= S:
        raise ValueError(f"snippet count {K} out of range [1, {S}]")
    N = n - m + 1
    ranges = segment_ranges(S, world_size())
    lo, hi = ranges[rank()]
    if backend is None:
        from . import _native

        dev = _native.context().device
        free = torch.cuda.mem_get_info(dev)[0]
        fits = (hi - lo) * N * 8 + (16 << 30) < free
        backend = (DeviceRows if fits else StreamedRows)(series, params, lo, hi)
    d = _dist()
    on_gpu = d is not None and d.get_backend() == "nccl"
    if on_gpu:  # the collectives run on the GPU of this rank's library context
        from . import _native

        tdev = torch.device("cuda", _native.context().device)
        torch.cuda.set_device(tdev)
    else:
        tdev = torch.device("cpu")

    def to_dev(a):
        return torch.as_tensor(np.ascontiguousarray(a)).to(tdev)

    def from_dev(t):
        return t.cpu().numpy()

    if comm is None:  # default: the library's NCCL on GPUs; PASTILA_COMM=torch selects torch.distributed (A/B)
        import os

        comm = os.environ.get("PASTILA_COMM", "lib" if on_gpu else "torch")
    if comm == "lib":  # library-owned NCCL data plane
        ss = DeviceShardedSearch(backend, ranges, N, LibComm.get())
    else:  # torch.distributed collectives (gloo CPU tests)
        ss = ShardedSearch(backend, ranges, N, to_dev, from_dev)
    chosen, curve, nearest, pmax = ss.run(K)
    counts = np.bincount(nearest, minlength=S).astype(np.int64)
    order = sorted(range(K), key=lambda r: (-(counts[chosen[r]] / N), chosen[r]))  # snippets.py:228
    snippets = tuple(Snippet(index=int(chosen[r]), start=int(chosen[r]) * m, length=m,
                             frac=float(counts[chosen[r]] / N),
                             neighbors=np.flatnonzero(nearest == chosen[r]).astype(np.int64)) for r in order)
    profiles = tuple(MPdistProfile(segment_index=int(chosen[r]), values=ss.chosen_rows[r]) for r in order)
    return SnippetResult(
        snippet_size=m, window_size=params.window_size, k=params.k, series_length=n, snippets=snippets,
        curve=curve, profile_area=curve_area(curve), profiles=profiles, profile_max=float(pmax),
        segment_window_counts=counts, unassigned_windows=int(N - sum(counts[c] for c in chosen)))


def curve_area(curve) -> float:
    """profile_area with the same device reduction as the single-GPU search
    (pst_areas_dev over one row: fixed-order block sum, pastila.cu k_areas), so
    results are byte-identical across GPU counts; numpy's sum without a GPU."""
    c = np.ascontiguousarray(curve, dtype=np.float64)
    try:
        import ctypes as C

        import torch

        from . import _native

        if not torch.cuda.is_available():
            raise RuntimeError("no GPU")
        ctx = _native.context()
    except Exception:
        return float(c.sum())
    dev = torch.device("cuda", ctx.device)
    ct = torch.as_tensor(c, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    ctx.call("pst_areas_dev", C.c_void_p(ct.data_ptr()), C.c_int64(1), C.c_int64(c.size), C.c_int64(c.size),
             None, C.c_void_p(out.data_ptr()))
    ctx.call("pst_sync")
    return float(out.item())


def timed(fn, *a, **kw):
    t0 = time.perf_counter()
    out = fn(*a, **kw)
    return out, time.perf_counter() - t0
