"""Multi-process sharding logic on CPU (gloo, world_size 2): the same combine
code the GPU path runs over NCCL, driven by an oracle backend.  Checks that
segment-row sharding and length sharding reproduce the single-process result
exactly (indices, curve, nearest segment, profile_max)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pastila_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class Job:
    """picklable stand-in for MPdistParams (all_gather_object ships results)"""

    def __init__(self, m):
        self.snippet_size = m


def _oracle_runner(series, jobs, K):
    return [(p, O.select_snippets(series, p.snippet_size, K)["indices"], 0.0) for p in jobs]


class OracleRows:
    def __init__(self, D):
        self.D = D

    def areas(self, curve):
        return (self.D if curve is None else np.minimum(self.D, curve)).sum(axis=1)

    def row(self, i):
        return self.D[i]

    def colmin(self):
        return self.D.min(axis=0), self.D.argmin(axis=0)

    def rowmax(self):
        return float(self.D.max()) if self.D.size else 0.0


def _series():
    from paper_2401_13680_b200.datagen import planted_walk

    x, _ = planted_walk(2400, m_act=40, A=3, seed=3)
    return x


def _worker_rows(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2401_13680_b200 import parallel

    x = _series()
    m, K = 40, 3
    D = O.all_profiles(x, m, O.window_default(m), O.order_default(m))
    ranges = parallel.segment_ranges(D.shape[0], ws)
    lo, hi = ranges[rank]
    ss = parallel.ShardedSearch(OracleRows(D[lo:hi]), ranges, D.shape[1],
                                lambda a: torch.from_numpy(np.ascontiguousarray(a)),
                                lambda t: t.numpy())
    chosen, curve, nearest, pmax = ss.run(K)
    if rank == 0:
        out.put((chosen, curve, nearest, pmax))
    dist.destroy_process_group()


def _worker_lengths(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2401_13680_b200 import parallel

    x = _series()
    grid = [24, 32, 40, 48, 56]

    res = parallel.run_sharded(x, [Job(m) for m in grid], 2, [float(m) for m in grid], runner=_oracle_runner)
    if rank == 0:
        out.put(sorted((p.snippet_size, r) for p, r, _ in res))
    dist.destroy_process_group()


def _worker_sharded_api(rank, ws, port, out):
    """public entry point (parallel.select_snippets_sharded) with an oracle backend"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import paper_2401_13680_b200 as P
    from paper_2401_13680_b200 import parallel

    x = _series()
    m, K = 40, 3
    D = O.all_profiles(x, m, O.window_default(m), O.order_default(m))
    lo, hi = parallel.segment_ranges(D.shape[0], ws)[rank]
    r = parallel.select_snippets_sharded(P.TimeSeries(x), P.MPdistParams(m), K, backend=OracleRows(D[lo:hi]))
    if rank == 0:
        out.put(([s.index for s in r.snippets], [s.frac for s in r.snippets],
                 [s.neighbors.tolist() for s in r.snippets], r.curve, np.vstack([p.values for p in r.profiles]),
                 r.profile_max, r.segment_window_counts, r.unassigned_windows))
    dist.destroy_process_group()


def _spawn(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_segment_row_sharding_matches_single_process():
    chosen, curve, nearest, pmax = _spawn(_worker_rows)
    x = _series()
    D = O.all_profiles(x, 40, O.window_default(40), O.order_default(40))
    ref_chosen, ref_curve = O.greedy_pick(D, 3)
    assert chosen == ref_chosen
    np.testing.assert_array_equal(curve, ref_curve)
    np.testing.assert_array_equal(nearest, np.argmin(D, axis=0))
    assert pmax == float(D.max())


def test_length_sharding_matches_single_process():
    res = _spawn(_worker_lengths)
    x = _series()
    ref = sorted((m, O.select_snippets(x, m, 2)["indices"]) for m in [24, 32, 40, 48, 56])
    assert res == ref


def test_partitions_cover_work():
    from paper_2401_13680_b200 import parallel

    assert parallel.segment_ranges(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    parts = parallel.length_partition([5.0, 4.0, 3.0, 3.0, 1.0], 8)
    assert sorted(i for p in parts for i in p) == [0, 1, 2, 3, 4] and len(parts) == 8


def test_sharded_select_api_matches_oracle():
    idx, fracs, neigh, curve, prof, pmax, counts, unassigned = _spawn(_worker_sharded_api)
    ref = O.select_snippets(_series(), 40, 3)
    assert idx == ref["indices"] and fracs == ref["fracs"]
    assert neigh == [a.tolist() for a in ref["neighbors"]]
    np.testing.assert_array_equal(curve, ref["curve"])
    np.testing.assert_array_equal(prof, ref["profiles"])
    assert pmax == ref["profile_max"] and unassigned == ref["unassigned_windows"]
    np.testing.assert_array_equal(counts, ref["counts"])
