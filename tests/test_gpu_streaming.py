"""Selection without a resident S x N profile matrix (config C4, n = 1e7: 3.1 TB):
the streamed greedy (profiles recomputed per round, pst_profile_reduce_dev) and the
segment-row sharded API must give exactly the resident result.  Chunking is forced
small with PASTILA_STREAM_ROWS so the streamed path runs at test sizes."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2401_13680_b200 as P  # noqa: E402
from paper_2401_13680_b200 import parallel  # noqa: E402
from paper_2401_13680_b200.datagen import planted_walk  # noqa: E402
from oracle import pastila_oracle as O  # noqa: E402


def _same(a, b):
    assert [s.index for s in a.snippets] == [s.index for s in b.snippets]
    assert [s.frac for s in a.snippets] == [s.frac for s in b.snippets]
    for sa, sb in zip(a.snippets, b.snippets):
        np.testing.assert_array_equal(sa.neighbors, sb.neighbors)
    np.testing.assert_array_equal(a.curve, b.curve)
    for pa, pb in zip(a.profiles, b.profiles):
        np.testing.assert_array_equal(pa.values, pb.values)
    assert a.profile_max == b.profile_max
    np.testing.assert_array_equal(a.segment_window_counts, b.segment_window_counts)
    assert a.unassigned_windows == b.unassigned_windows


@pytest.fixture
def series():
    x, _ = planted_walk(20000, m_act=120, A=3, seed=0)
    return x


@pytest.mark.parametrize("chunk", ["1", "7", "64"])
def test_streamed_select_equals_resident(series, monkeypatch, chunk):
    s, p = P.TimeSeries(series), P.MPdistParams(120)
    resident = P.select_snippets(s, p, 3)
    monkeypatch.setenv("PASTILA_STREAM_ROWS", chunk)
    streamed = P.select_snippets(P.TimeSeries(series.copy()), p, 3)
    _same(resident, streamed)
    assert streamed.profile_area == resident.profile_area
    assert streamed.criterion_ == resident.criterion_
    np.testing.assert_array_equal(streamed.labels_, resident.labels_)
    ref = O.select_snippets(series, 120, 3)
    assert [s.index for s in streamed.snippets] == ref["indices"]


def _pg_single():
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    return dist


@pytest.mark.parametrize("backend", ["DeviceRows", "StreamedRows"])
def test_sharded_api_device_backends(series, monkeypatch, backend):
    s, p = P.TimeSeries(series), P.MPdistParams(120)
    resident = P.select_snippets(s, p, 3)
    monkeypatch.setenv("PASTILA_STREAM_ROWS", "5")
    dist = _pg_single()
    try:
        S = series.size // 120
        b = getattr(parallel, backend)(s, p, 0, S)
        got = parallel.select_snippets_sharded(s, p, 3, backend=b)
    finally:
        dist.destroy_process_group()
    _same(resident, got)
    assert got.profile_area == resident.profile_area  # same device reduction: byte-identical


def test_threads_share_a_context():
    """Two threads, two series, one device context: results equal the sequential ones
    (every upload-then-compute sequence holds the context lock)."""
    import threading

    xa, _ = planted_walk(12000, m_act=60, A=3, seed=21)
    xb, _ = planted_walk(12000, m_act=80, A=2, seed=22)
    p = P.MPdistParams(60)
    ref = {k: [s.index for s in P.select_snippets(P.TimeSeries(x), p, 3).snippets] for k, x in (("a", xa), ("b", xb))}
    got, errs = {"a": [], "b": []}, []

    def work(key, x):
        try:
            for _ in range(4):
                got[key].append([s.index for s in P.select_snippets(P.TimeSeries(x), p, 3).snippets])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=("a", xa)), threading.Thread(target=work, args=("b", xb))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    assert all(g == ref["a"] for g in got["a"]) and all(g == ref["b"] for g in got["b"])


def _two_rank_worker(rank, port, backend_name, out):
    """one of two gloo ranks sharing cuda:0 (host-side collectives only)"""
    import torch.distributed as dist

    os.environ["PASTILA_DEVICE"] = "0"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    import paper_2401_13680_b200 as PP
    from paper_2401_13680_b200 import parallel as par
    from paper_2401_13680_b200.datagen import planted_walk as pw

    x, _ = pw(20000, m_act=120, A=3, seed=0)
    s, p = PP.TimeSeries(x), PP.MPdistParams(120)
    lo, hi = par.segment_ranges(x.size // 120, 2)[rank]
    if backend_name == "StreamedRows":
        os.environ["PASTILA_STREAM_ROWS"] = "9"
    b = getattr(par, backend_name)(s, p, lo, hi)
    r = par.select_snippets_sharded(s, p, 3, backend=b)
    if rank == 0:
        out.put(([q.index for q in r.snippets], [q.frac for q in r.snippets], r.curve,
                 np.vstack([q.values for q in r.profiles]), r.profile_max, r.segment_window_counts))
    dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["DeviceRows", "StreamedRows"])
def test_two_ranks_row_sharded_on_device(series, backend):
    """segment-row sharding with device backends across two processes (gloo, one GPU)
    == the single-process resident result"""
    import torch.multiprocessing as mp

    ref = P.select_snippets(P.TimeSeries(series), P.MPdistParams(120), 3)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, port, backend, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    idx, fr, curve, prof, pmax, counts = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert idx == [s_.index for s_ in ref.snippets] and fr == [s_.frac for s_ in ref.snippets]
    np.testing.assert_array_equal(curve, ref.curve)
    np.testing.assert_array_equal(prof, np.vstack([p_.values for p_ in ref.profiles]))
    assert pmax == ref.profile_max
    np.testing.assert_array_equal(counts, ref.segment_window_counts)


@pytest.mark.parametrize("backend", ["DeviceRows", "StreamedRows"])
def test_library_nccl_sharded_search_equals_resident(series, monkeypatch, backend):
    """The library-owned NCCL data plane (csrc/comm.cu: pst_comm_* collectives and the
    device glue kernels, DeviceShardedSearch) in a single-rank communicator: every
    collective, the on-device pick and the tie-index attribution run, and the result
    is byte-identical to the resident single-GPU search."""
    s, p = P.TimeSeries(series), P.MPdistParams(120)
    resident = P.select_snippets(s, p, 3)
    monkeypatch.setenv("PASTILA_STREAM_ROWS", "5")
    S = series.size // 120
    b = getattr(parallel, backend)(s, p, 0, S)
    got = parallel.select_snippets_sharded(s, p, 3, backend=b, comm="lib")
    _same(resident, got)
    assert got.profile_area == resident.profile_area
