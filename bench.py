"""Benchmark: PaSTiLa length sweep at n=1M (BASELINE.json config 3) on B200.

One "step" = one full snippet-length sweep over the C3 workload: synthetic
planted walk (n=1,000,000, A=4 activities, m_act=256, seed 0),
m in {64, 96, ..., 512} (15 lengths), K=4 snippets, l=ceil(m/2), k=ceil(m/10):
all S=n//m MPdist profiles per length, greedy pick, attribution, Eq. 18
criterion, labels, and the argmax length.  Unit of work = one subsequence
pair (ED_matr entry, Eq. 9): S*w*N_l per length (the reference's
default_cost, scheduler.py:90-102).  Metric: pairs/s (whole job).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pastila|reference]

N>1: launched by torchrun (one process per GPU), strong scaling (the total
work is fixed).  Default --shard rows: every length's segment rows are split
evenly over the ranks (parallel.select_snippets_sharded: per greedy step one
(area, index) all-gather + one profile broadcast over NCCL), so every rank has
1/N of every length.  --shard lengths: Karmarkar-Karp over whole lengths.
Timing: barrier + synchronize, CUDA events on the library stream, max over
ranks.  Inputs (8 MB) are far smaller than L2 and are re-derived inside the
step (prefix sums recomputed), and each length's working set (S*N profile
matrix, 15-125 GB) is far larger than L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

_T_START = time.perf_counter()
# wall-time budget of the whole run (the driver kills the bench at 1800 s): the
# e2e sweep and the CPU sample are skipped, and said so, when they would not fit
BUDGET_S = float(os.environ.get("PASTILA_BENCH_BUDGET_S", "1740"))

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_SERIES = 1_000_000
GRID = list(range(64, 513, 32))
K_SNIPPETS = 4
M_ACT, N_ACT, SEED = 256, 4, 0
FP64_FLOPS_PER_PAIR = 8  # 2 FMA QT update + 1 FMA + 2 MUL correlation
METRIC = "end-to-end PaSTiLa time (s) and subsequence-pairs/sec at n=1M, 1/2/4/8 B200"


def pairs_of(n: int, m: int) -> int:
    l = -(-m // 2)
    return (m - l + 1) * (n - l + 1) * (n // m)


def workload():
    from paper_2401_13680_b200.datagen import planted_walk

    x, _ = planted_walk(N_SERIES, m_act=M_ACT, A=N_ACT, seed=SEED)
    return x


def torch_dist_backend():
    import torch.distributed as dist

    return dist.get_backend() if dist.is_initialized() else None


def dist_init(force: bool = False):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1 and not force:
        return 1, 0, 0
    import torch
    import torch.distributed as dist

    lr = int(os.environ.get("LOCAL_RANK", "0"))
    # test only: PASTILA_FORCE_DEVICE / PASTILA_DIST_BACKEND=gloo run the N>1 code path
    # with several ranks on one GPU (host-side collectives, no cross-rank kernel waits)
    dev = int(os.environ.get("PASTILA_FORCE_DEVICE", lr))
    os.environ["PASTILA_DEVICE"] = str(dev)
    torch.cuda.set_device(dev)
    backend = os.environ.get("PASTILA_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    return ws, dist.get_rank(), dev


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [v.strip() for v in out.stdout.strip().split(",")]
                if len(f) == 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def host_cpu():
    """Host core count and CPU model of this box (lscpu), stated next to every CPU number."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count() or 1
    return {"os_cpu_count": os.cpu_count(), "usable_cores": usable, "model": model}


def fp64_peak():
    for name in ("r02_fp64_peak.json", "r01_fp64_peak.json"):
        p = ROOT / "profiles" / name
        if p.exists():
            return float(json.loads(p.read_text())["fp64_fma_tflops"]), f"measured (profiles/{name}, tools/fpeak.cu)"
    return 37.0, "datasheet"


def cpu_sample_pairs_per_s(x, seconds_budget: float = 20.0):
    """Oracle (numpy restatement of the reference) on 1 host core: MPdist profile
    rows of one segment per sampled length at the true n, bounded windows."""
    from oracle import pastila_oracle as O

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    done_pairs, t_tot, sample = 0, 0.0, []
    for m in (64, 256, 512):
        l, k = O.window_default(m), O.order_default(m)
        w = m - l + 1
        xs = x[: 200_000]   # window subset of the same series (pairs counted exactly)
        st = O.sliding_stats(xs, l)
        t0 = time.perf_counter()
        O.mpdist_profile(xs, 3, m, l, k, st, col_chunk=50_000)
        dt = time.perf_counter() - t0
        done_pairs += w * (xs.size - l + 1)
        t_tot += dt
        sample.append(f"m={m}: 1 segment x {xs.size - m + 1} windows {dt:.1f}s")
        if t_tot > seconds_budget:
            break
    return done_pairs / t_tot, "; ".join(sample)


def run_reference(args):
    """--impl reference: the CPU oracle port on all host cores, bounded sample of C3."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from concurrent.futures import ProcessPoolExecutor

    x = workload()
    host = host_cpu()
    cores = max(1, host["usable_cores"])
    # one job per usable core: (length, segment) pairs cycling through the C3 grid,
    # each the MPdist profile of one segment over a 100k-sample slice of the C3 series
    jobs = [(GRID[i % len(GRID)], 3 + i // len(GRID)) for i in range(cores)]

    def step():
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=cores) as pool:
            tot = sum(pool.map(_ref_job, jobs))
        return tot, time.perf_counter() - t0
    for _ in range(args.warmup):
        step()
    vals, secs = [], []
    for _ in range(args.steps):
        p, dt = step()
        vals.append(p / dt)
        secs.append(dt)
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(secs)),
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(ws),
            "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": cores, "kind": "port", "host": host,
                             "sample": f"{len(jobs)} jobs, one per usable core: (length, segment) pairs cycling "
                                       "through the 15 C3 lengths, each the MPdist profile of one segment over "
                                       "the first 100000 samples of the C3 series"},
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _ref_job(arg):
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import pastila_oracle as O

    m, seg = arg
    x = workload()[:100_000]
    l, k = O.window_default(m), O.order_default(m)
    st = O.sliding_stats(x, l)
    O.mpdist_profile(x, seg % (x.size // m), m, l, k, st, col_chunk=25_000)
    return (m - l + 1) * (x.size - l + 1)


def _config(ws, shard="rows"):
    return {"workload": "C3: planted walk n=1,000,000 (A=4, m_act=256, seed 0), m in 64..512 step 32 "
                        "(15 lengths), K=4, l=ceil(m/2), k=ceil(m/10)",
            "n": N_SERIES, "grid": [GRID[0], GRID[-1], 32], "K": K_SNIPPETS,
            "parallelism": (f"segment-row sharded x{ws}" if shard == "rows" else f"length-sharded x{ws}")
                           if ws > 1 else "1 GPU",
            "l2_flush": "not needed: per-length profile matrix 15-125 GB >> 126 MB L2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pastila", choices=["pastila", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grid", default=None, help="dev only: comma-separated lengths (invalidates the metric)")
    ap.add_argument("--shard", default="rows", choices=["rows", "lengths"],
                    help="N>1 work split: segment rows of every length (default) or whole lengths")
    ap.add_argument("--force-dist", action="store_true",
                    help="test only: create the NCCL group (and use the sharded path) even at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    ws, rank, local = dist_init(args.force_dist)
    sharded = (ws > 1 or args.force_dist) and args.shard == "rows"
    dist_on = ws > 1 or args.force_dist
    red_dev = (f"cuda:{local}" if not dist_on or torch_dist_backend() == "nccl" else "cpu")
    import torch

    import paper_2401_13680_b200 as P
    from paper_2401_13680_b200 import _native, parallel

    grid = [int(v) for v in args.grid.split(",")] if args.grid else GRID
    x = workload()
    ctx = _native.context(local)
    lib = _native.load_library()
    sh = C.c_void_p()
    ctx.call("pst_stream", C.byref(sh))
    stream = torch.cuda.ExternalStream(sh.value, device=torch.device("cuda", local))
    xd = torch.from_numpy(x).to(f"cuda:{local}")
    series = P.TimeSeries(x)
    parts = parallel.length_partition([P.default_cost(N_SERIES, m) for m in grid], ws)
    mine = grid if sharded else [grid[i] for i in parts[rank]]

    def search(s, m):
        """one length: this rank's share (all of it at N=1), plus the Eq. 18 score"""
        if sharded:
            r = parallel.select_snippets_sharded(s, P.MPdistParams(m), K_SNIPPETS)
        else:
            r = P.select_snippets(s, P.MPdistParams(m), K_SNIPPETS)
        return r, P.criterion_score(r)

    def device_step():
        # inputs resident in HBM: device-to-device reload + prefix sums, then all my lengths
        ctx.call("pst_set_series_dev", C.c_void_p(xd.data_ptr()), C.c_int64(x.size))
        ctx._series_key, ctx._series_ref = (id(series.values), series.values.ctypes.data, x.size), series.values
        return {m: search(series, m) for m in mine}

    def barrier():
        if ws > 1 or args.force_dist:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        device_step()
    ctx.call("pst_sync")
    barrier()
    ctx.call("pst_timing", 1)
    cert0 = np.zeros(8, dtype=np.int64)
    ctx.call("pst_cert_stats", _native.ptr(cert0, C.c_int64), 1)  # reset the certification counters
    l0 = ctx.launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(local)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            res = device_step()
        ev1.record(stream)
        ctx.call("pst_sync")
        torch.cuda.synchronize(local)
    ms = ev0.elapsed_time(ev1) / args.steps
    kms, klaunch = C.c_double(0), C.c_int64(0)
    ctx.call("pst_timing_read", C.byref(kms), C.byref(klaunch))
    ctx.call("pst_timing", 0)
    launches = ctx.launches() - l0
    cert = np.zeros(8, dtype=np.int64)
    ctx.call("pst_cert_stats", _native.ptr(cert, C.c_int64), 0)
    barrier()
    if ws > 1 or args.force_dist:
        t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # ---- e2e through the public API (host buffers in, results out) ----------------------
    def e2e_step():
        s = P.TimeSeries(np.array(x))  # fresh host object -> H2D upload inside the step
        if sharded:
            return {m: search(s, m)[1] for m in grid}
        if ws > 1:
            from paper_2401_13680_b200.scheduler import job_weights

            jobs = [P.MPdistParams(m) for m in grid]
            timings = parallel.run_sharded(s, jobs, K_SNIPPETS, job_weights(s, jobs, None))
            return {p.snippet_size: P.criterion_score(r) for p, r, _ in timings}
        rep, results = P.select_length(s, grid, K_SNIPPETS, training_log=False)
        return {c.snippet_size: c.score for c in rep.candidates}
    def elapsed_all():  # wall time since start, max over ranks (a decision every rank takes alike)
        el = time.perf_counter() - _T_START
        if ws > 1 or args.force_dist:
            t = torch.tensor([el], dtype=torch.float64, device=red_dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        return el

    barrier()
    e2e_res, e2e_s = None, None
    if elapsed_all() + 1.2 * ms / 1e3 + 30.0 <= BUDGET_S:
        t0 = time.perf_counter()
        e2e_res = e2e_step()
        e2e_s = time.perf_counter() - t0
        if ws > 1 or args.force_dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(t.item())

    total_pairs = sum(pairs_of(N_SERIES, m) for m in grid)
    if sharded:  # this rank's segment range of every length
        my_pairs = 0
        for m in grid:
            lo, hi = parallel.segment_ranges(N_SERIES // m, parallel.world_size())[parallel.rank()]
            my_pairs += pairs_of(N_SERIES, m) // (N_SERIES // m) * (hi - lo)
    else:
        my_pairs = sum(pairs_of(N_SERIES, m) for m in mine)
    value = total_pairs / (ms / 1e3)
    d2h = sum(K_SNIPPETS * (N_SERIES - m + 1) * 8 + (N_SERIES - m + 1) * 12 + N_SERIES * 8
              + (N_SERIES // m) * 8 for m in grid)
    peak, peak_src = fp64_peak()
    achieved = FP64_FLOPS_PER_PAIR * my_pairs * args.steps / (kms.value / 1e3) / 1e12 if kms.value > 0 else None
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        if time.perf_counter() - _T_START + 30.0 <= BUDGET_S:
            v, sample = cpu_sample_pairs_per_s(x)
            cpu = {"value": v, "unit": "pairs/s", "cores": 1, "kind": "port", "sample": sample, "host": host_cpu()}
        else:
            cpu = {"value": None, "unit": "pairs/s", "skipped": f"wall-time budget {BUDGET_S:.0f} s"}
    issue = None
    ip = next((ROOT / "profiles" / f for f in ("r02_full_m256_summary.json", "r01_full_g256_summary.json")
               if (ROOT / "profiles" / f).exists()), None)
    if ip is not None and achieved:
        # secondary roofline: the path is bound by instruction issue (order
        # comparisons, van Herk minima, selection counts), not by FP64 flops
        wipp = sum(l["warp_instructions_per_pair"] for l in json.loads(ip.read_text())["launches"])
        pps = achieved * 1e12 / FP64_FLOPS_PER_PAIR  # kernel pairs/s
        sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
        peak_issue = 148 * 4 * sm_mhz * 1e6  # warp instructions / s (1 per scheduler per clock)
        issue = {"warp_instr_per_pair": wipp, "achieved": pps * wipp, "peak": peak_issue,
                 "unit": "warp-instr/s", "frac": pps * wipp / peak_issue,
                 "source": f"instructions per pair from profiles/{ip.name} (ncu, m=256 batch: row loop + selection)"}
    if rank == 0:
        traffic = None
        tp = next((ROOT / "profiles" / f for f in ("r02_traffic.json", "r01_traffic.json")
                   if (ROOT / "profiles" / f).exists()), None)
        if tp is not None:
            traffic = json.loads(tp.read_text()).get("bytes_per_launch")
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "seconds_per_sweep": ms / 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(ws, args.shard), "host": host_cpu(),
            "e2e": ({"value": total_pairs / e2e_s, "unit": "pairs/s", "seconds": e2e_s,
                     "h2d_bytes_per_step": int(x.nbytes), "d2h_bytes_per_step": int(d2h)} if e2e_s else
                    {"value": None, "unit": "pairs/s", "skipped": f"wall-time budget {BUDGET_S:.0f} s",
                     "h2d_bytes_per_step": int(x.nbytes), "d2h_bytes_per_step": int(d2h)}),
            "roofline": {"bound": "fp64", "kernel": "profile pass (k_mpdist<int> row loop + k_select_run<int> "
                                                    "selection, key path)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "flops_per_pair": FP64_FLOPS_PER_PAIR, "peak_source": peak_src,
                         "kernel_ms_per_step": kms.value / args.steps,
                         "kernel_share_of_step": (kms.value / args.steps) / ms, "issue": issue},
            "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": int(launches),
            "certification": {"per_step": {k: int(v) // max(1, args.steps) for k, v in zip(
                ["lengths", "greedy_exact_candidates", "greedy_steps_multi", "attribution_uncertain_windows",
                 "exact_window_evals", "max_candidates", "fallbacks_to_exact", "windows"], cert.tolist())},
                "meaning": "key-path decisions resolved with exact fp64 values (pastila.cu run_select_keys)"},
            "m_best": max(e2e_res.items(), key=lambda t: (t[1], -t[0]))[0] if e2e_res else None,
        }
        if args.grid:
            line["config"]["dev_grid_override"] = grid
            line["invalid"] = "grid override: not the metric configuration"
        print(json.dumps(line), flush=True)
    if ws > 1 or args.force_dist:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
