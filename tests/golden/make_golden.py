"""Generate golden fixtures by running the REAL reference (sniplab) on seeded inputs.

Run in the dev container only (``/root/reference`` does not exist on the GPU box):

    python tests/golden/make_golden.py            # small + C1 fixtures (~1 min)
    python tests/golden/make_golden.py --c2       # adds the C2 sweep (~15 min, 8 workers)

The reference package and its test helpers are imported read-only from
``/root/reference/pkg/{src,tests}``; nothing is copied.  Every fixture stores
its own input series, so the fixtures are self-contained: the GPU parity tests
and the oracle tests read only ``tests/golden/*.npz`` / ``*.json``.

Reference call sites pinned here:
  compute_sliding_stats   series.py:152-190
  segment_distance_matrix zdist.py:191-225
  mpdist_profile          mpdist.py:179-232
  select_snippets         snippets.py:154-244
  criterion_score         length_select.py:56-87
  select_length           length_select.py:116-182
  label_series            labeling.py:91-119
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(HERE.parents[1]))

import sniplab  # noqa: E402  (reference, read-only)
from seriesgen import random_series, two_regime_series  # noqa: E402  (reference test helper)
from oracles import naive_distance_row, naive_mpdist_profile  # noqa: E402  (reference test oracle)

from paper_2401_13680_b200.datagen import planted_walk  # noqa: E402


def _result_doc(res) -> dict:
    """Flatten a reference SnippetResult into arrays + scalars."""
    return {
        "m": res.snippet_size,
        "l": res.window_size,
        "k": res.k,
        "n": res.series_length,
        "indices": [int(s.index) for s in res.snippets],
        "starts": [int(s.start) for s in res.snippets],
        "fracs": [float(s.frac) for s in res.snippets],
        "neighbor_counts": [int(s.neighbors.size) for s in res.snippets],
        "profile_area": float(res.profile_area),
        "profile_max": float(res.profile_max),
        "unassigned_windows": int(res.unassigned_windows),
    }


def _result_arrays(prefix: str, res, series_len: int) -> dict:
    labels = sniplab.label_series(res).labels
    nearest = np.full(res.curve.size, -1, dtype=np.int64)
    for s in res.snippets:
        nearest[s.neighbors] = s.index
    return {
        f"{prefix}_curve": res.curve,
        f"{prefix}_profiles": np.vstack([p.values for p in res.profiles]),
        f"{prefix}_counts": np.asarray(res.segment_window_counts, dtype=np.int64),
        f"{prefix}_labels": np.asarray(labels, dtype=np.int64),
        f"{prefix}_snip_nearest": nearest,
    }


def small_cases(out: dict, meta: dict) -> None:
    # --- sliding stats (series.py:152-190), incl. flat spells and huge offsets
    rng = np.random.default_rng(11)
    stats_cases = []
    for c in range(8):
        n = int(rng.integers(10, 600))
        l = int(rng.integers(1, n + 1))
        x = random_series(rng, n) * rng.uniform(0.1, 100)
        st = sniplab.compute_sliding_stats(sniplab.TimeSeries(x), l)
        out[f"stats{c}_x"] = x
        out[f"stats{c}_mean"] = st.means
        out[f"stats{c}_std"] = st.stds
        out[f"stats{c}_var"] = st.variances
        stats_cases.append({"l": l})
    x = np.full(64, 1e9)
    x[::7] += 1e-3
    st = sniplab.compute_sliding_stats(sniplab.TimeSeries(x), 8)
    out["stats8_x"], out["stats8_mean"], out["stats8_std"], out["stats8_var"] = x, st.means, st.stds, st.variances
    stats_cases.append({"l": 8})
    meta["stats"] = stats_cases

    # --- segment distance matrices (zdist.py:191-225)
    rng = np.random.default_rng(22)
    dm_cases = []
    for c in range(5):
        n = int(rng.integers(80, 400))
        m = int(rng.choice([8, 12, 16, 24]))
        l = int(rng.integers(2, m + 1))
        x = random_series(rng, n)
        st = sniplab.compute_sliding_stats(sniplab.TimeSeries(x), l)
        seg = int(rng.integers(0, n // m))
        mat = sniplab.segment_distance_matrix(sniplab.TimeSeries(x), st, seg * m, m)
        out[f"dm{c}_x"], out[f"dm{c}_mat"] = x, mat
        out[f"dm{c}_naive"] = np.vstack([naive_distance_row(x, seg * m + i, l) for i in range(m - l + 1)])
        dm_cases.append({"m": m, "l": l, "seg": seg})
    meta["dm"] = dm_cases

    # --- MPdist profiles (mpdist.py:179-232), default and explicit params
    rng = np.random.default_rng(33)
    prof_cases = []
    for c in range(12):
        n = int(rng.integers(60, 400))
        m = int(rng.choice([4, 8, 16, 20]))
        x = random_series(rng, n)
        if c == 10:
            l, k = 5, 100  # 2w <= k: max fallback (mpdist.py:228-231)
            m = 10
        elif c == 11:
            l, k = 2, 3
        else:
            l, k = None, None
        p = sniplab.MPdistParams(snippet_size=m, window_size=l, k=k)
        segs = sorted({0, (n // m) - 1, int(rng.integers(0, n // m))})
        D = np.vstack([sniplab.mpdist_profile(sniplab.TimeSeries(x), s, p).values for s in segs])
        out[f"prof{c}_x"], out[f"prof{c}_D"] = x, D
        out[f"prof{c}_naive"] = np.vstack([naive_mpdist_profile(x, s, m, p.window_size, p.k) for s in segs])
        prof_cases.append({"m": m, "l": p.window_size, "k": p.k, "segs": segs})
    meta["prof"] = prof_cases

    # --- select_snippets + label_series (snippets.py:154-244, labeling.py:91-119)
    snip_cases = []
    rng = np.random.default_rng(44)
    specs = []
    for c in range(6):
        n = int(rng.integers(100, 500))
        m = int(rng.choice([8, 10, 12, 16]))
        K = int(rng.integers(1, min(5, n // m) + 1))
        specs.append(("random", random_series(rng, n), m, K))
    v, _ = two_regime_series(n=384, period=32, block_len=96, noise=0.0)
    specs.append(("two_regime_exact", v, 32, 2))
    v, _ = two_regime_series(n=512, period=16, block_len=128, noise=0.0, seed=2)
    specs.append(("two_regime_labels_exact", v, 16, 2))
    v, _ = two_regime_series(n=512, period=16, block_len=128, noise=0.05, seed=2)
    specs.append(("two_regime_labels_noisy", v, 16, 2))
    specs.append(("constant", np.full(256, 3.5), 16, 2))
    specs.append(("tiled", np.tile([0.0, 2.0, 1.0, 3.0, 2.0, 0.0, 1.0, 2.0], 8), 8, 1))
    for c, (name, x, m, K) in enumerate(specs):
        res = sniplab.select_snippets(sniplab.TimeSeries(x), sniplab.MPdistParams(snippet_size=m), K)
        out[f"snip{c}_x"] = np.asarray(x, dtype=np.float64)
        out.update(_result_arrays(f"snip{c}", res, len(x)))
        doc = _result_doc(res)
        doc["name"], doc["K"] = name, K
        if K >= 2:
            doc["criterion"] = float(sniplab.criterion_score(res))
        snip_cases.append(doc)
    meta["snip"] = snip_cases

    # --- select_length (length_select.py:116-182)
    sweep_cases = []
    for c, (n, period, block, noise, seed, grid) in enumerate(
        [(2048, 32, 32, 0.05, 3, [16, 32, 64]), (512, 16, 64, 0.05, 6, [8, 16, 32]), (1024, 16, 64, 0.1, 1, [8, 12, 16, 24, 32])]
    ):
        v, _ = two_regime_series(n=n, period=period, block_len=block, noise=noise, seed=seed)
        rep, results = sniplab.select_length(sniplab.TimeSeries(v), grid, 2, training_log=False)
        out[f"sweep{c}_x"] = v
        sweep_cases.append({
            "grid": grid, "K": 2, "m_best": rep.m_best,
            "candidates": [[c2.snippet_size, c2.score, c2.profile_area] for c2 in rep.candidates],
            "winner": _result_doc(results[rep.m_best]),
        })
    meta["sweep"] = sweep_cases


def c1_case(out: dict, meta: dict) -> None:
    """BASELINE config 1: planted walk n=20000 (A=3, m_act=120, seed 0), m=120, K=3."""
    x, truth = planted_walk(20000, m_act=120, A=3, seed=0)
    t0 = time.perf_counter()
    res = sniplab.select_snippets(sniplab.TimeSeries(x), sniplab.MPdistParams(snippet_size=120), 3)
    el = time.perf_counter() - t0
    out.update(_result_arrays("c1", res, x.size))
    doc = _result_doc(res)
    doc["criterion"] = float(sniplab.criterion_score(res))
    doc["seconds_reference_1core"] = el
    meta["c1"] = doc


def c2_case(meta: dict) -> None:
    """BASELINE config 2: planted walk n=100000, m in 64..512 step 32, K=3 (select_length)."""
    x, _ = planted_walk(100000, m_act=120, A=3, seed=0)
    workers = int(os.environ.get("GOLDEN_WORKERS", "8"))
    t0 = time.perf_counter()
    rep, results = sniplab.select_length(sniplab.TimeSeries(x), list(range(64, 513, 32)), 3,
                                         workers=workers, training_log=False)
    el = time.perf_counter() - t0
    meta["c2"] = {
        "grid": list(range(64, 513, 32)), "K": 3, "m_best": rep.m_best,
        "candidates": [[c.snippet_size, c.score, c.profile_area] for c in rep.candidates],
        "results": {str(m): _result_doc(r) for m, r in results.items()},
        "seconds_reference": el, "workers": workers,
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true")
    args = ap.parse_args()
    if args.c2:
        meta = {}
        c2_case(meta)
        (HERE / "golden_c2.json").write_text(json.dumps(meta["c2"], indent=1))
        return
    out: dict = {}
    meta: dict = {"generator": "tests/golden/make_golden.py", "reference": "sniplab 0.1.0 (/root/reference/pkg)",
                  "numpy": np.__version__}
    small_cases(out, meta)
    c1_case(out, meta)
    np.savez_compressed(HERE / "golden.npz", **out)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
