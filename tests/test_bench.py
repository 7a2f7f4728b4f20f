"""bench.py host-side contract (no GPU): work accounting, CLI, and the reference
arm's JSON line (the CPU oracle port on a bounded sample of the C3 workload)."""

import json
import subprocess
import sys
from pathlib import Path

import paper_2401_13680_b200 as P

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_pairs_match_reference_cost():
    for m in bench.GRID:
        assert bench.pairs_of(bench.N_SERIES, m) == P.default_cost(bench.N_SERIES, m)
    assert len(bench.GRID) == 15 and bench.GRID[0] == 64 and bench.GRID[-1] == 512
    tot = sum(bench.pairs_of(bench.N_SERIES, m) for m in bench.GRID)
    assert abs(tot - 7.573e12) / 7.573e12 < 1e-3


def test_help():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "--shard" in r.stdout and "--impl" in r.stdout


def test_reference_arm_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "pairs/s" and line["value"] > 0
    assert line["metric"] == bench.METRIC and line["higher_is_better"] is True and line["ms_per_step"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
