"""CLI (python -m paper_2401_13680_b200): exit codes, usage errors and JSON documents.

Host-only paths (argument errors, eval, missing files) run on CPU; discover /
sweep / label run the GPU path and are checked against the CPU oracle.
Reference behaviour: sniplab/cli.py:94-281 and the reference's test_cli.py.
"""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2401_13680_b200 import cli
from paper_2401_13680_b200.datagen import planted_walk

ROOT = Path(__file__).resolve().parents[1]


def _run(args, capsys):
    rc = cli.main(args)
    out = capsys.readouterr()
    return rc, out.out, out.err


def _series_csv(tmp_path, x):
    p = tmp_path / "series.csv"
    np.savetxt(p, x, fmt="%.17g")
    return str(p)


class TestHostOnly:
    def test_usage_errors_exit_2(self, capsys, tmp_path):
        f = _series_csv(tmp_path, np.arange(50.0))
        rc, _, err = _run(["sweep", "--input", f, "--m-min", "16", "--m-max", "8"], capsys)
        assert rc == 2 and "exceeds" in err
        rc, _, err = _run(["sweep", "--input", f, "--m-min", "8", "--m-max", "16", "--l-frac", "0"], capsys)
        assert rc == 2 and "--l-frac" in err
        rc, _, err = _run(["discover", "--input", f, "--m", "8", "--k", "0"], capsys)
        assert rc == 2 and "--k" in err
        rc, _, err = _run(["sweep", "--input", f, "--m-min", "8", "--m-max", "16", "--workers", "0"], capsys)
        assert rc == 2 and "--workers" in err
        rc, _, _ = _run(["discover", "--input", f], capsys)  # --m missing: argparse usage error
        assert rc == 2
        rc, _, _ = _run(["bogus"], capsys)
        assert rc == 2

    def test_missing_file_exit_1(self, capsys, tmp_path):
        rc, _, err = _run(["discover", "--input", str(tmp_path / "nope.csv"), "--m", "8"], capsys)
        assert rc == 1 and err.startswith("error:")

    def test_eval_json(self, capsys, tmp_path):
        (tmp_path / "p.csv").write_text("0\n0\n1\n1\n")
        (tmp_path / "t.csv").write_text("0\n0\n1\n0\n")
        rc, out, _ = _run(["eval", "--pred", str(tmp_path / "p.csv"), "--truth", str(tmp_path / "t.csv")], capsys)
        assert rc == 0
        doc = json.loads(out)
        assert doc["schema"] == 1 and 0.0 < doc["macro_f1"] < 1.0
        rc, _, _ = _run(["eval", "--pred", str(tmp_path / "p.csv"), "--truth", str(tmp_path / "t.csv"),
                         "--output", str(tmp_path / "r.json")], capsys)
        assert rc == 0 and json.loads((tmp_path / "r.json").read_text()) == doc

    def test_module_entry_point(self):
        r = subprocess.run([sys.executable, "-m", "paper_2401_13680_b200", "--help"], capture_output=True, text=True)
        assert r.returncode == 0 and "discover" in r.stdout and "sweep" in r.stdout


@pytest.mark.gpu
class TestGPU:
    def test_discover_matches_oracle(self, capsys, tmp_path):
        from oracle import pastila_oracle as O

        x, _ = planted_walk(4000, m_act=60, A=3, seed=2)
        f = _series_csv(tmp_path, x)
        curve, prof = tmp_path / "curve.csv", tmp_path / "prof.csv"
        rc, out, err = _run(["discover", "--input", f, "--m", "60", "--k", "3", "--export-curve", str(curve),
                             "--export-profiles", str(prof)], capsys)
        assert rc == 0, err
        doc = json.loads(out)
        ref = O.select_snippets(x, 60, 3)
        assert doc["schema"] == 1 and (doc["m"], doc["l"], doc["k"]) == (60, 30, 6)
        assert [s["index"] for s in doc["snippets"]] == ref["indices"]
        assert [s["frac"] for s in doc["snippets"]] == pytest.approx(ref["fracs"], abs=0)
        assert doc["profile_area"] == pytest.approx(ref["profile_area"], rel=1e-9)
        np.testing.assert_allclose(np.loadtxt(curve), ref["curve"], atol=1e-6)
        P = np.loadtxt(prof, delimiter=",", skiprows=1)
        np.testing.assert_allclose(P, ref["profiles"].T, atol=1e-6)

    def test_sweep_and_label_match_oracle(self, capsys, tmp_path):
        from oracle import pastila_oracle as O

        x, _ = planted_walk(3000, m_act=40, A=2, seed=5)
        f = _series_csv(tmp_path, x)
        snip = tmp_path / "best.json"
        rc, out, err = _run(["sweep", "--input", f, "--m-min", "16", "--m-max", "64", "--k", "2", "--no-log",
                             "--output-snippets", str(snip)], capsys)
        assert rc == 0, err
        rep = json.loads(out)
        m_best, cands, results = O.select_length(x, [16, 32, 64], 2)
        assert rep["m_best"] == m_best
        assert json.loads(snip.read_text())["m"] == m_best
        rc, out, err = _run(["label", "--input", f, "--m", "32", "--k", "2"], capsys)
        assert rc == 0, err
        got = np.array([int(v) for v in out.split()])
        r = O.select_snippets(x, 32, 2)
        np.testing.assert_array_equal(got, O.labels(list(r["profiles"]), x.size))


@pytest.mark.gpu
def test_sweep_outputs_identical_across_workers(tmp_path):
    """Reference acceptance #7 (pkg/tests/test_acceptance.py:181-222): the sweep's report
    and snippet JSON are byte-identical for 1, 2 and 4 workers.  Workers are processes
    bound to GPUs (run_schedule, KK partition of the lengths); here all share one GPU."""
    from paper_2401_13680_b200.datagen import two_regime_series

    x, _ = two_regime_series(n=20000, period=32, block_len=1024, noise=0.1, seed=7)
    f = _series_csv(tmp_path, x)

    def run(workers):
        rep, snip = tmp_path / f"r{workers}.json", tmp_path / f"s{workers}.json"
        argv = [sys.executable, "-m", "paper_2401_13680_b200", "sweep", "--input", f, "--m-min", "8",
                "--m-max", "1024", "--k", "2", "--workers", str(workers), "--no-log",
                "--output", str(rep), "--output-snippets", str(snip)]
        proc = subprocess.run(argv, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
        assert proc.returncode == 0, proc.stderr
        return rep.read_bytes() + snip.read_bytes()

    solo = run(1)
    assert run(2) == solo
    assert run(4) == solo


def test_columns_usage_errors(capsys, tmp_path):
    f = _series_csv(tmp_path, np.arange(50.0))
    for bad in ("0,x", "1,1", "-1"):
        rc, out, err = _run(["discover", "--input", f, "--m", "8", "--columns", bad], capsys)
        assert rc == 2, (bad, err)


@pytest.mark.gpu
def test_multi_coordinate_loop_matches_single_columns(capsys, tmp_path):
    """d > 1 (Eq. 2) as the independent per-coordinate loop of SPEC.md:13: --columns runs each
    column exactly as --column would."""
    cols = [planted_walk(3000, m_act=40, A=2, seed=s)[0] for s in (1, 2, 3)]
    f = tmp_path / "multi.csv"
    np.savetxt(f, np.column_stack(cols), fmt="%.17g", delimiter=",")
    f = str(f)
    rc, out, err = _run(["discover", "--input", f, "--m", "32", "--k", "2", "--columns", "all"], capsys)
    assert rc == 0, err
    multi = json.loads(out)
    assert [d["column"] for d in multi["coordinates"]] == [0, 1, 2]
    for c in range(3):
        rc, out, err = _run(["discover", "--input", f, "--m", "32", "--k", "2", "--column", str(c)], capsys)
        one = json.loads(out)
        assert {k: v for k, v in multi["coordinates"][c].items() if k != "column"} == one
    rc, out, err = _run(["label", "--input", f, "--m", "32", "--k", "2", "--columns", "0,2"], capsys)
    assert rc == 0, err
    lab = np.array([[int(v) for v in ln.split(",")] for ln in out.split()])
    for j, c in enumerate((0, 2)):
        rc, o1, _ = _run(["label", "--input", f, "--m", "32", "--k", "2", "--column", str(c)], capsys)
        np.testing.assert_array_equal(lab[:, j], [int(v) for v in o1.split()])
    rc, out, err = _run(["sweep", "--input", f, "--m-min", "16", "--m-max", "64", "--k", "2", "--no-log",
                         "--columns", "1"], capsys)
    assert rc == 0, err
    rc, o1, _ = _run(["sweep", "--input", f, "--m-min", "16", "--m-max", "64", "--k", "2", "--no-log",
                      "--column", "1"], capsys)
    assert {k: v for k, v in json.loads(out)["coordinates"][0].items() if k != "column"} == json.loads(o1)
