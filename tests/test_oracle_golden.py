"""Pin the CPU oracle (oracle/pastila_oracle.py) to the reference's golden vectors.

The fixtures were produced by the real reference (tests/golden/make_golden.py);
the oracle restates the same numpy operation order, so agreement is bit-exact
on this machine.  CPU-only: no GPU needed."""

import hashlib

import numpy as np
import pytest

from oracle import pastila_oracle as O
from paper_2401_13680_b200.datagen import planted_walk


def test_stats_bit_exact(golden):
    g, meta = golden
    for c, cs in enumerate(meta["stats"]):
        mu, sd, var = O.sliding_stats(g[f"stats{c}_x"], cs["l"])
        np.testing.assert_array_equal(mu, g[f"stats{c}_mean"])
        np.testing.assert_array_equal(sd, g[f"stats{c}_std"])
        np.testing.assert_array_equal(var, g[f"stats{c}_var"])


def test_distance_block(golden):
    g, meta = golden
    for c, cs in enumerate(meta["dm"]):
        x = g[f"dm{c}_x"]
        mu, _, var = O.sliding_stats(x, cs["l"])
        mat = O.distance_block(x, mu, var, cs["seg"] * cs["m"], cs["m"] - cs["l"] + 1, cs["l"])
        np.testing.assert_allclose(mat, g[f"dm{c}_mat"], atol=1e-12)


def test_profiles(golden):
    g, meta = golden
    for c, cs in enumerate(meta["prof"]):
        x = g[f"prof{c}_x"]
        D = np.vstack([O.mpdist_profile(x, s, cs["m"], cs["l"], cs["k"]) for s in cs["segs"]])
        np.testing.assert_allclose(D, g[f"prof{c}_D"], atol=1e-12)
        # chunked evaluation gives identical values
        D2 = np.vstack([O.mpdist_profile(x, s, cs["m"], cs["l"], cs["k"], col_chunk=17) for s in cs["segs"]])
        np.testing.assert_array_equal(D, D2)


def test_snippets(golden):
    g, meta = golden
    for c, doc in enumerate(meta["snip"]):
        r = O.select_snippets(g[f"snip{c}_x"], doc["m"], doc["K"])
        assert r["indices"] == doc["indices"]
        assert r["fracs"] == doc["fracs"]
        assert [int(v.size) for v in r["neighbors"]] == doc["neighbor_counts"]
        assert r["profile_area"] == doc["profile_area"]
        assert r["profile_max"] == doc["profile_max"]
        assert r["unassigned_windows"] == doc["unassigned_windows"]
        np.testing.assert_array_equal(r["counts"], g[f"snip{c}_counts"])
        np.testing.assert_array_equal(O.labels(list(r["profiles"]), len(g[f"snip{c}_x"])), g[f"snip{c}_labels"])
        if "criterion" in doc:
            assert O.criterion(r["profiles"], r["profile_max"]) == doc["criterion"]


def test_sweeps(golden):
    g, meta = golden
    for c, doc in enumerate(meta["sweep"]):
        best, cands, _ = O.select_length(g[f"sweep{c}_x"], doc["grid"], doc["K"])
        assert best == doc["m_best"]
        for a, b in zip(cands, doc["candidates"]):
            assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]


def test_planted_walk_matches_baseline_sha():
    """BASELINE.md §5 lists the SHA-256 of the generator's bytes for A=3, seed 0."""
    for n, sha, first in [
        (20000, "8a988f9c9ee47b5bd21680e262743a7fbaac5881ccbfebab2260d44d2e147e9c", 0.01680838699850235),
        (100000, "faf0a92e8516e1bd08753ffeb38e3ac0e6c41ee37d4c0da3611945b8027050fe", 0.059380029287820234),
    ]:
        x, _ = planted_walk(n, m_act=120, A=3, seed=0)
        assert hashlib.sha256(x.astype("<f8").tobytes()).hexdigest() == sha
        assert x[0] == first


@pytest.mark.slow
def test_c1_oracle(golden):
    g, meta = golden
    x, _ = planted_walk(20000, m_act=120, A=3, seed=0)
    r = O.select_snippets(x, 120, 3)
    assert r["indices"] == meta["c1"]["indices"]
    assert r["profile_area"] == meta["c1"]["profile_area"]
