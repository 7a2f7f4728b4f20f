"""Seeded synthetic series for tests and the benchmark (no datasets: no network).

``planted_walk`` is the builder-defined generator of BASELINE.md §5: a slow
random walk with A planted periodic activities; for A=3 it reproduces the
SHA-256 values listed there bit-for-bit (checked in tests/test_host.py).
``two_regime_series`` follows the published behaviour of the reference test
helper (pkg/tests/seriesgen.py:6-29): quantized sine / square regimes whose
noise-free repeats are bit-identical, so exact-tie rules can be tested.
"""

from __future__ import annotations

import numpy as np


def planted_walk(n: int, m_act: int = 120, A: int = 3, seed: int = 0):
    """Random walk (0.1*cumsum N(0,1)) with A activity templates of period ``m_act``.

    Blocks of ``10*m_act`` samples cycle through the activities; inside a block
    value = 0.05*walk + template, plus 0.05*N(0,1) noise drawn after the walk
    from the same generator.  Returns (values f64[n], truth int64[n]).
    """
    rng = np.random.default_rng(seed)
    walk = 0.1 * np.cumsum(rng.standard_normal(n))
    t = np.arange(m_act)
    templates = [
        np.sin(2 * np.pi * t / m_act),
        np.where(t < m_act // 2, 1.0, -1.0),
        2 * t / m_act - 1,
        1 - 2 * np.abs(2 * t / m_act - 1),                                   # triangle
        0.5 * np.sin(2 * np.pi * t / m_act) + 0.5 * np.sin(6 * np.pi * t / m_act),  # two-tone
    ]
    if not 1 <= A <= len(templates):
        raise ValueError(f"A must be in [1, {len(templates)}], got {A}")
    truth = (np.arange(n) // (10 * m_act)) % A
    vals = np.zeros(n)
    reps = n // m_act + 1
    for a in range(A):
        vals = np.where(truth == a, 0.05 * walk + np.tile(templates[a], reps)[:n], vals)
    values = vals + 0.05 * rng.standard_normal(n)
    return values, truth.astype(np.int64)


def two_regime_series(n: int, period: int = 32, block_len: int = 32, noise: float = 0.1, seed: int = 0):
    """Alternating quantized-sine / square regimes (exact float sums when noise=0)."""
    rng = np.random.default_rng(seed)
    t = np.arange(period)
    sine = np.round(np.sin(2 * np.pi * t / period) * 64) / 64
    square = np.where(t < period // 2, 1.0, -1.0)
    reps = n // period + 1
    regime = (np.arange(n) // block_len) % 2
    values = np.where(regime == 0, np.tile(sine, reps)[:n], np.tile(square, reps)[:n])
    if noise:
        values = values + noise * rng.standard_normal(n)
    return values, regime
