"""Synthetic data for the benchmark configs (BASELINE.json).

`friedman1` is the DGP the BASELINE configs name; it is not in the reference
(SURVEY.md §8d defines it): X ~ U(0,1)^{n x p},
f = 10 sin(pi x1 x2) + 20 (x3 - 1/2)^2 + 10 x4 + 5 x5, y = f + N(0, 1).
`friedman1_binned` produces the uint8 binned matrix directly in bounded
memory (row blocks), equal to quantize(build_grid_uniform(X, k)) on the
same draws.  `gen_timing`/`gen_easy` follow the reference (dgp.py:45-72).
"""

from __future__ import annotations

import numpy as np

from .grid import CutpointGrid, build_grid_uniform, quantize


def friedman1(n: int, p: int, seed: int = 0, noise_sd: float = 1.0):
    if p < 5:
        raise ValueError("Friedman #1 needs p >= 5")
    rng = np.random.default_rng(seed)
    X = rng.uniform(0.0, 1.0, size=(n, p))
    f = 10 * np.sin(np.pi * X[:, 0] * X[:, 1]) + 20 * (X[:, 2] - 0.5) ** 2 + 10 * X[:, 3] + 5 * X[:, 4]
    return X, f + rng.normal(0.0, noise_sd, size=n), f


def friedman1_binned(n: int, p: int, seed: int = 0, n_cutpoints: int = 100, block: int = 1 << 18):
    """(Xq uint8 (n,p), y f64, f f64, grid) without holding the f64 X for large n.

    X is drawn block-by-block from one Generator; each block is binned on a
    uniform grid over [0, 1]-ish observed range computed in a first pass of
    the same stream (two passes over identical draws).
    """
    lo = np.full(p, np.inf)
    hi = np.full(p, -np.inf)
    rng = np.random.default_rng(seed)
    for s in range(0, n, block):
        Xb = rng.uniform(0.0, 1.0, size=(min(block, n - s), p))
        lo = np.minimum(lo, Xb.min(axis=0))
        hi = np.maximum(hi, Xb.max(axis=0))
    frac = np.arange(1, n_cutpoints + 1) / (n_cutpoints + 1)
    grid = CutpointGrid([np.empty(0) if a == b else a + (b - a) * frac for a, b in zip(lo, hi)])
    rng = np.random.default_rng(seed)
    Xq = np.empty((n, p), np.uint8)
    f = np.empty(n)
    for s in range(0, n, block):
        Xb = rng.uniform(0.0, 1.0, size=(min(block, n - s), p))
        Xq[s:s + Xb.shape[0]] = quantize(Xb, grid).data
        f[s:s + Xb.shape[0]] = (10 * np.sin(np.pi * Xb[:, 0] * Xb[:, 1]) + 20 * (Xb[:, 2] - 0.5) ** 2
                                + 10 * Xb[:, 3] + 5 * Xb[:, 4])
    y = f + np.random.default_rng(seed + 1).normal(0.0, 1.0, size=n)
    return Xq, y, f, grid


def gen_timing(n: int, p: int):
    """Deterministic timing inputs (dgp.py:45-58)."""
    if n < 2:
        raise ValueError("need n >= 2")
    i = np.arange(1, n + 1)
    j = np.arange(1, p + 1)
    y = np.cos(2.0 * n * np.pi / 32.0 * (i - 1) / (n - 1))
    X = np.mod(i[:, None] + (p + 1) * j[None, :], 256).astype(np.float64)
    return X, y


def gen_easy(n: int, p: int, seed: int = 0, noise_sd: float = 0.1):
    """Smooth additive signal (dgp.py:61-72)."""
    rng = np.random.default_rng(seed)
    X = rng.uniform(-2.0, 2.0, size=(n, p))
    f = np.cos(np.pi * X).sum(axis=1) / np.sqrt(p)
    return X, f + rng.normal(0.0, noise_sd, size=n), f


__all__ = ["friedman1", "friedman1_binned", "gen_timing", "gen_easy", "build_grid_uniform"]
