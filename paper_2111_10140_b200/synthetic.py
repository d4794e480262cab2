"""Seeded synthetic workloads C1..C5 (BASELINE.json ``configs``).

The reference measures nothing on public data for this path; these
generators produce inputs with the shapes, sizes and value distributions
BASELINE.json names.  All randomness is numpy PCG64 (``default_rng(seed)``,
reference data.py:16-20) with seed = config number, so both the GPU path
and the CPU oracle see identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from itertools import combinations

import numpy as np


def zscore(X, means=None, stds=None):
    """Population-std z-score with zero std -> 1 (reference data.py:133-150)."""
    X = np.asarray(X, dtype=np.float64)
    if means is None:
        means = X.mean(axis=0)
        stds = X.std(axis=0)
        stds = np.where(stds == 0.0, 1.0, stds)
    return (X - means) / stds, means, stds


@dataclass
class Workload:
    name: str
    X: np.ndarray                 # (N, d) sources
    alpha: np.ndarray             # (N,) or (N, R)
    windows: list                 # tuples of 0-based feature indices
    sigma: float
    M: int                        # coefficient grid (BASELINE's "n")
    m: int                        # window cutoff
    oversampling: float = 2.0
    weights: list | None = None   # eta per window (1/P when None)
    y: np.ndarray | None = None   # labels / targets for CG configs
    Z: np.ndarray | None = None   # held-out targets
    beta: float | None = None
    extra: dict = field(default_factory=dict)

    @property
    def N(self):
        return self.X.shape[0]

    @property
    def R(self):
        return 1 if self.alpha.ndim == 1 else self.alpha.shape[1]

    @property
    def P(self):
        return len(self.windows)


C3_WINDOWS = [(0, 1, 2), (3, 4, 5), (6, 7, 8)] + list(combinations(range(9), 2))
C5_WINDOWS = [(i,) for i in range(20)] + [(2 * k, 2 * k + 1) for k in range(10)]


def c1(N: int = 10_000, seed: int = 1) -> Workload:
    """BASELINE config 0: N=10k, d=9 N(0,1) z-scored, 3 triples, sigma=100, M=32, m=2."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, 9))
    X, _, _ = zscore(X)
    alpha = rng.standard_normal(N)
    return Workload("C1", X, alpha, [(0, 1, 2), (3, 4, 5), (6, 7, 8)], 100.0, 32, 2)


def c2(N: int = 100_000, n_test: int = 20_000, seed: int = 2) -> Workload:
    """BASELINE config 1: CG-KRR, N=100k, 3 triples, sigma=1, beta=1, default profile."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, 9))
    w = rng.standard_normal(9)
    eps = rng.standard_normal(N)
    y = np.where(np.sin(X) @ w + 0.1 * eps >= 0.0, 1.0, -1.0)
    Zraw = rng.standard_normal((n_test, 9))
    Xs, mu, sd = zscore(X)
    Zs, _, _ = zscore(Zraw, mu, sd)
    return Workload("C2", Xs, y.copy(), [(0, 1, 2), (3, 4, 5), (6, 7, 8)], 1.0, 64, 4,
                    y=y, Z=Zs, beta=1.0)


def c3(N: int = 10_000_000, seed: int = 3) -> Workload:
    """BASELINE config 2: N=10M, d=9 U[-1/4,1/4), 3 triples + 36 pairs, sigma=0.5, M=64, m=4."""
    rng = np.random.default_rng(seed)
    X = rng.uniform(-0.25, 0.25, size=(N, 9))
    alpha = rng.standard_normal(N)
    return Workload("C3", X, alpha, list(C3_WINDOWS), 0.5, 64, 4)


def c4(N: int = 100_000_000, R: int = 8, seed: int = 4) -> Workload:
    """BASELINE config 3: 16-cluster Gaussian mixture (std 0.02) clipped to [-1/4,1/4)^3,
    one 3-D window, sigma=0.1, M=128, m=4, R right-hand sides."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-0.2, 0.2, size=(16, 3))
    labels = rng.integers(0, 16, size=N)
    X = centers[labels] + 0.02 * rng.standard_normal((N, 3))
    np.clip(X, -0.25, np.nextafter(0.25, 0.0), out=X)
    alpha = rng.standard_normal((N, R))
    return Workload("C4", X, alpha, [(0, 1, 2)], 0.1, 128, 4)


def c4_shard(N_total: int = 100_000_000, R: int = 8, rank: int = 0, world: int = 1,
             seed: int = 4) -> Workload:
    """This rank's rows of a C4-distributed workload for the point-sharded bench: the 16
    cluster centers come from ``seed`` (shared by all ranks, as in ``c4``); labels, noise and
    alpha of the rank's N_total/world rows from the stream (seed, rank), so no rank draws
    the other ranks' 1e8 x 11 values.  Same distribution as ``c4``, not the same draw."""
    centers = np.random.default_rng(seed).uniform(-0.2, 0.2, size=(16, 3))
    lo = N_total * rank // world
    hi = N_total * (rank + 1) // world
    rng = np.random.default_rng([seed, rank])
    labels = rng.integers(0, 16, size=hi - lo)
    X = centers[labels] + 0.02 * rng.standard_normal((hi - lo, 3))
    np.clip(X, -0.25, np.nextafter(0.25, 0.0), out=X)
    alpha = rng.standard_normal((hi - lo, R))
    return Workload("C4", X, alpha, [(0, 1, 2)], 0.1, 128, 4, extra={"N_total": N_total})


def c5(N: int = 1_000_000, seed: int = 5) -> Workload:
    """BASELINE config 4: d=20 in 5 equicorrelated blocks (rho=0.7), z-scored, 20 singles +
    10 pairs (2k,2k+1), y = sum_k f_k(x_Wk) + 0.1 eps (random-Fourier f_k), sigma=1, beta=0.1."""
    rng = np.random.default_rng(seed)
    rho = 0.7
    zb = rng.standard_normal((N, 5))
    zi = rng.standard_normal((N, 20))
    X = np.sqrt(rho) * zb[:, np.arange(20) // 4] + np.sqrt(1.0 - rho) * zi
    X, _, _ = zscore(X)
    y = np.zeros(N)
    for w in C5_WINDOWS:
        u = X[:, list(w)]
        a = rng.standard_normal(8) / 8.0
        om = rng.standard_normal((8, len(w)))
        ph = rng.uniform(0.0, 2.0 * np.pi, 8)
        y += np.cos(u @ om.T + ph) @ a
    y += 0.1 * rng.standard_normal(N)
    return Workload("C5", X, y.copy(), list(C5_WINDOWS), 1.0, 64, 4, y=y, beta=0.1)


GENERATORS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}
