"""Shared helpers for the named-size goldens (make_golden_full.py on the reference side,
tests/test_gpu_fullsize.py on the GPU side); importing this does not need /root/reference."""

import numpy as np

SAMPLE_SEED = 20211110


def sample_rows(N, k):
    """Seeded sorted sample of k distinct row indices out of N."""
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.sort(rng.choice(N, size=min(k, N), replace=False))


def functionals(v):
    """Full-vector linear/quadratic functionals: [sum, sum of squares, dot with seeded N(0,1)]."""
    v = np.asarray(v, dtype=np.float64)
    w = np.random.default_rng(SAMPLE_SEED + 1).standard_normal(v.shape[0])
    return np.array([v.sum(), v @ v, v @ w])
