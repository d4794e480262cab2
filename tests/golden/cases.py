"""Golden-vector case table shared by make_golden.py (reference side) and the
tests (GPU box side); importing it does not need /root/reference."""

import numpy as np

# (tag, d, M, m, oversampling, sigma, N, n_targets)
FASTSUM_CASES = [
    ("fs_d1_M32_m4", 1, 32, 4, 2.0, 0.3, 500, 0),
    ("fs_d1_M16_m2_tgt", 1, 16, 2, 2.0, 0.8, 300, 200),
    ("fs_d2_M16_m2_tgt", 2, 16, 2, 2.0, 0.5, 400, 300),
    ("fs_d2_M64_m6", 2, 64, 6, 2.0, 0.05, 300, 0),
    ("fs_d3_M16_m3_os15", 3, 16, 3, 1.5, 0.2, 300, 0),
    ("fs_d3_M32_m4", 3, 32, 4, 2.0, 1.0, 800, 0),
    ("fs_d3_M16_m4_tgt", 3, 16, 4, 2.0, 0.4, 500, 350),
    # 2-D windows at m = 4 take the fp64 tensor-core kernels (csrc/tc2d.cuh): targets,
    # a non-power-of-two grid (n = 48, second compile-time table), many nodes per half-cell
    ("fs_d2_M32_m4_tgt", 2, 32, 4, 2.0, 0.3, 2000, 700),
    ("fs_d2_M32_m4_os15", 2, 32, 4, 1.5, 0.3, 1500, 0),
    ("fs_d2_M16_m4_dense", 2, 16, 4, 2.0, 0.2, 20000, 0),
]


def fastsum_inputs(tag, d, N, n_tgt):
    seed = sum(ord(c) * (i + 1) for i, c in enumerate(tag))
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(N, d)) * rng.uniform(0.5, 2.0, size=d)
    Z = rng.normal(size=(n_tgt, d)) if n_tgt else None
    alpha = rng.standard_normal(N)
    return X, Z, alpha


def krr_inputs(seed=31, n=700, n_test=300, d=7):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n + n_test, d)) * rng.uniform(0.5, 3.0, size=d) + rng.normal(size=d)
    w = rng.normal(size=d)
    y = np.where(np.sin(X) @ w + 0.2 * rng.normal(size=n + n_test) >= 0, 1, -1)
    return X[:n], y[:n], X[n:], y[n:]
