"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from
``/root/reference/pkg/src/nfftkrr`` and writes ``tests/golden/golden.npz``.
Inputs are regenerated from seeds by the tests (numpy PCG64 is
version-stable); only small inputs are stored alongside the outputs.
Nothing on the GPU box reads /root/reference: the committed .npz is the
parity anchor there.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import nfftkrr  # noqa: E402  (the reference)
from nfftkrr import (AccuracyProfile, AnovaKernelOperator, FastsumOperator,  # noqa: E402
                     GaussianKernel, GridSpec, NfftPlan, PeriodizationConfig, cg_solve,
                     regularize_kernel)

from paper_2111_10140_b200 import synthetic  # noqa: E402

from cases import FASTSUM_CASES, fastsum_inputs  # noqa: E402


def composed(X, windows, sigma, M, m, alpha, Z=None, weights=None):
    """Sum eta_l FastsumOperator_l(alpha) in window order (SURVEY §8(c) recipe for C3/C4/C5)."""
    P = len(windows)
    weights = weights if weights is not None else [1.0 / P] * P
    prof = AccuracyProfile("bench", 2.0, m)
    cfg = PeriodizationConfig(coeff_grid=M)
    out = np.zeros(X.shape[0] if Z is None else Z.shape[0])
    for eta, w in zip(weights, windows):
        op = FastsumOperator(GaussianKernel(sigma), cfg, X[:, list(w)],
                             None if Z is None else Z[:, list(w)], prof)
        out += eta * op.apply(alpha)
    return out


def main():
    g = {}
    meta = {"numpy": np.__version__, "reference": getattr(nfftkrr, "__version__", "?")}
    import scipy
    meta["scipy"] = scipy.__version__

    # --- NFFT known-answer vectors (forward / adjoint), all dims and profiles
    for d in (1, 2, 3):
        for prof in ("rough", "default", "fine"):
            rng = np.random.default_rng(100 + 10 * d + len(prof))
            M = 16 if d < 3 else 8
            grid = GridSpec((M,) * d)
            x = rng.uniform(-0.5, 0.5, size=(40, d))
            fh = rng.normal(size=grid.n_modes) + 1j * rng.normal(size=grid.n_modes)
            c = rng.normal(size=40) + 1j * rng.normal(size=40)
            plan = NfftPlan(grid, x, prof)
            key = f"nfft_d{d}_{prof}"
            g[key + "_x"] = x
            g[key + "_fhat"] = fh
            g[key + "_c"] = c
            g[key + "_fwd"] = plan.forward(fh)
            g[key + "_adj"] = plan.adjoint(c)

    # --- kernel Fourier coefficients (fastsum.py:138-159)
    for sigma, M, d in ((0.1, 16, 1), (0.05, 32, 2), (0.3, 16, 3), (2.0, 8, 3)):
        key = f"coef_s{sigma}_M{M}_d{d}"
        g[key] = regularize_kernel(GaussianKernel(sigma), PeriodizationConfig(coeff_grid=M), d)

    # --- single-window fast summation
    for tag, d, M, m, os_, sigma, N, n_tgt in FASTSUM_CASES:
        X, Z, alpha = fastsum_inputs(tag, d, N, n_tgt)
        op = FastsumOperator(GaussianKernel(sigma), PeriodizationConfig(coeff_grid=M), X, Z,
                             AccuracyProfile("golden", os_, m))
        g[tag + "_X"] = X
        if Z is not None:
            g[tag + "_Z"] = Z
        g[tag + "_alpha"] = alpha
        g[tag + "_out"] = op.apply(alpha)
        g[tag + "_scale"] = np.array(op.scale)
        g[tag + "_center"] = op.center
        meta[tag] = dict(d=d, M=M, m=m, oversampling=os_, sigma=sigma, N=N, n_tgt=n_tgt)

    # --- C1 at full size through AnovaKernelOperator (anova.py:146-183)
    w1 = synthetic.c1()
    op = AnovaKernelOperator(w1.X, w1.windows, w1.sigma, profile=AccuracyProfile("c1", 2.0, 2),
                             config=PeriodizationConfig(coeff_grid=32))
    g["c1_out"] = op.apply(w1.alpha)

    # --- C3 / C4 / C5 at reduced N through the composed recipe
    w3 = synthetic.c3(N=1500)
    g["c3s_out"] = composed(w3.X, w3.windows, w3.sigma, w3.M, w3.m, w3.alpha)
    w4 = synthetic.c4(N=2000, R=3)
    g["c4s_out"] = np.stack([composed(w4.X, w4.windows, w4.sigma, w4.M, w4.m, w4.alpha[:, r])
                             for r in range(w4.R)], axis=1)
    w5 = synthetic.c5(N=2000)
    g["c5s_out"] = composed(w5.X, w5.windows, w5.sigma, w5.M, w5.m, w5.alpha)

    # --- C2 CG (krr.py:76-110 as used by fit, krr.py:162-167) + predict (krr.py:181-196)
    w2 = synthetic.c2(N=1200, n_test=400)
    op2 = AnovaKernelOperator(w2.X, w2.windows, w2.sigma, "default")
    res = cg_solve(lambda v: op2.apply(v) + w2.beta * v, w2.y, tol=1e-6, maxiter=200)
    tight = cg_solve(lambda v: op2.apply(v) + w2.beta * v, w2.y, tol=1e-12, maxiter=400)
    g["c2s_x"] = res.x
    g["c2s_iters"] = np.array(res.iterations)
    g["c2s_resid"] = np.array(res.residual)
    g["c2s_x_tight"] = tight.x
    g["c2s_iters_tight"] = np.array(tight.iterations)
    g["c2s_apply_y"] = op2.apply(w2.y)
    pred = AnovaKernelOperator(w2.X, w2.windows, w2.sigma, "default", targets=w2.Z)
    g["c2s_decision"] = pred.apply(res.x)

    g["meta_json"] = np.array(json.dumps(meta))
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes;", len(g), "arrays")


if __name__ == "__main__":
    main()
