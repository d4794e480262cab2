"""Golden vectors at the NAMED config sizes, produced by running the REFERENCE itself.

Run in the build container (where /root/reference exists), one job per process
(they are independent and take minutes to ~35 min each on one core):

    python tests/golden/make_golden_full.py c2      # N=100k: apply(y), 200-it CG, decision (20k)
    python tests/golden/make_golden_full.py c2cg50  # N=100k: 50-it CG (trajectory checkpoint)
    python tests/golden/make_golden_full.py c3      # N=1M composed 39-window matvec
    python tests/golden/make_golden_full.py c4      # N=1M, R=8 one 3-D window
    python tests/golden/make_golden_full.py c5      # N=1M composed 30-window matvec
    python tests/golden/make_golden_full.py c5cg    # C5 recipe CG at N=2000/8000 (converges)
    python tests/golden/make_golden_full.py complex # FastsumOperator.apply_complex cases
    python tests/golden/make_golden_full.py c2pertK # K=0,1,2: C2 CG with reordered windows

Inputs are regenerated from seeds (``paper_2111_10140_b200.synthetic``) on both
sides; only outputs are stored.  Vectors up to 1M entries are stored whole
(C2, C5).  For C3 (1M) and C4 (1M x 8) a seeded index sample is stored
together with full-vector linear functionals (sum, sum of squares, dot with a
seeded N(0,1) vector), so the tests check every entry in aggregate and a
sampled subset entry by entry.  SURVEY.md §8(c) recipes; reference files:
anova.py:175-183, fastsum.py:243-256, krr.py:76-110, krr.py:181-196.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import nfftkrr  # noqa: E402  (the reference)
from nfftkrr import (AccuracyProfile, AnovaKernelOperator, FastsumOperator,  # noqa: E402
                     GaussianKernel, PeriodizationConfig, cg_solve)

from paper_2111_10140_b200 import synthetic  # noqa: E402

from full_cases import SAMPLE_SEED, functionals, sample_rows  # noqa: E402


def _meta(**kw):
    import scipy
    kw.update(numpy=np.__version__, scipy=scipy.__version__,
              reference=getattr(nfftkrr, "__version__", "?"))
    return np.array(json.dumps(kw))


def _ops(w, Z=None):
    prof = AccuracyProfile("bench", w.oversampling, w.m)
    cfg = PeriodizationConfig(coeff_grid=w.M)
    return [FastsumOperator(GaussianKernel(w.sigma), cfg, w.X[:, list(win)],
                            None if Z is None else Z[:, list(win)], prof) for win in w.windows]


def _composed(ops, alpha):
    """sum_l (1/P) op_l(alpha) in window order (anova.py:179-183)."""
    P = len(ops)
    out = np.zeros(ops[0].n_targets)
    for op in ops:
        out += (1.0 / P) * op.apply(alpha)
    return out


def _save(name, **g):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **g)
    print("wrote", path, os.path.getsize(path), "bytes", flush=True)


def job_c2(maxiter=200, tag="c2full"):
    w = synthetic.c2()
    op = AnovaKernelOperator(w.X, w.windows, w.sigma, "default")
    g = {}
    t0 = time.time()
    if maxiter == 200:
        g["apply_y"] = op.apply(w.y)
        print("apply", time.time() - t0, flush=True)
    res = cg_solve(lambda v: op.apply(v) + w.beta * v, w.y, tol=1e-6, maxiter=maxiter)
    print("cg", res.iterations, res.residual, res.converged, time.time() - t0, flush=True)
    g["x"] = res.x
    g["iters"] = np.array(res.iterations)
    g["resid"] = np.array(res.residual)
    g["converged"] = np.array(res.converged)
    if maxiter == 200:
        pred = AnovaKernelOperator(w.X, w.windows, w.sigma, "default", targets=w.Z)
        g["decision"] = pred.apply(res.x)
    g["meta_json"] = _meta(job=tag, N=w.N, maxiter=maxiter, seconds=time.time() - t0)
    _save(f"golden_{tag}.npz", **g)


def job_c3():
    w = synthetic.c3(N=1_000_000)
    t0 = time.time()
    out = _composed(_ops(w), w.alpha)
    idx = sample_rows(w.N, 1 << 17)
    _save("golden_c3_1m.npz", idx=idx, out_sample=out[idx], func=functionals(out),
          meta_json=_meta(job="c3", N=w.N, seconds=time.time() - t0, sample_seed=SAMPLE_SEED))


def job_c4():
    w = synthetic.c4(N=1_000_000, R=8)
    t0 = time.time()
    (op,) = _ops(w)
    out = np.stack([op.apply(w.alpha[:, r]) for r in range(w.R)], axis=1)
    idx = sample_rows(w.N, 1 << 14)
    _save("golden_c4_1m.npz", idx=idx, out_sample=out[idx],
          func=np.stack([functionals(out[:, r]) for r in range(w.R)]),
          meta_json=_meta(job="c4", N=w.N, R=w.R, seconds=time.time() - t0,
                          sample_seed=SAMPLE_SEED))


def job_c5():
    w = synthetic.c5()
    t0 = time.time()
    out = _composed(_ops(w), w.alpha)
    _save("golden_c5_1m.npz", out=out, func=functionals(out),
          meta_json=_meta(job="c5", N=w.N, seconds=time.time() - t0))


def job_c5cg():
    g = {}
    meta = {}
    for N in (2000, 8000):
        w = synthetic.c5(N=N)
        ops = _ops(w)
        t0 = time.time()
        res = cg_solve(lambda v: _composed(ops, v) + w.beta * v, w.y, tol=1e-6, maxiter=1000)
        tight = cg_solve(lambda v: _composed(ops, v) + w.beta * v, w.y, tol=1e-11, maxiter=2000)
        # the reference's own roundoff sensitivity: the same recipe with the windows summed in
        # other orders (reverse + 3 seeded permutations; equally valid compositions whose
        # matvecs differ by ~1e-16)
        orders = [list(range(len(ops)))[::-1]] + [
            list(np.random.default_rng(100 + k).permutation(len(ops))) for k in range(3)]
        for k, order in enumerate(orders):
            perm_ops = [ops[i] for i in order]
            pert = cg_solve(lambda v: _composed(perm_ops, v) + w.beta * v, w.y, tol=1e-6,
                            maxiter=1000)
            g[f"n{N}_x_pert{k}"] = pert.x
            g[f"n{N}_iters_pert{k}"] = np.array(pert.iterations)
            print(N, "perturbation", k, pert.iterations,
                  np.linalg.norm(pert.x - res.x) / np.linalg.norm(res.x), flush=True)
        print(N, res.iterations, res.residual, tight.iterations, tight.residual,
              time.time() - t0, flush=True)
        g[f"n{N}_x"] = res.x
        g[f"n{N}_iters"] = np.array(res.iterations)
        g[f"n{N}_resid"] = np.array(res.residual)
        g[f"n{N}_x_tight"] = tight.x
        g[f"n{N}_iters_tight"] = np.array(tight.iterations)
        meta[N] = dict(iters=res.iterations, tight_iters=tight.iterations,
                       seconds=time.time() - t0)
    g["meta_json"] = _meta(job="c5cg", runs=meta)
    _save("golden_c5cg.npz", **g)


def job_c2pert(k):
    """The reference's own roundoff sensitivity on the named C2 solve: the same recipe with
    the three windows summed in another order (FastsumOperators composed as
    AnovaKernelOperator.apply does, anova.py:179-183), CG at 50 and 200 iterations.
    With three windows only two orders change the rounding ((c+b)+a and (a+c)+b; k = 0, 2):
    k = 1 ((b+a)+c) reproduces the golden bit for bit and is not kept."""
    order = [[2, 1, 0], [1, 0, 2], [0, 2, 1]][k]
    w = synthetic.c2()
    prof = AccuracyProfile("default", 2.0, 4)
    ops = _ops(w)
    ops = [ops[i] for i in order]
    t0 = time.time()
    g = {}
    for maxiter in (50, 200):
        res = cg_solve(lambda v: _composed(ops, v) + w.beta * v, w.y, tol=1e-6, maxiter=maxiter)
        g[f"x{maxiter}"] = res.x
        g[f"iters{maxiter}"] = np.array(res.iterations)
        g[f"resid{maxiter}"] = np.array(res.residual)
        print("c2pert", k, maxiter, res.iterations, res.residual, time.time() - t0, flush=True)
    g["meta_json"] = _meta(job=f"c2pert{k}", order=order, seconds=time.time() - t0)
    _save(f"golden_c2pert{k}.npz", **g)


def job_complex():
    """FastsumOperator.apply_complex (fastsum.py:243-252) on real and complex alpha."""
    from cases import FASTSUM_CASES, fastsum_inputs

    g = {}
    for tag, d, M, m, os_, sigma, N, n_tgt in FASTSUM_CASES[:7]:
        X, Z, alpha = fastsum_inputs(tag, d, N, n_tgt)
        op = FastsumOperator(GaussianKernel(sigma), PeriodizationConfig(coeff_grid=M), X, Z,
                             AccuracyProfile("golden", os_, m))
        calpha = alpha + 1j * np.random.default_rng(len(tag)).standard_normal(N)
        g[tag + "_real"] = op.apply_complex(alpha)
        g[tag + "_cplx"] = op.apply_complex(calpha)
    g["meta_json"] = _meta(job="complex")
    _save("golden_complex.npz", **g)


JOBS = {"c2": job_c2, "c2cg50": lambda: job_c2(50, "c2cg50"), "c3": job_c3, "c4": job_c4,
        "c5": job_c5, "c5cg": job_c5cg, "complex": job_complex,
        "c2pert0": lambda: job_c2pert(0), "c2pert1": lambda: job_c2pert(1),
        "c2pert2": lambda: job_c2pert(2)}

if __name__ == "__main__":
    for name in sys.argv[1:] or JOBS:
        JOBS[name]()
