"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck/racecheck):

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
covers 1-D/2-D/3-D windows, the tensor-core 2-D and (AFS_TC3=1) 3-D kernels, targets,
multi-RHS, deterministic mode and the device CG."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402

os.environ.setdefault("AFS_TC3", "1")
rng = np.random.default_rng(0)
N, Nt = 3000, 1000
centers = rng.uniform(-0.2, 0.2, size=(3, 6))
X = np.clip(centers[rng.integers(0, 3, N)] + 0.02 * rng.standard_normal((N, 6)), -0.25, 0.2499)
Z = rng.uniform(-0.25, 0.25, size=(Nt, 6))
windows = [(0, 1, 2), (3, 4), (5,), (1, 4)]
prof, cfg = afs.AccuracyProfile("s", 2.0, 4), afs.PeriodizationConfig(coeff_grid=16)
A = rng.standard_normal((N, 3))
for tgt in (None, Z):
    op = afs.AnovaKernelOperator(X, windows, 0.3, prof, tgt, cfg, strict=False, max_rhs=3)
    print("tensor-core windows", op._plan.info()["tensor_core_windows"])
    y = op.apply(A)
    y1 = op.apply(A[:, 0])
    print("rhs consistency", float(np.max(np.abs(y[:, 0] - y1))))
det = afs.AnovaKernelOperator(X, windows, 0.3, prof, None, cfg, strict=False, max_rhs=3, deterministic=True)
det.apply(A)
res = afs.cg_solve(afs.KernelSystem(det, 0.5), A[:, 1], tol=1e-8, maxiter=30)
print("cg", res.iterations, res.residual)
