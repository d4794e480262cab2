"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck/racecheck):

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
covers 1-D/2-D/3-D windows, the tensor-core 2-D kernels (window-matrix and, forced on here,
Chebyshev; the sub-cell kernels in a second, forced pass), the (AFS_TC3=1) 3-D tensor-core kernels,
the table-based fused 1-D gather, targets, multi-RHS, the per-window
pipeline, deterministic mode, the device CG (whole-solve graph, fused cooperative epilogue),
concurrent applies on workspace clones, apply_complex and the sharded-CG vector kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402

os.environ.setdefault("AFS_TC3", "1")
os.environ.setdefault("AFS_CHEB", "1")
os.environ.setdefault("AFS_CHEB_SPREAD", "1")
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
# the sub-cell 2-D kernels (forced regardless of density) and two 1-D windows (fused table gather)
os.environ["AFS_SC"] = "2"
for tgt in (None, Z):
    ops = afs.AnovaKernelOperator(X, [(3, 4), (1, 4), (5,), (0,)], 0.3, prof, tgt, cfg, strict=False, max_rhs=3)
    ys = ops.apply(A)
    os.environ["AFS_SC"] = "0"
    oph = afs.AnovaKernelOperator(X, [(3, 4), (1, 4), (5,), (0,)], 0.3, prof, tgt, cfg, strict=False, max_rhs=3)
    os.environ["AFS_SC"] = "2"
    print("sub-cell vs half-cell kernels", float(np.max(np.abs(ys - oph.apply(A))) / np.max(np.abs(ys))))
os.environ.pop("AFS_SC")
det = afs.AnovaKernelOperator(X, windows, 0.3, prof, None, cfg, strict=False, max_rhs=3, deterministic=True)
det.apply(A)
res = afs.cg_solve(afs.KernelSystem(det, 0.5), A[:, 1], tol=1e-8, maxiter=30)
print("cg", res.iterations, res.residual)

res = afs.cg_solve(afs.KernelSystem(op_sq := afs.AnovaKernelOperator(X, windows, 0.3, prof, None, cfg,
                                                                     strict=False), 0.5),
                   A[:, 2], tol=1e-8, maxiter=30)
print("cg (atomic, pipeline)", res.iterations, res.residual)

import threading  # noqa: E402

import torch  # noqa: E402

outs = [None] * 4


def worker(k):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        outs[k] = op_sq.apply(torch.from_numpy(A[:, k % 3].copy()).cuda()).cpu().numpy()


ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
for t in ths:
    t.start()
for t in ths:
    t.join()
print("concurrent applies", float(np.max(np.abs(outs[0] - outs[3]))))

fs = afs.FastsumOperator(afs.GaussianKernel(0.3), cfg, X[:, :2], Z[:, :2], prof)
print("apply_complex", float(np.abs(fs.apply_complex(A[:, 0] + 1j * A[:, 1])).max()))

from paper_2111_10140_b200.cg import CudaCgVectors, run_cg  # noqa: E402

b = torch.from_numpy(A[:, 0].copy()).cuda()
r = run_cg(lambda v: op_sq.apply(v), b, 0.5, 1e-8, 20, CudaCgVectors(b.device))
print("vector-kernel cg", r.iterations, r.residual)
