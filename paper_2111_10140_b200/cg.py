"""One conjugate-gradient control loop for every driver of the path (reference: cg_solve,
krr.py:68-110).

The reference runs CG as an inline numpy loop.  Here the loop is written once
against a small "vector backend" interface, so that the same stopping rule,
iteration count and breakdown checks drive

* host numpy vectors for an arbitrary ``apply_A`` callable (``NumpyCgVectors``:
  the same elementwise expressions as krr.py:91-109, hence the same rounding),
* device tensors through the fused C-ABI kernels (``CudaCgVectors``,
  ``afs_cg_vec_*``) for sharded multi-GPU solves, and
* a torch CPU mirror of those kernels (``TorchCgVectors``) for the gloo tests.

The single-plan GPU solve does not come through here: it is one CUDA graph with a
device-side loop (``afs_cg_solve``, csrc/cg.cu) applying the same rule.

Workspace layout shared by all backends (include/anovafs.h, AFS_CG_WORKSPACE_DOUBLES):
``ws[0]`` rs = r.r, ``ws[1]`` p.Ap, ``ws[2]`` rs_new, ``ws[3]`` non-finite flag of Ap,
``ws[9]`` the shift beta.  Each backend writes LOCAL partial sums; ``reduce(view)``
(an all-reduce for row-sharded vectors, a no-op otherwise) makes them global.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import NumericalError

WS_DOUBLES = 640


@dataclass
class CgResult:
    """Outcome of a solve: x, iterations used, final relative residual, converged flag
    (the reference's CgResult fields, krr.py:68-73)."""

    x: object
    iterations: int
    residual: float
    converged: bool


def _breakdown(it, pAp, rs_new, bad):
    """The reference's three breakdown checks in its order (krr.py:93-106)."""
    if bad:
        return f"CG breakdown: non-finite operator output at iteration {it}"
    if not (math.isfinite(pAp) and pAp > 0.0):
        return f"CG breakdown: non-positive curvature {pAp:.3e} at iteration {it}"
    if not math.isfinite(rs_new):
        return f"CG breakdown: non-finite residual at iteration {it}"
    return None


def run_cg(matvec, b, beta, tol, maxiter, vectors, reduce=None):
    """Plain CG on (A + beta I) x = b from x0 = 0, A given by ``matvec``.

    Stops when sqrt(r.r) <= tol ||b|| (recurrence residual) or after ``maxiter``
    iterations; raises NumericalError naming the iteration on breakdown.  ``reduce``
    sums a workspace slice across ranks in place (row-sharded vectors)."""
    ws = vectors.workspace()
    x, r, p = vectors.init(b, beta, ws)
    if reduce is not None:
        reduce(ws, 0, 1)
    b_norm = math.sqrt(vectors.scalars(ws, 0, 1)[0])
    if b_norm == 0.0:
        return CgResult(x, 0, 0.0, True)
    bar = tol * b_norm
    for it in range(1, maxiter + 1):
        ap = matvec(p)
        vectors.ap(ap, p, ws)
        if reduce is not None:
            reduce(ws, 1, 4)
        vectors.update(x, r, p, ap, ws)
        if reduce is not None:
            reduce(ws, 2, 3)
        pAp, rs_new, bad = vectors.scalars(ws, 1, 4)
        msg = _breakdown(it, pAp, rs_new, bad != 0.0)
        if msg:
            raise NumericalError(msg)
        if math.sqrt(rs_new) <= bar:
            return CgResult(x, it, math.sqrt(rs_new) / b_norm, True)
        vectors.direction(p, r, ws)
    return CgResult(x, maxiter, math.sqrt(vectors.scalars(ws, 0, 1)[0]) / b_norm, False)


class NumpyCgVectors:
    """Host vectors for a generic ``apply_A`` callable (the shift is already inside it)."""

    def workspace(self):
        return np.zeros(WS_DOUBLES)

    def scalars(self, ws, lo, hi):
        return [float(v) for v in ws[lo:hi]]

    def init(self, b, beta, ws):
        ws[:16] = 0.0
        ws[9] = beta
        ws[0] = float(b @ b)
        return np.zeros_like(b), b.copy(), b.copy()

    def ap(self, ap, p, ws):
        if ws[9] != 0.0:
            ap += ws[9] * p
        ws[3] = 0.0 if np.all(np.isfinite(ap)) else 1.0
        ws[1] = float(p @ ap)

    def update(self, x, r, p, ap, ws):
        step = ws[0] / ws[1]
        x += step * p
        r -= step * ap
        ws[2] = float(r @ r)

    def direction(self, p, r, ws):
        p[:] = r + (ws[2] / ws[0]) * p
        ws[0] = ws[2]


class TorchCgVectors(NumpyCgVectors):
    """torch CPU mirror of the afs_cg_vec_* kernels (gloo tests of the sharded drivers)."""

    def __init__(self):
        import torch

        self.torch = torch

    def workspace(self):
        return self.torch.zeros(WS_DOUBLES, dtype=self.torch.float64)

    def scalars(self, ws, lo, hi):
        return [float(v) for v in ws[lo:hi].tolist()]

    def init(self, b, beta, ws):
        ws[:16] = 0.0
        ws[9] = beta
        ws[0] = self.torch.dot(b, b)
        return self.torch.zeros_like(b), b.clone(), b.clone()

    def ap(self, ap, p, ws):
        ap.add_(ws[9] * p)
        ws[3] = 0.0 if bool(self.torch.isfinite(ap).all()) else 1.0
        ws[1] = self.torch.dot(p, ap)

    def update(self, x, r, p, ap, ws):
        step = ws[0] / ws[1]
        x.add_(step * p)
        r.sub_(step * ap)
        ws[2] = self.torch.dot(r, r)

    def direction(self, p, r, ws):
        p.copy_(r + (ws[2] / ws[0]) * p)
        ws[0] = ws[2]


class CudaCgVectors:
    """Device vectors updated by the fused C-ABI kernels (afs_cg_vec_*, csrc/cg.cu):
    one pass per update with its dot product, fixed-order reductions."""

    def __init__(self, device):
        import torch

        from . import _native

        self.torch = torch
        self.native = _native
        self.lib = _native.load()
        self.device = device

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def workspace(self):
        return self.torch.zeros(WS_DOUBLES, dtype=self.torch.float64, device=self.device)

    def scalars(self, ws, lo, hi):
        return [float(v) for v in ws[lo:hi].cpu().tolist()]   # the one sync per iteration

    def init(self, b, beta, ws):
        t = self.torch
        x, r, p = t.empty_like(b), t.empty_like(b), t.empty_like(b)
        self.native.check(self.lib.afs_cg_vec_init(b.data_ptr(), x.data_ptr(), r.data_ptr(),
                                                   p.data_ptr(), b.numel(), float(beta),
                                                   ws.data_ptr(), self._stream()))
        return x, r, p

    def ap(self, ap, p, ws):
        self.native.check(self.lib.afs_cg_vec_ap(ap.data_ptr(), p.data_ptr(), p.numel(),
                                                 ws.data_ptr(), self._stream()))

    def update(self, x, r, p, ap, ws):
        self.native.check(self.lib.afs_cg_vec_update(x.data_ptr(), r.data_ptr(), p.data_ptr(),
                                                     ap.data_ptr(), p.numel(), ws.data_ptr(),
                                                     self._stream()))

    def direction(self, p, r, ws):
        self.native.check(self.lib.afs_cg_vec_direction(p.data_ptr(), r.data_ptr(), p.numel(),
                                                        ws.data_ptr(), self._stream()))
