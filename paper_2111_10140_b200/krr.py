"""Conjugate-gradient kernel ridge regression on the GPU operator (krr.py:68-110).

``cg_solve(apply_A, b, tol, maxiter)`` keeps the reference signature.  When
``apply_A`` is a ``KernelSystem`` (``op + beta*I`` on an ``AnovaKernelOperator``),
the whole loop runs device-resident through ``afs_cg_solve`` (fused vector
updates, deterministic reductions, one scalar read-back per iteration).  Any
other callable gets the reference's host loop unchanged (it is the
compatibility path for user-defined operators, not the hot path).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import NumericalError, ShapeError, ValidationError
from .operators import AnovaKernelOperator, _torch


@dataclass
class CgResult:
    x: np.ndarray
    iterations: int
    residual: float
    converged: bool


class KernelSystem:
    """The SPD system matrix K + beta I of KRR training (krr.py:162-167)."""

    def __init__(self, operator: AnovaKernelOperator, beta: float):
        if not isinstance(operator, AnovaKernelOperator):
            raise ValidationError("KernelSystem needs an AnovaKernelOperator")
        if operator.n_targets != operator.n_sources:
            raise ValidationError("KernelSystem needs a square operator (no targets)")
        if not beta > 0:
            raise ValidationError(f"lambda must be positive, got {beta}")
        self.operator = operator
        self.beta = float(beta)

    def __call__(self, v):
        return self.operator.apply(v) + self.beta * v


def _device_cg(system: KernelSystem, b, tol, maxiter):
    torch = _torch()
    plan = system.operator._plan
    on_dev = hasattr(b, "is_cuda") and b.is_cuda
    bd = (b if on_dev else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)))
    bd = bd.to(device=plan.device, dtype=torch.float64).contiguous()
    if bd.dim() != 1 or bd.shape[0] != plan.N:
        raise ShapeError(f"b must have length {plan.N}, got {tuple(bd.shape)}")
    x = torch.empty_like(bd)
    it, res, conv = plan.cg_device(bd, x, system.beta, tol, maxiter)
    torch.cuda.current_stream(plan.device).synchronize()
    return CgResult(x if on_dev else x.cpu().numpy(), it, res, conv)


def cg_solve(apply_A, b, tol=1e-3, maxiter=1000):
    """CG for SPD systems from x0 = 0 without preconditioner; stops when
    ||r|| <= tol ||b|| (recurrence residual) or after maxiter iterations."""
    if isinstance(apply_A, KernelSystem):
        return _device_cg(apply_A, b, tol, maxiter)
    b = np.asarray(b, dtype=np.float64)
    b_norm = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    if b_norm == 0.0:
        return CgResult(x, 0, 0.0, True)
    r = b.copy()
    p = r.copy()
    rs = float(r @ r)
    for it in range(1, maxiter + 1):
        Ap = np.asarray(apply_A(p), dtype=np.float64)
        if not np.all(np.isfinite(Ap)):
            raise NumericalError(f"CG breakdown: non-finite operator output at iteration {it}")
        pAp = float(p @ Ap)
        if not math.isfinite(pAp) or pAp <= 0.0:
            raise NumericalError(f"CG breakdown: non-positive curvature {pAp:.3e} at iteration {it}")
        step = rs / pAp
        x += step * p
        r -= step * Ap
        rs_new = float(r @ r)
        if not math.isfinite(rs_new):
            raise NumericalError(f"CG breakdown: non-finite residual at iteration {it}")
        if math.sqrt(rs_new) <= tol * b_norm:
            return CgResult(x, it, math.sqrt(rs_new) / b_norm, True)
        p = r + (rs_new / rs) * p
        rs = rs_new
    return CgResult(x, maxiter, math.sqrt(rs) / b_norm, False)
