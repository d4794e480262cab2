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


MODEL_FORMAT = "krr-model/1"
RNG_NAME = "numpy-pcg64"


@dataclass(frozen=True)
class KrrConfig:
    """KRR hyper-parameters (krr.py:25-65): sigma, lam, CG tol/maxiter, profile, MIS threshold."""

    sigma: float = 1.0
    lam: float = 1.0
    cg_tol: float = 1e-3
    cg_maxiter: int = 1000
    profile: str = "default"
    mis_threshold: float = 0.0

    def __post_init__(self):
        if self.sigma <= 0:
            raise ValidationError(f"sigma must be positive, got {self.sigma}")
        if self.lam <= 0:
            raise ValidationError(f"lambda must be positive, got {self.lam}")
        if not 0.0 < self.cg_tol < 1.0:
            raise ValidationError(f"cg_tol must lie in (0, 1), got {self.cg_tol}")
        if self.cg_maxiter < 1:
            raise ValidationError("cg_maxiter must be at least 1")
        if self.mis_threshold < 0:
            raise ValidationError("mis_threshold must be nonnegative")

    def to_dict(self):
        return {"sigma": self.sigma, "lambda": self.lam, "cg_tol": self.cg_tol,
                "cg_maxiter": self.cg_maxiter, "profile": self.profile,
                "mis_threshold": self.mis_threshold}

    @classmethod
    def from_dict(cls, d):
        return cls(sigma=d["sigma"], lam=d["lambda"], cg_tol=d["cg_tol"],
                   cg_maxiter=d["cg_maxiter"], profile=d["profile"],
                   mis_threshold=d["mis_threshold"])


class KrrModel:
    """Fitted KRR classifier: coefficients, windows, scaler, training nodes (krr.py:113-135)."""

    def __init__(self, alpha, config, windows, scaler, train_scaled, column_names,
                 cg_iterations, cg_residual, cg_converged):
        self.alpha = np.asarray(alpha, dtype=np.float64)
        self.config = config
        self.windows = windows
        self.scaler = scaler
        self.train_scaled = np.asarray(train_scaled, dtype=np.float64)
        self.column_names = tuple(column_names)
        self.cg_iterations = int(cg_iterations)
        self.cg_residual = float(cg_residual)
        self.cg_converged = bool(cg_converged)

    @property
    def n_train(self):
        return self.train_scaled.shape[0]

    @property
    def n_features(self):
        return self.train_scaled.shape[1]


def _training_input(X, y):
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    y = np.asarray(y)
    if X.ndim != 2 or X.shape[0] < 2:
        raise ValidationError("training needs at least 2 samples")
    if y.shape != (X.shape[0],):
        raise ShapeError("labels must match the number of training rows")
    vals = np.unique(y)
    if not np.all(np.isin(vals, (-1, 1))):
        raise ValidationError(f"labels must be -1 or +1, got {vals}")
    if vals.size < 2:
        raise ValidationError("training data must contain both classes")
    return X, y.astype(np.float64)


def fit(X_train, y_train, config, column_names=None):
    """z-score -> MIS ranking -> windows -> GPU ANOVA operator -> device CG (krr.py:152-178)."""
    from .windowing import build_windows, mis_scores, zscore_apply, zscore_fit

    X, y = _training_input(X_train, y_train)
    if column_names is None:
        column_names = tuple(f"f{i}" for i in range(X.shape[1]))
    scaler = zscore_fit(X)
    Xs = zscore_apply(scaler, X)
    windows = build_windows(mis_scores(Xs, y_train), config.mis_threshold)
    op = AnovaKernelOperator(Xs, windows, config.sigma, config.profile)
    res = cg_solve(KernelSystem(op, config.lam), y, tol=config.cg_tol, maxiter=config.cg_maxiter)
    return KrrModel(res.x, config, windows, scaler, Xs, column_names, res.iterations,
                    res.residual, res.converged)


def decision_values(model, X_test):
    """s(z) = sum_j alpha_j k_anova(z, x_j): operator rebuilt with targets (krr.py:181-196)."""
    from .windowing import zscore_apply

    X_test = np.atleast_2d(np.asarray(X_test, dtype=np.float64))
    if X_test.shape[1] != model.n_features:
        raise ValidationError(
            f"test data has {X_test.shape[1]} columns, model was trained on {model.n_features}")
    Zs = zscore_apply(model.scaler, X_test)
    op = AnovaKernelOperator(model.train_scaled, model.windows, model.config.sigma,
                             model.config.profile, targets=Zs)
    return op.apply(model.alpha)


def predict(model, X_test):
    """Labels in {-1, +1}; sign(0) -> +1 (krr.py:199-202)."""
    return np.where(decision_values(model, X_test) >= 0.0, 1, -1).astype(np.int64)


def _enc(arr):
    import base64

    return base64.b64encode(np.ascontiguousarray(arr, dtype="<f8").tobytes()).decode("ascii")


def _dec(text, shape):
    import base64

    return np.frombuffer(base64.b64decode(text.encode("ascii")), dtype="<f8").reshape(shape).astype(
        np.float64)


def model_to_dict(model):
    """The reference's versioned "krr-model/1" document (krr.py:269-297)."""
    return {
        "format": MODEL_FORMAT,
        "config": model.config.to_dict(),
        "column_names": list(model.column_names),
        "windows": model.windows.to_dict(),
        "scaler": {"means": [float(v) for v in model.scaler.means],
                   "stds": [float(v) for v in model.scaler.stds]},
        "train_shape": list(model.train_scaled.shape),
        "alpha_b64": _enc(model.alpha),
        "train_scaled_b64": _enc(model.train_scaled),
        "cg": {"iterations": model.cg_iterations, "residual": model.cg_residual,
               "converged": model.cg_converged},
        "rng": RNG_NAME,
    }


def model_from_dict(doc):
    from .operators import WindowSet
    from .windowing import ScalerStats

    if doc.get("format") != MODEL_FORMAT:
        raise ValidationError(
            f"unsupported model format {doc.get('format')!r}, expected {MODEL_FORMAT}")
    shape = tuple(doc["train_shape"])
    return KrrModel(
        alpha=_dec(doc["alpha_b64"], (shape[0],)),
        config=KrrConfig.from_dict(doc["config"]),
        windows=WindowSet(tuple(tuple(w) for w in doc["windows"]["windows"])),
        scaler=ScalerStats(means=np.asarray(doc["scaler"]["means"], dtype=np.float64),
                           stds=np.asarray(doc["scaler"]["stds"], dtype=np.float64)),
        train_scaled=_dec(doc["train_scaled_b64"], shape),
        column_names=tuple(doc["column_names"]),
        cg_iterations=doc["cg"]["iterations"],
        cg_residual=doc["cg"]["residual"],
        cg_converged=doc["cg"]["converged"],
    )


def save_model(model, path):
    import json

    with open(path, "w", encoding="utf-8") as fh:
        json.dump(model_to_dict(model), fh, indent=1)
        fh.write("\n")


def load_model(path):
    import json

    with open(path, encoding="utf-8") as fh:
        return model_from_dict(json.load(fh))


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
