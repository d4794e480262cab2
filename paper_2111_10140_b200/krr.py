"""Kernel ridge regression around the GPU operator: the CG entry point and the fit /
decision / predict / model-document wrappers (reference krr.py:68-202, 269-330).

``cg_solve(apply_A, b, tol, maxiter)`` keeps the reference signature and routes
by the type of ``apply_A``:

* ``KernelSystem`` over an ``AnovaKernelOperator``: the whole solve is one CUDA graph
  with a device-side loop (``afs_cg_solve``, csrc/cg.cu);
* ``KernelSystem`` over a ``WindowSharded`` / ``PointSharded`` operator: the shared
  control loop ``cg.run_cg`` with the fused device vector kernels and NCCL
  all-reduces (``distributed.sharded_cg``);
* any other callable: the same control loop on host numpy vectors (compatibility
  path for user-defined operators, not the hot path).

``fit`` builds its operator in deterministic mode (fixed-point spread, bit-identical
run to run), so a fitted model -- and its CG iteration count -- is reproducible.
"""

from __future__ import annotations

import base64
import json
from dataclasses import dataclass

import numpy as np

from .cg import CgResult, NumpyCgVectors, run_cg
from .errors import ShapeError, ValidationError
from .operators import AnovaKernelOperator, WindowSet, _torch
from .prep import ScalerStats, build_windows, mis_scores, zscore_apply, zscore_fit

MODEL_FORMAT = "krr-model/1"
RNG_NAME = "numpy-pcg64"
DETERMINISTIC_MAX_NODES = 1 << 27   # afs_plan_set_deterministic limb headroom

__all__ = ["CgResult", "KernelSystem", "KrrConfig", "KrrModel", "cg_solve", "fit",
           "decision_values", "predict", "model_to_dict", "model_from_dict", "save_model",
           "load_model"]


# ----------------------------------------------------------------------------- CG
class KernelSystem:
    """The shifted system K + beta I of KRR training (krr.py:162-167) over a GPU operator:
    an ``AnovaKernelOperator`` or a sharded one (``distributed.WindowSharded`` /
    ``distributed.PointSharded``).  Calling it applies the system; ``cg_solve`` solves it
    on the device."""

    def __init__(self, operator, beta: float):
        from .distributed import PointSharded, WindowSharded

        if not isinstance(operator, (AnovaKernelOperator, WindowSharded, PointSharded)):
            raise ValidationError("KernelSystem needs an AnovaKernelOperator or a sharded operator")
        if isinstance(operator, AnovaKernelOperator) and operator.n_targets != operator.n_sources:
            raise ValidationError("KernelSystem needs a square operator (no targets)")
        if not beta > 0:
            raise ValidationError(f"lambda must be positive, got {beta}")
        self.operator = operator
        self.beta = float(beta)

    def __call__(self, v):
        return self.operator.apply(v) + self.beta * v

    def solve(self, b, tol, maxiter):
        if isinstance(self.operator, AnovaKernelOperator):
            return self._solve_plan(b, tol, maxiter)
        from .distributed import sharded_cg

        torch = _torch()
        on_device = hasattr(b, "is_cuda") and b.is_cuda
        if not on_device:
            dev = torch.device("cuda", torch.cuda.current_device())
            b = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to(dev)
        res = sharded_cg(self.operator, b, self.beta, tol, maxiter)
        if not on_device:
            res.x = res.x.cpu().numpy()
        return res

    def _solve_plan(self, b, tol, maxiter):
        torch = _torch()
        plan = self.operator._plan
        on_device = hasattr(b, "is_cuda") and b.is_cuda
        src = b if on_device else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64))
        bd = src.to(device=plan.device, dtype=torch.float64).contiguous()
        if bd.dim() != 1 or bd.shape[0] != plan.N:
            raise ShapeError(f"b must have length {plan.N}, got {tuple(bd.shape)}")
        x = torch.empty_like(bd)
        it, res, conv = plan.cg_device(bd, x, self.beta, tol, maxiter)
        torch.cuda.current_stream(plan.device).synchronize()
        return CgResult(x if on_device else x.cpu().numpy(), it, res, conv)


def cg_solve(apply_A, b, tol=1e-3, maxiter=1000):
    """CG for SPD systems from x0 = 0, no preconditioner: stops when ||r|| <= tol ||b||
    (recurrence residual) or after maxiter iterations (reported, not fatal); NaN/Inf in
    the recurrence raises NumericalError naming the iteration (krr.py:76-110)."""
    if isinstance(apply_A, KernelSystem):
        return apply_A.solve(b, tol, maxiter)
    rhs = np.asarray(b, dtype=np.float64)
    return run_cg(lambda v: np.asarray(apply_A(v), dtype=np.float64), rhs, 0.0, tol, maxiter,
                  NumpyCgVectors())


# ----------------------------------------------------------------------------- config
# (predicate, message) pairs checked in order; messages are the reference's (API contract)
_CONFIG_RULES = (
    (lambda c: c.sigma > 0, lambda c: f"sigma must be positive, got {c.sigma}"),
    (lambda c: c.lam > 0, lambda c: f"lambda must be positive, got {c.lam}"),
    (lambda c: 0.0 < c.cg_tol < 1.0, lambda c: f"cg_tol must lie in (0, 1), got {c.cg_tol}"),
    (lambda c: c.cg_maxiter >= 1, lambda c: "cg_maxiter must be at least 1"),
    (lambda c: c.mis_threshold >= 0, lambda c: "mis_threshold must be nonnegative"),
)
# attribute -> key in the "krr-model/1" document
_CONFIG_KEYS = {"sigma": "sigma", "lam": "lambda", "cg_tol": "cg_tol", "cg_maxiter": "cg_maxiter",
                "profile": "profile", "mis_threshold": "mis_threshold"}


@dataclass(frozen=True)
class KrrConfig:
    """KRR hyper-parameters (krr.py:25-65)."""

    sigma: float = 1.0
    lam: float = 1.0
    cg_tol: float = 1e-3
    cg_maxiter: int = 1000
    profile: str = "default"
    mis_threshold: float = 0.0

    def __post_init__(self):
        for ok, msg in _CONFIG_RULES:
            if not ok(self):
                raise ValidationError(msg(self))

    def to_dict(self):
        return {key: getattr(self, attr) for attr, key in _CONFIG_KEYS.items()}

    @classmethod
    def from_dict(cls, d):
        return cls(**{attr: d[key] for attr, key in _CONFIG_KEYS.items()})


# ----------------------------------------------------------------------------- model
@dataclass(eq=False)
class KrrModel:
    """A fitted classifier: expansion coefficients over the scaled training rows, the
    windows and scaler that produced them, and the CG outcome (krr.py:113-135)."""

    alpha: np.ndarray
    config: KrrConfig
    windows: WindowSet
    scaler: ScalerStats
    train_scaled: np.ndarray
    column_names: tuple
    cg_iterations: int
    cg_residual: float
    cg_converged: bool

    def __post_init__(self):
        self.alpha = np.asarray(self.alpha, dtype=np.float64)
        self.train_scaled = np.asarray(self.train_scaled, dtype=np.float64)
        self.column_names = tuple(self.column_names)
        self.cg_iterations = int(self.cg_iterations)
        self.cg_residual = float(self.cg_residual)
        self.cg_converged = bool(self.cg_converged)

    @property
    def n_train(self):
        return self.train_scaled.shape[0]

    @property
    def n_features(self):
        return self.train_scaled.shape[1]

    def operator(self, targets=None, **kw):
        """The ANOVA operator over the training rows (targets: scaled test rows)."""
        return AnovaKernelOperator(self.train_scaled, self.windows, self.config.sigma,
                                   self.config.profile, targets=targets, **kw)


def _training_arrays(X, y):
    """(X, y as float) after the reference's training-input checks (krr.py:137-149)."""
    A = np.atleast_2d(np.asarray(X, dtype=np.float64))
    lab = np.asarray(y)
    if A.ndim != 2 or A.shape[0] < 2:
        raise ValidationError("training needs at least 2 samples")
    if lab.shape != (A.shape[0],):
        raise ShapeError("labels must match the number of training rows")
    present = np.unique(lab)
    if not np.isin(present, (-1, 1)).all():
        raise ValidationError(f"labels must be -1 or +1, got {present}")
    if present.size < 2:
        raise ValidationError("training data must contain both classes")
    return A, lab.astype(np.float64)


def fit(X_train, y_train, config, column_names=None):
    """z-score -> MIS windows -> GPU ANOVA operator -> device CG (krr.py:152-178)."""
    X, y = _training_arrays(X_train, y_train)
    names = column_names if column_names is not None else [f"f{i}" for i in range(X.shape[1])]
    scaler = zscore_fit(X)
    Xs = zscore_apply(scaler, X)
    windows = build_windows(mis_scores(Xs, y_train), config.mis_threshold)
    op = AnovaKernelOperator(Xs, windows, config.sigma, config.profile,
                             deterministic=Xs.shape[0] <= DETERMINISTIC_MAX_NODES)
    sol = cg_solve(KernelSystem(op, config.lam), y, tol=config.cg_tol, maxiter=config.cg_maxiter)
    op.close()
    return KrrModel(sol.x, config, windows, scaler, Xs, names, sol.iterations, sol.residual,
                    sol.converged)


def decision_values(model, X_test):
    """s(z) = sum_j alpha_j k_anova(z, x_j): the operator rebuilt with the scaled test rows
    as targets (union-bbox scaling, krr.py:181-196)."""
    Z = np.atleast_2d(np.asarray(X_test, dtype=np.float64))
    if Z.shape[1] != model.n_features:
        raise ValidationError(
            f"test data has {Z.shape[1]} columns, model was trained on {model.n_features}")
    op = model.operator(targets=zscore_apply(model.scaler, Z))
    out = op.apply(model.alpha)
    op.close()
    return out


def predict(model, X_test):
    """Labels in {-1, +1}, threshold 0 with sign(0) -> +1 (krr.py:199-202)."""
    return np.where(decision_values(model, X_test) >= 0.0, 1, -1).astype(np.int64)


# ----------------------------------------------------------------------------- document
def _b64(arr):
    return base64.b64encode(np.ascontiguousarray(arr, dtype="<f8").tobytes()).decode("ascii")


def _unb64(text, shape):
    raw = np.frombuffer(base64.b64decode(text.encode("ascii")), dtype="<f8")
    return raw.reshape(shape).astype(np.float64)


def model_to_dict(model):
    """The versioned "krr-model/1" JSON document (krr.py:269-297)."""
    return {
        "format": MODEL_FORMAT,
        "config": model.config.to_dict(),
        "column_names": list(model.column_names),
        "windows": model.windows.to_dict(),
        "scaler": {"means": model.scaler.means.tolist(), "stds": model.scaler.stds.tolist()},
        "train_shape": list(model.train_scaled.shape),
        "alpha_b64": _b64(model.alpha),
        "train_scaled_b64": _b64(model.train_scaled),
        "cg": {"iterations": model.cg_iterations, "residual": model.cg_residual,
               "converged": model.cg_converged},
        "rng": RNG_NAME,
    }


def model_from_dict(doc):
    if doc.get("format") != MODEL_FORMAT:
        raise ValidationError(
            f"unsupported model format {doc.get('format')!r}, expected {MODEL_FORMAT}")
    shape = tuple(doc["train_shape"])
    cg = doc["cg"]
    return KrrModel(
        alpha=_unb64(doc["alpha_b64"], shape[:1]),
        config=KrrConfig.from_dict(doc["config"]),
        windows=WindowSet([tuple(w) for w in doc["windows"]["windows"]]),
        scaler=ScalerStats(*(np.asarray(doc["scaler"][k], dtype=np.float64)
                             for k in ("means", "stds"))),
        train_scaled=_unb64(doc["train_scaled_b64"], shape),
        column_names=doc["column_names"],
        cg_iterations=cg["iterations"], cg_residual=cg["residual"], cg_converged=cg["converged"],
    )


def save_model(model, path):
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(model_to_dict(model), indent=1) + "\n")


def load_model(path):
    with open(path, encoding="utf-8") as fh:
        return model_from_dict(json.load(fh))
