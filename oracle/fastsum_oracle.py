"""CPU oracle for the ANOVA fast-summation matvec — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(arXiv 2111.10140 reference package ``nfftkrr``).  It exists so that the
GPU product path can be checked against the reference's arithmetic on the
GPU box, where ``/root/reference`` is not available.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
it; the product package ``paper_2111_10140_b200`` never does.

Parity pinning: every function below is checked against golden vectors
produced by running the reference itself (``tests/golden/make_golden.py``
imports ``/root/reference/pkg/src/nfftkrr``); see
``tests/test_oracle_golden.py``.

Reference file:line citations are relative to ``/root/reference/pkg/src/nfftkrr``.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.fft as sfft
from scipy.special import i0

# fastsum.py:52-87 (PeriodizationConfig defaults)
BALL_RADIUS = 0.25 - 1.0 / 32.0
TRANSITION_WIDTH = 1.0 / 16.0
SMOOTHNESS = 7
COEFF_OVERSAMPLE = 2

# nfft.py:54-58 (profile table: oversampling, cutoff)
PROFILE_TABLE = {"rough": (1.5, 3), "default": (2.0, 4), "fine": (2.0, 6)}
# fastsum.py:22 (coefficient grid per named profile; unknown names -> 64)
COEFF_GRID_TABLE = {"rough": 32, "default": 64, "fine": 128}


# ----------------------------------------------------------------------------
# NFFT building blocks
# ----------------------------------------------------------------------------

def oversampled_size(M: int, oversampling: float, m: int) -> int:
    """nfft.py:151-153: n = max(2m, even(ceil(sigma_os * M)))."""
    n = int(np.ceil(oversampling * M))
    n += n % 2
    return max(n, 2 * m)


def kb_shape(M: int, n: int) -> float:
    """nfft.py:156: b = pi (2 - M/n)."""
    return np.pi * (2.0 - M / n)


def kb_window(dist, m: int, b: float):
    """nfft.py:118-122: phi(t) = sinh(b s)/(pi s), s = sqrt(max(m^2-t^2,0)); b/pi at s<=1e-12."""
    dist = np.asarray(dist, dtype=np.float64)
    s = np.sqrt(np.maximum(m * m - dist * dist, 0.0))
    out = np.full(s.shape, b / np.pi)
    live = s > 1e-12
    out[live] = np.sinh(b * s[live]) / (np.pi * s[live])
    return out


def kb_fourier(k, n: int, m: int, b: float):
    """nfft.py:125-128: phi_hat(k) = I0(m sqrt(max(b^2-(2 pi k/n)^2,0))) / n."""
    k = np.asarray(k, dtype=np.float64)
    return i0(m * np.sqrt(np.maximum(b * b - (2.0 * np.pi * k / n) ** 2, 0.0))) / n


class NodeGeometry:
    """Per-dimension window cells and values of a node set (nfft.py:139-177).

    ``cells[t]`` is (N, 2m) int64 (already reduced mod n), ``vals[t]`` the
    matching (N, 2m) window values.
    """

    def __init__(self, coords, M: int, m: int, oversampling: float):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        if coords.ndim == 1:
            coords = coords[:, None]
        self.N, self.d = coords.shape
        self.M, self.m = int(M), int(m)
        self.n = oversampled_size(M, oversampling, m)
        self.b = kb_shape(M, self.n)
        modes = np.arange(-self.M // 2, self.M // 2)
        self.deconv = 1.0 / kb_fourier(modes, self.n, self.m, self.b)   # nfft.py:158-162
        shifts = np.arange(1 - self.m, self.m + 1)                       # nfft.py:166
        self.cells, self.vals = [], []
        for t in range(self.d):
            nx = self.n * coords[:, t]
            base = np.floor(nx).astype(np.int64)                          # nfft.py:170
            c = base[:, None] + shifts[None, :]
            self.vals.append(kb_window(nx[:, None] - c, self.m, self.b))  # nfft.py:172,174
            self.cells.append(np.mod(c, self.n))                          # nfft.py:173

    def _tensor(self, lo: int, hi: int):
        """Row-major flat cell index and product weight over the (2m)^d stencil."""
        flat = self.cells[0][lo:hi]
        w = self.vals[0][lo:hi]
        for t in range(1, self.d):
            flat = (flat[:, :, None] * self.n + self.cells[t][lo:hi, None, :]).reshape(hi - lo, -1)
            w = (w[:, :, None] * self.vals[t][lo:hi, None, :]).reshape(hi - lo, -1)
        return flat, w

    def _blocks(self, budget: int = 1 << 20):
        step = max(1, budget // (2 * self.m) ** self.d)
        for lo in range(0, self.N, step):
            yield lo, min(self.N, lo + step)

    def _mode_index(self):
        return np.ix_(*([np.arange(-self.M // 2, self.M // 2) % self.n] * self.d))

    def _scale_modes(self, arr):
        for t in range(self.d):
            shape = [1] * self.d
            shape[t] = -1
            arr = arr * self.deconv.reshape(shape)
        return arr

    def adjoint(self, c):
        """nfft.py:232-250: spread, fftn/n^d, keep I_M, deconvolve."""
        c = np.asarray(c).astype(np.complex128)
        total = self.n ** self.d
        g = np.zeros(total, dtype=np.complex128)
        for lo, hi in self._blocks():
            flat, w = self._tensor(lo, hi)
            contrib = c[lo:hi, None] * w
            g.real += np.bincount(flat.ravel(), contrib.real.ravel(), minlength=total)
            g.imag += np.bincount(flat.ravel(), contrib.imag.ravel(), minlength=total)
        spec = np.conj(sfft.ifftn(np.conj(g.reshape((self.n,) * self.d))))
        return self._scale_modes(spec[self._mode_index()]).ravel()

    def forward(self, fhat):
        """nfft.py:220-230: deconvolve, zero-pad, ifftn, interpolate."""
        fhat = np.asarray(fhat).astype(np.complex128).reshape((self.M,) * self.d)
        padded = np.zeros((self.n,) * self.d, dtype=np.complex128)
        padded[self._mode_index()] = self._scale_modes(fhat)
        g = sfft.ifftn(padded).ravel()
        out = np.empty(self.N, dtype=np.complex128)
        for lo, hi in self._blocks():
            flat, w = self._tensor(lo, hi)
            out[lo:hi] = (g[flat] * w).sum(axis=1)
        return out


# ----------------------------------------------------------------------------
# Fast summation (fastsum.py)
# ----------------------------------------------------------------------------

def gaussian_derivative(order: int, r: float, sigma: float) -> float:
    """fastsum.py:39-46: d^j/dr^j exp(-(r/sigma)^2) via physicists' Hermite H_j."""
    t = np.float64(r) / sigma
    # numpy's Clenshaw evaluation of H_order, as the reference does (bit-identical c_hat)
    sel = np.zeros(order + 1)
    sel[order] = 1.0
    return (-1.0 / sigma) ** order * np.polynomial.hermite.hermval(t, sel) * np.exp(-t * t)


def blend_coefficients(sigma: float, L: float = BALL_RADIUS, ell: float = TRANSITION_WIDTH,
                       p: int = SMOOTHNESS):
    """fastsum.py:90-114: monomial coefficients of the Hermite blend on [0,1]."""
    size = 2 * p
    A = np.zeros((size, size))
    rhs = np.zeros(size)
    for j in range(p):
        A[j, j] = math.factorial(j)
        rhs[j] = ell ** j * gaussian_derivative(j, L, sigma)
    for j in range(1, p + 1):
        for i in range(j, size):
            A[p + j - 1, i] = math.factorial(i) / math.factorial(i - j)
    cond = np.linalg.cond(A)
    if not np.isfinite(cond) or cond > 1.0 / np.finfo(np.float64).eps:
        raise ArithmeticError("Hermite transition system is singular")
    return np.linalg.solve(A, rhs)


def periodized_radial(r, sigma: float, L: float = BALL_RADIUS, ell: float = TRANSITION_WIDTH,
                      p: int = SMOOTHNESS):
    """fastsum.py:117-135: kappa on [0,L], polynomial blend on (L,L+ell), constant beyond."""
    coef = blend_coefficients(sigma, L, ell, p)
    r = np.abs(np.asarray(r, dtype=np.float64))
    out = np.empty_like(r)
    inner = r <= L
    blend = (r > L) & (r < L + ell)
    out[inner] = np.exp(-((r[inner] / sigma) ** 2))
    out[blend] = np.polyval(coef[::-1], (r[blend] - L) / ell)
    out[~inner & ~blend] = float(np.polyval(coef[::-1], 1.0))
    return out


def kernel_coefficients(sigma: float, M: int, d: int, oversample: int = COEFF_OVERSAMPLE):
    """fastsum.py:138-159: real centred M^d block of the periodized kernel's Fourier series."""
    n = M * oversample
    axis = np.arange(-n // 2, n // 2) / n
    grids = np.meshgrid(*([axis] * d), indexing="ij")
    r = np.sqrt(sum(g * g for g in grids))
    samples = periodized_radial(r, sigma)
    spec = sfft.fftshift(sfft.fftn(sfft.ifftshift(samples)) / n ** d)
    lo = n // 2 - M // 2
    return np.ascontiguousarray(spec[(slice(lo, lo + M),) * d].real)


def window_scaling(X, Z=None, L: float = BALL_RADIUS):
    """fastsum.py:210-217: bbox over sources (and targets) -> (center, scale)."""
    pts = X if Z is None else np.vstack([X, Z])
    lo = pts.min(axis=0)
    hi = pts.max(axis=0)
    diameter = float(np.linalg.norm(hi - lo))
    scale = L / diameter if diameter > 0 else 1.0
    return (lo + hi) / 2.0, scale


def fastsum_apply(X, alpha, sigma: float, M: int, m: int, oversampling: float = 2.0, Z=None):
    """fastsum.py:189-256: Re(forward_Z(c_hat * adjoint_X(alpha)))."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    Zm = None if Z is None else np.atleast_2d(np.asarray(Z, dtype=np.float64))
    center, scale = window_scaling(X, Zm)
    d = X.shape[1]
    coeffs = kernel_coefficients(sigma * scale, M, d)
    src = NodeGeometry((X - center) * scale, M, m, oversampling)
    tgt = src if Zm is None else NodeGeometry((Zm - center) * scale, M, m, oversampling)
    shat = coeffs.ravel() * src.adjoint(np.asarray(alpha, dtype=np.float64))
    return tgt.forward(shat).real


def anova_apply(X, windows, alpha, sigma: float, M: int, m: int, oversampling: float = 2.0,
                Z=None, weights=None):
    """anova.py:175-183: out = sum_l eta_l * fastsum_l(alpha), fixed window order, eta = 1/P."""
    X = np.asarray(X, dtype=np.float64)
    P = len(windows)
    if weights is None:
        weights = [1.0 / P] * P
    n_out = X.shape[0] if Z is None else np.asarray(Z).shape[0]
    out = np.zeros(n_out)
    for eta, w in zip(weights, windows):
        cols = list(w)
        out += eta * fastsum_apply(X[:, cols], alpha, sigma, M, m, oversampling,
                                   None if Z is None else np.asarray(Z)[:, cols])
    return out


def cg_solve(apply_A, b, tol: float = 1e-3, maxiter: int = 1000):
    """krr.py:76-110: plain CG from x0=0; returns (x, iterations, residual, converged)."""
    b = np.asarray(b, dtype=np.float64)
    bnorm = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    if bnorm == 0.0:
        return x, 0, 0.0, True
    r = b.copy()
    p = r.copy()
    rs = float(r @ r)
    for it in range(1, maxiter + 1):
        Ap = np.asarray(apply_A(p), dtype=np.float64)
        if not np.all(np.isfinite(Ap)):
            raise ArithmeticError(f"non-finite operator output at iteration {it}")
        pAp = float(p @ Ap)
        if not math.isfinite(pAp) or pAp <= 0.0:
            raise ArithmeticError(f"non-positive curvature at iteration {it}")
        step = rs / pAp
        x += step * p
        r -= step * Ap
        rs_new = float(r @ r)
        if not math.isfinite(rs_new):
            raise ArithmeticError(f"non-finite residual at iteration {it}")
        if math.sqrt(rs_new) <= tol * bnorm:
            return x, it, math.sqrt(rs_new) / bnorm, True
        p = r + (rs_new / rs) * p
        rs = rs_new
    return x, maxiter, math.sqrt(rs) / bnorm, False


# ----------------------------------------------------------------------------
# Direct (quadratic) oracles, used only as independent checks
# ----------------------------------------------------------------------------

def ndft_forward(M_list, coords, fhat):
    """nfft.py:263-281 restated: sum_k fhat_k exp(2 pi i <k,x>)."""
    coords = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    axes = [np.arange(-M // 2, M // 2) for M in M_list]
    modes = np.stack([g.ravel() for g in np.meshgrid(*axes, indexing="ij")], axis=1)
    return np.exp(2j * np.pi * coords @ modes.T) @ np.asarray(fhat, dtype=np.complex128)


def ndft_adjoint(M_list, coords, c):
    """nfft.py:284-300 restated: sum_j c_j exp(-2 pi i <k,x_j>)."""
    coords = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    axes = [np.arange(-M // 2, M // 2) for M in M_list]
    modes = np.stack([g.ravel() for g in np.meshgrid(*axes, indexing="ij")], axis=1)
    return np.exp(-2j * np.pi * coords @ modes.T).T @ np.asarray(c, dtype=np.complex128)


def dense_gaussian(X, Z, alpha, sigma):
    """fastsum.py:162-179 restated: exact sum_j alpha_j exp(-|z-x_j|^2/sigma^2)."""
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    Z = np.atleast_2d(np.asarray(Z, dtype=np.float64))
    d2 = ((Z[:, None, :] - X[None, :, :]) ** 2).sum(axis=2)
    return np.exp(-d2 / sigma ** 2) @ np.asarray(alpha, dtype=np.float64)
