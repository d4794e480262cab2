"""Plan-time spectral tables (host, fp64): kernel Fourier coefficients c_hat
and the per-window real multiplier E handed to the device.

- ``regularize_kernel``: fastsum.py:90-159 (Hermite blend, periodized radial
  profile, (M*oversample)^d FFT, centred M^d block, real part).
- ``kb_fourier``: nfft.py:125-128; the deconvolution factors 1/phi_hat
  (nfft.py:158-162).
- ``window_multiplier``: folds c_hat, both deconvolutions (adjoint nfft.py:250 and
  forward nfft.py:223), the adjoint's 1/n^d (nfft.py:248) and the inverse
  FFT's 1/n^d (nfft.py:226) into one real table, symmetrised
  D_sym(k) = (D(k)+D(-k))/2 so that a real pipeline reproduces the
  reference's ``.real`` (fastsum.py:256) exactly; stored on the pruned
  half-spectrum layout the device stage uses (include/anovafs.h).
"""

from __future__ import annotations

import math

import os

import numpy as np
import scipy.fft as sfft
from scipy.special import i0

from .errors import NumericalError, ValidationError
from .params import GaussianKernel, PeriodizationConfig


_FFT_WORKERS = max(1, min(16, os.cpu_count() or 1))


def _blend_poly(kernel: GaussianKernel, cfg: PeriodizationConfig) -> np.ndarray:
    """Monomial coefficients of q on t in [0,1]: q^(j)(0) = ell^j kappa^(j)(L) (j<p),
    q^(j)(1) = 0 (j=1..p)  (fastsum.py:90-114)."""
    L, ell, p = cfg.ball_radius, cfg.transition_width, cfg.smoothness_degree
    size = 2 * p
    sysm = np.zeros((size, size))
    rhs = np.zeros(size)
    for j in range(p):
        sysm[j, j] = math.factorial(j)
        rhs[j] = ell ** j * kernel.derivative(j, L)
    for j in range(1, p + 1):
        sysm[p + j - 1, j:] = [math.factorial(i) / math.factorial(i - j) for i in range(j, size)]
    cond = np.linalg.cond(sysm)
    if not np.isfinite(cond) or cond > 1.0 / np.finfo(np.float64).eps:
        raise NumericalError(
            f"Hermite transition system is numerically singular at smoothness_degree={p} "
            f"(condition number {cond:.2e})")
    return np.linalg.solve(sysm, rhs)


def periodized_profile(kernel: GaussianKernel, cfg: PeriodizationConfig):
    """r -> kappa_tilde(r) (fastsum.py:117-135)."""
    poly = _blend_poly(kernel, cfg)[::-1]
    L, ell = cfg.ball_radius, cfg.transition_width
    tail = float(np.polyval(poly, 1.0))

    def profile(r):
        r = np.abs(np.asarray(r, dtype=np.float64))
        out = np.full(r.shape, tail)
        core = r <= L
        mid = (r > L) & (r < L + ell)
        out[core] = kernel(r[core])
        out[mid] = np.polyval(poly, (r[mid] - L) / ell)
        return out

    return profile


def regularize_kernel(kernel: GaussianKernel, config: PeriodizationConfig, dims: int,
                      fft: str = "host") -> np.ndarray:
    """Real (coeff_grid,)*dims Fourier coefficients of the periodized kernel, centred order.

    ``fft="host"`` (default) runs the (M*oversample)^d transform with scipy's pocketfft, as the
    reference does, so c_hat is bit-identical to it.  ``fft="device"`` runs it with cuFFT on
    the current CUDA device (the samples are still built on the host, exactly): the 256^3
    transform of C4 drops from ~1 s to milliseconds, and c_hat moves by ~1e-16 relative,
    roundoff-level like the matvec itself (it can move a loose-tolerance CG's iteration count
    within the reference's own roundoff spread)."""
    if fft not in ("host", "device"):
        raise ValidationError(f"fft must be 'host' or 'device', got {fft!r}")
    if not 1 <= dims <= 3:
        raise ValidationError(f"dimension must be 1..3, got {dims}")
    M = config.coeff_grid
    nn = M * config.coeff_oversample
    prof = periodized_profile(kernel, config)
    if nn & (nn - 1) == 0:
        # nn a power of two: (i/nn)^2 and their sums are exact, so r depends only on the
        # integer s = sum_t i_t^2 -- evaluate the profile once per distinct s (<= d nn^2/4 + 1
        # values instead of nn^d) and build the ifftshift-ed samples by lookup
        i = sfft.ifftshift(np.arange(-nn // 2, nn // 2, dtype=np.int64))
        sq = i * i
        s2 = np.zeros((1,) * dims, dtype=np.int64)
        for t in range(dims):
            shape = [1] * dims
            shape[t] = nn
            s2 = s2 + sq.reshape(shape)
        table = prof(np.sqrt(np.arange(dims * (nn // 2) ** 2 + 1) / float(nn * nn)))
        shifted = table[s2]
    else:
        ax = np.arange(-nn // 2, nn // 2) / nn
        r2 = np.zeros((nn,) * dims)
        for t in range(dims):
            shape = [1] * dims
            shape[t] = nn
            r2 = r2 + (ax * ax).reshape(shape)
        shifted = sfft.ifftshift(prof(np.sqrt(r2)))
    # the centred M^d block of fftshift(spec) / nn^d, taken before shifting: frequencies
    # -M/2 .. M/2-1 sit at indices k mod nn (elementwise the same division as the reference)
    k = np.arange(-M // 2, M // 2) % nn
    if fft == "device":
        import torch

        if not torch.cuda.is_available():
            raise ValidationError("fft='device' needs a CUDA device")
        dev = torch.device("cuda", torch.cuda.current_device())
        spec_d = torch.fft.fftn(torch.from_numpy(np.ascontiguousarray(shifted)).to(dev))
        kd = torch.from_numpy(k).to(dev)
        for t in range(dims):
            spec_d = spec_d.index_select(t, kd)
        block = (spec_d / nn ** dims).real.cpu().numpy()
        return np.ascontiguousarray(block)
    # scipy.fft (pocketfft) as the reference (fastsum.py:154-155); threads over the
    # untransformed axes do not change any 1-D transform, so the result is bit-identical
    spec = sfft.fftn(shifted, workers=_FFT_WORKERS)
    block = spec[np.ix_(*([k] * dims))] / nn ** dims
    return np.ascontiguousarray(block.real)


def kb_fourier(k, n: int, m: int, b: float):
    """Continuous Fourier transform of the Kaiser-Bessel window at integer k."""
    k = np.asarray(k, dtype=np.float64)
    return i0(m * np.sqrt(np.maximum(b * b - (2.0 * np.pi * k / n) ** 2, 0.0))) / n


def window_multiplier(coeffs: np.ndarray, M: int, n: int, m: int) -> np.ndarray:
    """Pruned real multiplier E for one window (layout: include/anovafs.h)."""
    d = coeffs.ndim
    b = np.pi * (2.0 - M / n)
    deconv = 1.0 / kb_fourier(np.arange(-M // 2, M // 2), n, m, b)
    D = np.asarray(coeffs, dtype=np.float64).copy()
    for t in range(d):
        shape = [1] * d
        shape[t] = M
        D = D * (deconv * deconv).reshape(shape)
    D = D / float(n) ** d                    # adjoint fftn/n^d
    full = np.zeros((M + 1,) * d)            # index j = k + M/2, k in -M/2..M/2
    full[(slice(0, M),) * d] = D             # D(+M/2) = 0 (asymmetric I_M)
    sym = 0.5 * (full + full[(slice(None, None, -1),) * d])
    sym = sym / float(n) ** d                # unnormalised inverse DFT
    half = sym[(Ellipsis, slice(M // 2, M + 1))].copy()   # last axis k in 0..M/2
    half[..., 1:] *= 2.0                     # Hermitian pairs of the real last axis
    return np.ascontiguousarray(half)
