"""GPU NFFT primitives with the reference's ``NfftPlan`` API (nfft.py:139-250).

``forward(f_hat)`` evaluates sum_k f_hat[k] exp(2 pi i <k, x_j>) at the plan's
nodes and ``adjoint(c)`` aggregates sum_j c_j exp(-2 pi i <k, x_j>) onto I_M,
both through the same native stages as the fast summation:

* adjoint: the real and imaginary parts of c are spread as two right-hand
  sides; the forward half of the spectral stage (afs_spectral_forward, with
  the multiplier set to the deconvolution 1/(phi_hat n^d)) returns each part's
  pruned half spectrum; the M^d block is completed on the host by Hermitian
  symmetry, F(-k) = conj F(k) for a real grid.
* forward: f_hat * deconvolution is folded into two Hermitian half spectra
  (real and imaginary part of the grid, Re ifftn(P) and Re ifftn(-iP));
  afs_spectral_inverse turns them into two real grids, and the gather
  evaluates both at the nodes.

Only the O(M^d) spectrum folding runs on the host; spread, transforms and
gather run on the GPU.  The native plan has one grid size for all axes.  Unequal
bandwidths (nfft.py:72-99, 139-177 allow them) are embedded in the largest one:
the trigonometric sums are the same with the missing coefficients set to zero
(forward) or dropped (adjoint), so the result approximates the same exact NDFT
to the profile's accuracy -- it is not the reference's unequal-grid transform
bit for bit (its window shape b_t = pi (2 - M_t / n_t) differs per axis).
"""

from __future__ import annotations

import numpy as np

from .errors import ShapeError, ValidationError
from .operators import _Plan, _torch
from .params import GridSpec, PeriodizationConfig, resolve_profile
from .spectrum import kb_fourier


def validate_nodes(coords, dims=None):
    """Node coordinates in the half-open torus box [-1/2, 1/2) (nfft.py:102-115)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    if coords.ndim == 1:
        coords = coords[:, None]
    if coords.ndim != 2 or coords.shape[0] == 0:
        raise ShapeError("nodes must form a nonempty (N, d) matrix")
    if dims is not None and coords.shape[1] != dims:
        raise ShapeError(f"nodes have {coords.shape[1]} columns, grid has {dims}")
    if not np.all(np.isfinite(coords)):
        raise ValidationError("node coordinates must be finite")
    if coords.min() < -0.5 or coords.max() >= 0.5:
        raise ValidationError("node coordinates must lie in [-1/2, 1/2)")
    return coords


class NfftPlan:
    """NFFT plan for fixed nodes and bandwidths (nfft.py:139-177), evaluated on the GPU."""

    def __init__(self, grid, nodes, profile="default", *, device=None, window_eval="poly"):
        if not isinstance(grid, GridSpec):
            grid = GridSpec(tuple(grid))
        profile = resolve_profile(profile)
        coords = validate_nodes(nodes, grid.dims)
        M = max(grid.bandwidths)   # unequal bandwidths: embedded in the largest (module docstring)
        self._embed = None if all(b == M for b in grid.bandwidths) else tuple(
            slice(M // 2 - b // 2, M // 2 + b // 2) for b in grid.bandwidths)
        self.grid = grid
        self.profile = profile
        self.node_count = coords.shape[0]
        d = grid.dims
        m = profile.cutoff
        n = profile.grid_size(M)
        self._d, self._M, self._n, self._m = d, M, n, m
        b = np.pi * (2.0 - M / n)                                    # nfft.py:156
        # deconvolution 1/phi_hat on the pruned frequencies -M/2..M/2 (nfft.py:158-162)
        f = np.arange(-M // 2, M // 2 + 1)
        self._deconv = 1.0 / kb_fourier(f, n, m, b)
        H = M // 2 + 1
        dec_last = self._deconv[M // 2:]                             # k = 0..M/2
        E = dec_last / float(n) ** d
        for _ in range(d - 1):
            E = self._deconv[:, None] * E.reshape(1, -1)
        E = np.ascontiguousarray(E.reshape((M + 1,) * (d - 1) + (H,)), dtype=np.float64)
        self._plan = _Plan(coords, None, [tuple(range(d))], [1.0], None,
                           PeriodizationConfig(coeff_grid=M), profile, device, 2, window_eval,
                           scaling=[(np.zeros(d), 1.0)], multipliers=[E])
        self._spec = None

    # ---------------------------------------------------------------- helpers
    def _spectra(self):
        torch = _torch()
        if self._spec is None:
            per = self._plan.spectrum_doubles_per_rhs()
            self._spec = torch.zeros(2 * per, dtype=torch.float64, device=self._plan.device)
            self._plan.bind_spectra(self._spec)
        return self._spec

    def _half_shape(self):
        return (self._M + 1,) * (self._d - 1) + (self._M // 2 + 1,)

    def _freqs(self, shape, offsets):
        return np.meshgrid(*[np.arange(s) - o for s, o in zip(shape, offsets)], indexing="ij")

    def _check_coeffs(self, f_hat):
        f_hat = np.asarray(f_hat)
        if f_hat.shape == tuple(self.grid.bandwidths):
            f_hat = f_hat.ravel()
        if f_hat.ndim != 1 or f_hat.shape[0] != self.grid.n_modes:
            raise ShapeError(f"coefficient vector must have length {self.grid.n_modes}, "
                             f"got shape {f_hat.shape}")
        return f_hat.astype(np.complex128, copy=False)

    # ---------------------------------------------------------------- transforms
    def adjoint(self, c):
        """sum_j c_j exp(-2 pi i <k, x_j>) for k in I_M, centered order, flattened."""
        torch = _torch()
        c = np.asarray(c)
        if c.ndim != 1 or c.shape[0] != self.node_count:
            raise ShapeError(f"node vector must have length {self.node_count}, got shape {c.shape}")
        c = c.astype(np.complex128, copy=False)
        d, M = self._d, self._M
        spec = self._spectra()
        a = torch.from_numpy(np.stack([c.real, c.imag])).to(self._plan.device)
        self._plan.spread_device(a, 2)
        self._plan.spectral_forward_device(2)
        S = spec.cpu().numpy().view(np.complex128).reshape((2,) + self._half_shape())
        # complete I_M from the half spectrum of each real grid: F(-k) = conj F(k)
        fr = self._freqs((M,) * d, (M // 2,) * d)
        pos = fr[-1] >= 0
        idx_p = tuple(f + M // 2 for f in fr[:-1]) + (np.where(pos, fr[-1], 0),)
        idx_n = tuple(-f + M // 2 for f in fr[:-1]) + (np.where(pos, 0, -fr[-1]),)
        out = []
        for part in (S[0], S[1]):
            out.append(np.where(pos, part[idx_p], np.conj(part[idx_n])))
        full = out[0] + 1j * out[1]
        if self._embed is not None:   # keep I_{M_1} x ... x I_{M_d} of the embedding grid
            full = full[self._embed]
        return full.ravel()

    def forward(self, f_hat):
        """sum_k f_hat[k] exp(2 pi i <k, x_j>) at the plan's nodes."""
        torch = _torch()
        f_hat = self._check_coeffs(f_hat)
        d, M, n = self._d, self._M, self._n
        # deconvolve on I_M, pad to the pruned frequencies -M/2..M/2 (the +M/2 row is zero)
        if self._embed is None:
            fh = f_hat.reshape((M,) * d)
        else:                          # zero coefficients outside I_{M_1} x ... x I_{M_d}
            fh = np.zeros((M,) * d, dtype=np.complex128)
            fh[self._embed] = f_hat.reshape(self.grid.bandwidths)
        for t in range(d):
            fh = fh * self._deconv[:M].reshape((-1,) + (1,) * (d - 1 - t))
        P = np.zeros((M + 1,) * d, dtype=np.complex128)
        P[(slice(0, M),) * d] = fh                                   # index f + M/2
        half = self._half_shape()
        fr = self._freqs(half, (M // 2,) * (d - 1) + (0,))
        idx = tuple(f + M // 2 for f in fr)
        idx_neg = tuple(-f + M // 2 for f in fr)
        pos = fr[-1] > 0
        scale = 1.0 / float(n) ** d
        S = np.empty((2,) + half, dtype=np.complex128)
        for r, Q in enumerate((P, -1j * P)):   # Re ifftn(P), Im ifftn(P) = Re ifftn(-iP)
            S[r] = (Q[idx] + np.where(pos, np.conj(Q[idx_neg]), 0.0)) * scale
        spec = self._spectra()
        spec.copy_(torch.from_numpy(S.view(np.float64).ravel()))
        self._plan.spectral_inverse_device(2)
        out = torch.empty((2, self.node_count), dtype=torch.float64, device=self._plan.device)
        self._plan.gather_device(out, 2)
        o = out.cpu().numpy()
        return o[0] + 1j * o[1]

    def close(self):
        self._plan.close()


def nfft_forward(plan, f_hat):
    """Fast evaluation of sum_k f_hat[k] exp(2*pi*i <k, x_j>) (nfft.py:253-255)."""
    return plan.forward(f_hat)


def nfft_adjoint(plan, c):
    """Fast evaluation of sum_j c_j exp(-2*pi*i <k, x_j>) (nfft.py:258-260)."""
    return plan.adjoint(c)
