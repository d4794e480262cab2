"""Parameter types of the fast-summation path, with the reference's names,
defaults and validation errors.

- ``AccuracyProfile`` / ``PROFILES`` / ``resolve_profile``: nfft.py:31-69
- ``GridSpec``: nfft.py:72-99
- ``GaussianKernel``: fastsum.py:25-49
- ``PeriodizationConfig``: fastsum.py:52-87
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class AccuracyProfile:
    """NFFT accuracy parameters: oversampling sigma_os > 1 and window cutoff m >= 1."""

    name: str
    oversampling: float
    cutoff: int

    def __post_init__(self):
        if self.oversampling <= 1.0:
            raise ValidationError("oversampling factor must exceed 1")
        if self.cutoff < 1:
            raise ValidationError("window cutoff must be at least 1")

    def grid_size(self, M: int) -> int:
        """Oversampled FFT length n = max(2m, even(ceil(sigma_os*M))) (nfft.py:151-153)."""
        n = int(np.ceil(self.oversampling * M))
        n += n % 2
        return max(n, 2 * self.cutoff)


PROFILES = {
    "rough": AccuracyProfile("rough", 1.5, 3),
    "default": AccuracyProfile("default", 2.0, 4),
    "fine": AccuracyProfile("fine", 2.0, 6),
}


def resolve_profile(profile) -> AccuracyProfile:
    if isinstance(profile, AccuracyProfile):
        return profile
    try:
        return PROFILES[profile]
    except (KeyError, TypeError):
        raise ValidationError(
            f"unknown profile {profile!r}; expected one of {sorted(PROFILES)}") from None


@dataclass(frozen=True)
class GridSpec:
    """Frequency grid: per-dimension even bandwidths M = (M_1, ..., M_d), d <= 3."""

    bandwidths: tuple

    def __post_init__(self):
        bw = tuple(int(b) for b in self.bandwidths)
        object.__setattr__(self, "bandwidths", bw)
        if not 1 <= len(bw) <= 3:
            raise ValidationError(f"grid dimension must be 1..3, got {len(bw)}")
        for b in bw:
            if b < 2 or b % 2 != 0:
                raise ValidationError(f"bandwidths must be even and >= 2, got {b}")

    @property
    def dims(self):
        return len(self.bandwidths)

    @property
    def n_modes(self):
        return int(np.prod(self.bandwidths))


@dataclass(frozen=True)
class GaussianKernel:
    """Radial Gaussian kernel kappa(r) = exp(-r^2 / sigma^2)."""

    sigma: float

    def __post_init__(self):
        if not (self.sigma > 0 and math.isfinite(self.sigma)):
            raise ValidationError(f"kernel shape parameter must be positive, got {self.sigma}")

    def __call__(self, r):
        r = np.asarray(r, dtype=np.float64)
        return np.exp(-((r / self.sigma) ** 2))

    def derivative(self, order: int, r):
        """order-th radial derivative via Rodrigues' formula with physicists' Hermite H_j."""
        t = np.asarray(r, dtype=np.float64) / self.sigma
        sel = np.zeros(order + 1)
        sel[order] = 1.0
        return (-1.0 / self.sigma) ** order * np.polynomial.hermite.hermval(t, sel) * np.exp(-t * t)

    def rescaled(self, factor: float) -> "GaussianKernel":
        return replace(self, sigma=self.sigma * factor)


_COEFF_GRIDS = {"rough": 32, "default": 64, "fine": 128}


@dataclass(frozen=True)
class PeriodizationConfig:
    """Smooth periodic extension of the kernel (period 1): exact on [0, ball_radius],
    Hermite blend of ``smoothness_degree`` derivatives over ``transition_width``,
    Fourier coefficients on a ``coeff_grid``^d grid refined by ``coeff_oversample``."""

    ball_radius: float = 0.25 - 1.0 / 32.0
    transition_width: float = 1.0 / 16.0
    smoothness_degree: int = 7
    coeff_grid: int = 64
    coeff_oversample: int = 2

    def __post_init__(self):
        if not 0.0 < self.ball_radius < 0.5:
            raise ValidationError("ball_radius must lie in (0, 1/2)")
        if self.transition_width <= 0:
            raise ValidationError("transition_width must be positive")
        if self.ball_radius + self.transition_width > 0.5 + 1e-12:
            raise ValidationError("ball_radius + transition_width must not exceed 1/2")
        if self.smoothness_degree < 1:
            raise ValidationError("smoothness_degree must be at least 1")
        if self.coeff_grid < 2 or self.coeff_grid % 2 != 0:
            raise ValidationError("coeff_grid must be even and >= 2")
        if self.coeff_oversample < 1:
            raise ValidationError("coeff_oversample must be at least 1")

    @classmethod
    def for_profile(cls, profile):
        return cls(coeff_grid=_COEFF_GRIDS.get(resolve_profile(profile).name, 64))
