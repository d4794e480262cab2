"""B200-native ANOVA fast-summation matvec (arXiv 2111.10140 hot path).

Drop-in for the reference's operator API on the hot path:
``FastsumOperator`` / ``AnovaKernelOperator`` ``.apply`` and ``cg_solve``,
running hand-written sm_100a CUDA kernels behind the C ABI in
``include/anovafs.h`` (``libanovafs.so``).
"""

__version__ = "0.1.0"

from .errors import DeviceError, NumericalError, ShapeError, ValidationError
from .params import (PROFILES, AccuracyProfile, GaussianKernel, GridSpec, PeriodizationConfig,
                     resolve_profile)
from .spectrum import regularize_kernel
from .operators import (AnovaKernelOperator, FastsumOperator, FreeWindowSet, WindowSet,
                        anova_apply, anova_build, fastsum_apply, fastsum_build)
from .krr import CgResult, KernelSystem, cg_solve

__all__ = [
    "AccuracyProfile", "AnovaKernelOperator", "CgResult", "DeviceError", "FastsumOperator",
    "FreeWindowSet", "GaussianKernel", "GridSpec", "KernelSystem", "NumericalError", "PROFILES",
    "PeriodizationConfig", "ShapeError", "ValidationError", "WindowSet", "anova_apply",
    "anova_build", "cg_solve", "fastsum_apply", "fastsum_build", "regularize_kernel",
    "resolve_profile",
]
