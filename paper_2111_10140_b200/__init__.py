"""B200-native ANOVA fast-summation matvec (arXiv 2111.10140 hot path).

Drop-in for the reference's operator API on the hot path:
``FastsumOperator`` / ``AnovaKernelOperator`` ``.apply`` and ``cg_solve``,
running hand-written sm_100a CUDA kernels behind the C ABI in
``include/anovafs.h`` (``libanovafs.so``); plus the KRR wrappers that call it
(``fit`` / ``decision_values`` / ``predict`` / model IO).
"""

__version__ = "0.1.0"

from .errors import DeviceError, NumericalError, ShapeError, ValidationError
from .params import (PROFILES, AccuracyProfile, GaussianKernel, GridSpec, PeriodizationConfig,
                     resolve_profile)
from .spectrum import regularize_kernel
from .operators import (AnovaKernelOperator, FastsumOperator, FreeWindowSet, WindowSet,
                        anova_apply, anova_build, fastsum_apply, fastsum_build)
from .krr import (CgResult, KernelSystem, KrrConfig, KrrModel, cg_solve, decision_values, fit,
                  load_model, model_from_dict, model_to_dict, predict, save_model)
from .prep import MisReport, ScalerStats, build_windows, mis_scores, zscore_apply, zscore_fit
from .nfft import NfftPlan, nfft_adjoint, nfft_forward, validate_nodes
from .harness import bench_mvm, direct_sum, ndft_adjoint_direct, ndft_direct
from .distributed import PointSharded, WindowSharded, sharded_cg

__all__ = [
    "AccuracyProfile", "AnovaKernelOperator", "bench_mvm", "direct_sum", "ndft_adjoint_direct", "ndft_direct", "CgResult", "DeviceError", "FastsumOperator",
    "FreeWindowSet", "GaussianKernel", "GridSpec", "KernelSystem", "KrrConfig", "KrrModel",
    "MisReport", "NfftPlan", "NumericalError", "PROFILES", "PeriodizationConfig", "PointSharded", "ScalerStats", "ShapeError",
    "ValidationError", "WindowSet", "anova_apply", "anova_build", "build_windows", "cg_solve",
    "decision_values", "fastsum_apply", "fastsum_build", "fit", "load_model", "mis_scores",
    "model_from_dict", "model_to_dict", "nfft_adjoint", "nfft_forward", "predict", "regularize_kernel", "resolve_profile",
    "save_model", "validate_nodes", "WindowSharded", "sharded_cg", "zscore_apply", "zscore_fit",
]
