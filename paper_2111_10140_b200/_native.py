"""ctypes binding of the native library ``libanovafs.so`` (include/anovafs.h).

There is no fallback: if the library is missing or no CUDA device is present,
every operator constructor raises.  Build with ``python -m
paper_2111_10140_b200.build`` (``__graft_entry__.build()`` does it too).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import STATUS_EXCEPTIONS, DeviceError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libanovafs.so")
# tuning hook: AFS_LIB selects an in-tree variant build (tools/build_variant.sh)
if os.environ.get("AFS_LIB"):
    LIB_PATH = os.path.abspath(os.environ["AFS_LIB"])

AFS_OK, AFS_ERR_SHAPE, AFS_ERR_VALIDATION, AFS_ERR_NUMERICAL, AFS_ERR_CUDA, AFS_ERR_NOMEM = range(6)

c_double_p = ctypes.POINTER(ctypes.c_double)
ABI_VERSION = 3
CG_WORKSPACE_DOUBLES = 640   # AFS_CG_WORKSPACE_DOUBLES


class WindowDesc(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int32),
        ("features", ctypes.c_int32 * 3),
        ("center", ctypes.c_double * 3),
        ("scale", ctypes.c_double),
        ("weight", ctypes.c_double),
        ("multiplier", c_double_p),
    ]


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("n_windows", ctypes.c_int32),
        ("windows", ctypes.POINTER(WindowDesc)),
        ("d_total", ctypes.c_int32),
        ("n_sources", ctypes.c_int64),
        ("sources", ctypes.c_void_p),
        ("n_targets", ctypes.c_int64),
        ("targets", ctypes.c_void_p),
        ("bandwidth", ctypes.c_int32),
        ("cutoff", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("max_rhs", ctypes.c_int32),
        ("window_eval", ctypes.c_int32),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("device_bytes", ctypes.c_int64),
        ("n_windows", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("n_sources", ctypes.c_int64),
        ("n_targets", ctypes.c_int64),
        ("kernel_launches_per_apply", ctypes.c_int32),
        ("tensor_core_windows", ctypes.c_int32),
    ]


# every symbol include/anovafs.h declares, with its ctypes signature
SIGNATURES = {
    "afs_abi_version": (ctypes.c_int, []),
    "afs_last_error": (ctypes.c_char_p, []),
    "afs_plan_create": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "afs_plan_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "afs_plan_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PlanInfo)]),
    "afs_apply": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]),
    "afs_spread": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                  ctypes.c_void_p]),
    "afs_spectral": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "afs_gather": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                  ctypes.c_void_p]),
    "afs_plan_grids": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(ctypes.c_int64)]),
    "afs_plan_bind_grids": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]),
    "afs_spectral_forward": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "afs_spectral_inverse": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "afs_plan_spectra": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_int64)]),
    "afs_plan_bind_spectra": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]),
    "afs_plan_set_profiling": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "afs_plan_set_deterministic": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "afs_plan_stage_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                            ctypes.c_int32]),
    "afs_plan_window_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_double), ctypes.c_int32]),
    "afs_cg_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p]),
    "afs_cg_vec_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "afs_cg_vec_ap": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_void_p]),
    "afs_cg_vec_update": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "afs_cg_vec_direction": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_void_p, ctypes.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and return the native library; raises loudly if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"native library {path} is missing; build it with "
                "`python -m paper_2111_10140_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.afs_abi_version() != ABI_VERSION:
            raise ImportError("libanovafs ABI version mismatch")
        _lib = lib
        return lib


def check(status: int):
    """Map a C-ABI status onto the reference's exception classes."""
    if status == AFS_OK:
        return
    msg = (_lib.afs_last_error() or b"").decode("utf-8", "replace") if _lib else ""
    exc = STATUS_EXCEPTIONS.get(status)
    if exc is not None:
        raise exc(msg)
    raise DeviceError(msg or f"anovafs status {status}")
