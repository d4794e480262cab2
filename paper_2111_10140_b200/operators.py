"""GPU operators with the reference's API: ``FastsumOperator`` (fastsum.py:182-256)
and ``AnovaKernelOperator`` (anova.py:138-183), plus ``WindowSet`` (anova.py:91-121).

Host work here is plan construction only (bbox scaling, c_hat, multiplier
tables); every matvec runs through the native library (``_native``) on the
GPU.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native
from .errors import ShapeError, ValidationError
from .params import GaussianKernel, PeriodizationConfig, resolve_profile
from .spectrum import regularize_kernel, window_multiplier

WINDOW_SIZE = 3


def _torch():
    import torch  # plumbing: device memory, streams, pinned host buffers

    if not torch.cuda.is_available():
        raise _native.DeviceError("no CUDA device: the anovafs operators run only on the GPU")
    return torch


class WindowSet:
    """Disjoint feature windows, all of size 3 except possibly the last; eta_l = 1/P."""

    def __init__(self, windows):
        windows = tuple(tuple(int(i) for i in w) for w in windows)
        if not windows:
            raise ValidationError("window set must not be empty")
        seen = set()
        for w in windows:
            if not 1 <= len(w) <= WINDOW_SIZE:
                raise ValidationError(f"window size must be 1..{WINDOW_SIZE}, got {len(w)}")
            if seen.intersection(w):
                raise ValidationError("windows must be pairwise disjoint")
            seen.update(w)
        for w in windows[:-1]:
            if len(w) != WINDOW_SIZE:
                raise ValidationError("only the last window may hold fewer than 3 features")
        self.windows = windows
        self.weights = tuple([1.0 / len(windows)] * len(windows))

    def __len__(self):
        return len(self.windows)

    def __iter__(self):
        return iter(self.windows)

    def retained_features(self):
        return sorted(i for w in self.windows for i in w)

    def to_dict(self):
        return {"windows": [list(w) for w in self.windows], "weights": list(self.weights)}


class FreeWindowSet:
    """Arbitrary (possibly overlapping) windows of 1..3 features with explicit weights.

    The reference's ``WindowSet`` rejects the C3/C5 window lists; the SURVEY
    oracle recipe for them composes FastsumOperators with eta = 1/P
    (SURVEY.md §8(c)).  This type carries that recipe through one plan.
    """

    def __init__(self, windows, weights=None):
        windows = tuple(tuple(int(i) for i in w) for w in windows)
        if not windows:
            raise ValidationError("window set must not be empty")
        for w in windows:
            if not 1 <= len(w) <= WINDOW_SIZE:
                raise ValidationError(f"window size must be 1..{WINDOW_SIZE}, got {len(w)}")
            if len(set(w)) != len(w):
                raise ValidationError(f"window {w} repeats a feature")
        if weights is None:
            weights = [1.0 / len(windows)] * len(windows)
        if len(weights) != len(windows):
            raise ShapeError("one weight per window is required")
        self.windows = windows
        self.weights = tuple(float(x) for x in weights)

    def __len__(self):
        return len(self.windows)

    def __iter__(self):
        return iter(self.windows)


class WindowOperator:
    """One window's term K_l of an ANOVA operator, as the reference's ``operators[l]``
    (anova.py:163-172): the FastsumOperator attributes (fastsum.py:219-232) are the plan's
    own; ``apply`` / ``apply_complex`` / ``source_plan`` / ``target_plan`` build a GPU
    ``FastsumOperator`` on the window's columns at first use (the ANOVA apply itself never
    needs it: all windows run in one plan)."""

    def __init__(self, features, kernel, config, profile, center, scale, coeffs, n_sources,
                 n_targets, nodes=None, device=None, window_eval="poly"):
        self.features = tuple(features)
        self.kernel = kernel
        self.config = config
        self.profile = profile
        self.dims = len(features)
        self.center = center
        self.scale = scale
        self.scaled_kernel = kernel.rescaled(scale)
        self.coeffs = coeffs
        self.n_sources = n_sources
        self.n_targets = n_targets
        self._nodes = nodes              # (X, Z) of the whole operator, or None
        self._device = device
        self._window_eval = window_eval
        self._op = None

    def _fastsum(self):
        if self._op is None:
            if self._nodes is None:
                raise ValidationError("this window view has no nodes to build an operator on")
            X, Z = self._nodes
            cols = list(self.features)
            self._op = FastsumOperator(self.kernel, self.config, X[:, cols],
                                       None if Z is None else Z[:, cols], self.profile,
                                       device=self._device, window_eval=self._window_eval)
        return self._op

    def apply(self, alpha):
        return self._fastsum().apply(alpha)

    def apply_complex(self, alpha):
        return self._fastsum().apply_complex(alpha)

    @property
    def source_plan(self):
        return self._fastsum().source_plan

    @property
    def target_plan(self):
        return self._fastsum().target_plan


def bbox_scaling(lo, hi, config):
    """(center, scale) from per-column min/max (fastsum.py:210-217, same arithmetic)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    diameter = float(np.linalg.norm(hi - lo))                       # fastsum.py:213
    scale = config.ball_radius / diameter if diameter > 0 else 1.0  # fastsum.py:216
    center = (lo + hi) / 2.0                                        # fastsum.py:217
    return center, scale


def _chunks(n, size=1 << 20):
    """[lo, hi) ranges of ~8 MB (fp64) for pipelined host<->device copies."""
    return [(lo, min(n, lo + size)) for lo in range(0, n, size)]


def _columns_minmax(A, cols):
    """(mins, maxs) of the selected columns, computed where A lives."""
    if isinstance(A, np.ndarray):
        sub = A[:, list(cols)]
        return sub.min(axis=0), sub.max(axis=0)
    sub = A[:, list(cols)]
    return sub.amin(dim=0).cpu().numpy(), sub.amax(dim=0).cpu().numpy()


def _all_columns_minmax(A):
    """Per-column (mins, maxs) of the whole matrix in one pass; a window's bbox is the
    subset of its columns (min/max are exact, so this equals fastsum.py:210-212 on X[:, w])."""
    if isinstance(A, np.ndarray):
        return A.min(axis=0), A.max(axis=0)
    lo, hi = A.aminmax(dim=0)
    return lo.cpu().numpy(), hi.cpu().numpy()


def _as_matrix(A, name):
    if isinstance(A, np.ndarray) or not hasattr(A, "is_cuda"):
        A = np.asarray(A, dtype=np.float64)
        if A.ndim == 1:
            A = A[:, None]
        if A.ndim != 2 or A.shape[0] == 0:
            raise ShapeError(f"{name} must form a nonempty (N, d) matrix")
        if not np.all(np.isfinite(A)):
            raise ValidationError(f"{name} coordinates must be finite")
        return np.ascontiguousarray(A)
    torch = _torch()
    A = A.to(dtype=torch.float64)
    if A.dim() == 1:
        A = A[:, None]
    if A.dim() != 2 or A.shape[0] == 0:
        raise ShapeError(f"{name} must form a nonempty (N, d) matrix")
    if not bool(torch.isfinite(A).all()):
        raise ValidationError(f"{name} coordinates must be finite")
    return A.contiguous()


class _Plan:
    """Owns one native plan (afs_plan*) and its staging buffers."""

    def __init__(self, X, Z, feats, weights, kernel, config, profile, device, max_rhs,
                 window_eval="poly", scaling=None, multipliers=None, coeff_fft="host"):
        torch = _torch()
        self.lib = _native.load()
        self.device = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        self.profile = profile
        self.config = config
        M = config.coeff_grid
        m = profile.cutoff
        n = profile.grid_size(M)
        self.M, self.m, self.n = M, m, n
        self.N = X.shape[0]
        self.Nt = X.shape[0] if Z is None else Z.shape[0]
        self.d_total = X.shape[1]
        self.max_rhs = int(max_rhs)
        self.windows = []
        descs = (_native.WindowDesc * len(feats))()
        self.n_windows = len(feats)
        self._keep = []
        # upload first: the bbox reductions run on the device copy (exact, like numpy's)
        Xd = X if not isinstance(X, np.ndarray) else torch.from_numpy(X)
        Xd = Xd.to(self.device, non_blocking=False).contiguous()
        Zd = None
        if Z is not None:
            Zd = (Z if not isinstance(Z, np.ndarray) else torch.from_numpy(Z)).to(self.device).contiguous()
        if scaling is None:
            xlo, xhi = _all_columns_minmax(Xd)
            if Z is not None:
                zlo, zhi = _all_columns_minmax(Zd)
        for l, (w, eta) in enumerate(zip(feats, weights)):
            if scaling is not None:
                # externally fixed (e.g. bbox all-reduced over point shards)
                center, scale = np.asarray(scaling[l][0], dtype=np.float64), float(scaling[l][1])
            else:
                cols = list(w)
                lo, hi = xlo[cols], xhi[cols]
                if Z is not None:
                    lo, hi = np.minimum(lo, zlo[cols]), np.maximum(hi, zhi[cols])
                center, scale = bbox_scaling(lo, hi, config)
            if multipliers is not None:
                # caller-supplied spectral multiplier (e.g. the bare NFFT: deconvolution only)
                coeffs = None
                mult = np.ascontiguousarray(multipliers[l], dtype=np.float64)
            else:
                with torch.cuda.device(self.device):
                    coeffs = regularize_kernel(kernel.rescaled(scale), config, len(w), coeff_fft)
                mult = window_multiplier(coeffs, M, n, m)
                self.windows.append(WindowOperator(w, kernel, config, profile, center, scale,
                                                   coeffs, self.N, self.Nt, nodes=(X, Z),
                                                   device=self.device.index,
                                                   window_eval=window_eval))
            self._keep.append(mult)
            dsc = descs[l]
            dsc.dims = len(w)
            for t in range(len(w)):
                dsc.features[t] = w[t]
                dsc.center[t] = center[t]
            dsc.scale = scale
            dsc.weight = float(eta)
            dsc.multiplier = mult.ctypes.data_as(_native.c_double_p)
        desc = _native.PlanDesc()
        desc.device = self.device.index
        desc.n_windows = len(feats)
        desc.windows = descs
        desc.d_total = self.d_total
        desc.n_sources = self.N
        desc.sources = Xd.data_ptr()
        desc.n_targets = 0 if Z is None else self.Nt
        desc.targets = None if Zd is None else Zd.data_ptr()
        desc.bandwidth = M
        desc.cutoff = m
        desc.grid = n
        desc.max_rhs = self.max_rhs
        if window_eval not in ("poly", "exact"):
            raise ValidationError("window_eval must be 'poly' or 'exact'")
        desc.window_eval = 0 if window_eval == "poly" else 1
        self.window_eval = window_eval
        handle = ctypes.c_void_p()
        torch.cuda.synchronize(self.device)
        _native.check(self.lib.afs_plan_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        del Xd, Zd
        self._tls = threading.local()   # per-thread staging: applies are reentrant (api.cu)

    def _staging(self, key, make):
        """This thread's host/device staging buffers for `key` (created on first use)."""
        st = getattr(self._tls, "stage", None)
        if st is None:
            st = self._tls.stage = {}
        if key not in st:
            st[key] = make()
        return st[key]

    def info(self):
        inf = _native.PlanInfo()
        _native.check(self.lib.afs_plan_get_info(self.handle, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in _native.PlanInfo._fields_}

    def set_deterministic(self, enable: bool):
        """Bit-reproducible spread (fixed-point grid accumulation; include/anovafs.h)."""
        _native.check(self.lib.afs_plan_set_deterministic(self.handle, 1 if enable else 0))

    def set_profiling(self, enable: bool):
        _native.check(self.lib.afs_plan_set_profiling(self.handle, 1 if enable else 0))

    def stage_times(self, reset: bool = True):
        buf = (ctypes.c_double * 4)()
        _native.check(self.lib.afs_plan_stage_times(self.handle, buf, 1 if reset else 0))
        return {"spread_ms": buf[0], "spectral_ms": buf[1], "gather_ms": buf[2],
                "applies": int(buf[3])}

    def window_times(self, reset: bool = True):
        """Per-window (spread_ms, gather_ms) lists accumulated over profiled applies."""
        P = self.n_windows
        sp = (ctypes.c_double * P)()
        ga = (ctypes.c_double * P)()
        _native.check(self.lib.afs_plan_window_times(self.handle, sp, ga, 1 if reset else 0))
        return list(sp), list(ga)

    def close(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.afs_plan_destroy(h)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device-level entry points -------------------------------------------------
    def apply_device(self, alpha, out, nrhs):
        """alpha: cuda float64 (nrhs, N) contiguous; out: cuda float64 (nrhs, Nt)."""
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(self.lib.afs_apply(self.handle, alpha.data_ptr(), self.N, out.data_ptr(),
                                         self.Nt, int(nrhs), stream))

    # -- stage-level entry points (point-sharded multi-GPU) ---------------------------
    def grid_doubles_per_rhs(self):
        ptr = ctypes.c_void_p()
        n = ctypes.c_int64()
        _native.check(self.lib.afs_plan_grids(self.handle, ctypes.byref(ptr), ctypes.byref(n)))
        return int(n.value)

    def bind_grids(self, buf):
        """Make the plan spread into / read from `buf` (cuda float64, >= per_rhs*max_rhs)."""
        _native.check(self.lib.afs_plan_bind_grids(self.handle, buf.data_ptr(), buf.numel()))
        self._bound_grids = buf   # keep alive

    def spread_device(self, alpha, nrhs):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(self.lib.afs_spread(self.handle, alpha.data_ptr(), self.N, int(nrhs), stream))

    def spectral_device(self, nrhs):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(self.lib.afs_spectral(self.handle, int(nrhs), stream))

    def spectrum_doubles_per_rhs(self):
        ptr = ctypes.c_void_p()
        n = ctypes.c_int64()
        _native.check(self.lib.afs_plan_spectra(self.handle, ctypes.byref(ptr), ctypes.byref(n)))
        return int(n.value)

    def bind_spectra(self, buf):
        """Make the split spectral stage use `buf` (cuda float64, >= per_rhs*max_rhs)."""
        _native.check(self.lib.afs_plan_bind_spectra(self.handle, buf.data_ptr(), buf.numel()))
        self._bound_spectra = buf   # keep alive

    def spectral_forward_device(self, nrhs):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(self.lib.afs_spectral_forward(self.handle, int(nrhs), stream))

    def spectral_inverse_device(self, nrhs):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(self.lib.afs_spectral_inverse(self.handle, int(nrhs), stream))

    def gather_device(self, out, nrhs):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(self.lib.afs_gather(self.handle, out.data_ptr(), self.Nt, int(nrhs), stream))

    def cg_device(self, b, x, beta, tol, maxiter):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        it = ctypes.c_int32()
        res = ctypes.c_double()
        conv = ctypes.c_int32()
        st = self.lib.afs_cg_solve(self.handle, b.data_ptr(), x.data_ptr(), float(beta),
                                   float(tol), int(maxiter), ctypes.byref(it), ctypes.byref(res),
                                   ctypes.byref(conv), stream)
        _native.check(st)
        return int(it.value), float(res.value), bool(conv.value)

    def apply(self, alpha):
        """Reference-facing apply: numpy in -> numpy out (host buffers, copies included);
        torch CUDA tensor in -> torch CUDA tensor out."""
        torch = _torch()
        if hasattr(alpha, "is_cuda") and alpha.is_cuda:
            a = alpha.to(torch.float64)
            one = a.dim() == 1
            if one:
                a = a[None, :]
            elif a.dim() == 2:
                a = a.t()
            if a.shape[1] != self.N:
                raise ShapeError(f"alpha must have length {self.N}, got {tuple(alpha.shape)}")
            R = a.shape[0]
            if R > self.max_rhs:
                raise ShapeError(f"at most {self.max_rhs} right-hand sides per apply")
            a = a.contiguous()
            out = torch.empty((R, self.Nt), dtype=torch.float64, device=self.device)
            self.apply_device(a, out, R)
            return out[0] if one else out.t()
        if torch.is_tensor(alpha):
            return self._apply_host_tensor(alpha)
        arr = np.asarray(alpha, dtype=np.float64)
        one = arr.ndim == 1
        if not (arr.ndim in (1, 2) and arr.shape[0] == self.N):
            raise ShapeError(f"alpha must have length {self.N}, got shape {arr.shape}")
        R = 1 if one else arr.shape[1]
        if R > self.max_rhs:
            raise ShapeError(f"at most {self.max_rhs} right-hand sides per apply")
        h_in, d_in, d_out, h_out = self._staging(R, lambda: (
            torch.empty((R, self.N), dtype=torch.float64, pin_memory=True),
            torch.empty((R, self.N), dtype=torch.float64, device=self.device),
            torch.empty((R, self.Nt), dtype=torch.float64, device=self.device),
            torch.empty((R, self.Nt), dtype=torch.float64, pin_memory=True)))
        stream = torch.cuda.current_stream(self.device)
        src = torch.from_numpy(np.ascontiguousarray(arr.T) if not one else arr)
        src = src[None, :] if one else src
        # chunked host->pinned (multi-threaded torch copy) overlapped with async H2D
        for lo, hi in _chunks(self.N):
            h_in[:, lo:hi].copy_(src[:, lo:hi])
            d_in[:, lo:hi].copy_(h_in[:, lo:hi], non_blocking=True)
        self.apply_device(d_in, d_out, R)
        res = np.empty((R, self.Nt))
        dst = torch.from_numpy(res)
        events = []
        for lo, hi in _chunks(self.Nt):
            h_out[:, lo:hi].copy_(d_out[:, lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            events.append((lo, hi, ev))
        for lo, hi, ev in events:   # pinned->host copy of chunk k overlaps D2H of k+1..
            ev.synchronize()
            dst[:, lo:hi].copy_(h_out[:, lo:hi])
        return res[0] if one else res.T

    def _apply_host_tensor(self, alpha):
        """torch CPU tensor in -> torch CPU tensor out.  From pinned memory the H2D copy is
        one async DMA straight into the device staging buffer (no host staging), and the
        result comes back into pinned memory."""
        torch = _torch()
        if alpha.dim() not in (1, 2) or alpha.shape[0] != self.N:
            raise ShapeError(f"alpha must have length {self.N}, got {tuple(alpha.shape)}")
        one = alpha.dim() == 1
        R = 1 if one else alpha.shape[1]
        if R > self.max_rhs:
            raise ShapeError(f"at most {self.max_rhs} right-hand sides per apply")
        a = alpha.to(torch.float64)
        pinned = a.is_pinned()
        d_raw, d_in, d_out = self._staging(("tensor", R), lambda: (
            torch.empty((self.N, R), dtype=torch.float64, device=self.device),
            torch.empty((R, self.N), dtype=torch.float64, device=self.device),
            torch.empty((R, self.Nt), dtype=torch.float64, device=self.device)))
        stream = torch.cuda.current_stream(self.device)
        if one:
            d_in[0].copy_(a, non_blocking=pinned)
        else:   # (N, R) row-major on the host: copy as is, transpose on the device
            d_raw.copy_(a.contiguous(), non_blocking=pinned)
            d_in.copy_(d_raw.t())
        self.apply_device(d_in, d_out, R)
        res = torch.empty((R, self.Nt), dtype=torch.float64, pin_memory=pinned)
        res.copy_(d_out, non_blocking=pinned)
        stream.synchronize()
        return res[0] if one else res.t()


class AnovaKernelOperator:
    """Matrix-free multiplication by K = sum_l eta_l K_l on the GPU (anova.py:138-183).

    ``windows`` follows the reference (a ``WindowSet`` or a list validated as
    one).  ``strict=False`` accepts arbitrary, possibly overlapping windows
    (the C3/C5 recipes); ``weights`` overrides eta_l = 1/P in that mode.
    ``max_rhs`` sizes the workspace for multi-column alpha.  ``coeff_fft="device"``
    computes c_hat's plan-time transform with cuFFT instead of scipy's pocketfft
    (spectrum.regularize_kernel).
    """

    def __init__(self, X, windows, sigma, profile="default", targets=None, config=None, *,
                 strict=True, weights=None, device=None, max_rhs=1, window_eval="poly",
                 scaling=None, deterministic=False, coeff_fft="host"):
        X = _as_matrix(X, "sources")
        if strict:
            if not isinstance(windows, WindowSet):
                windows = WindowSet(windows)
            if weights is not None:
                raise ValidationError("weights are fixed to 1/P for a strict WindowSet")
        elif not isinstance(windows, (WindowSet, FreeWindowSet)):
            windows = FreeWindowSet(windows, weights)
        d = X.shape[1]
        for w in windows:
            if max(w) >= d or min(w) < 0:
                raise ValidationError(f"window {w} out of range for {d} columns")
        Z = None
        if targets is not None:
            Z = _as_matrix(targets, "targets")
            if Z.shape[1] != d:
                raise ShapeError(f"targets have {Z.shape[1]} columns, expected {d}")
        profile = resolve_profile(profile)
        if config is None:
            config = PeriodizationConfig.for_profile(profile)
        kernel = GaussianKernel(sigma)
        self.windows = windows
        self.sigma = float(sigma)
        self.profile = profile
        self.config = config
        self.n_sources = X.shape[0]
        self.n_targets = X.shape[0] if Z is None else Z.shape[0]
        self._plan = _Plan(X, Z, list(windows.windows), list(windows.weights), kernel, config,
                           profile, device, max_rhs, window_eval, scaling, coeff_fft=coeff_fft)
        if deterministic:
            self._plan.set_deterministic(True)
        self.operators = self._plan.windows

    def apply(self, alpha):
        a = alpha if hasattr(alpha, "is_cuda") else np.asarray(alpha, dtype=np.float64)
        if a.shape[0] != self.n_sources or len(a.shape) not in (1, 2):
            raise ShapeError(f"alpha must have length {self.n_sources}, got {tuple(a.shape)}")
        return self._plan.apply(a)

    def info(self):
        return self._plan.info()

    def close(self):
        self._plan.close()


class FastsumOperator:
    """Single-window fast Gaussian summation on the GPU (fastsum.py:182-256).

    ``apply`` returns the reference's ``apply`` (= Re of ``apply_complex``);
    the imaginary residue the reference discards is never formed.
    """

    def __init__(self, kernel, config, sources, targets=None, profile="default", *, device=None,
                 max_rhs=1, window_eval="poly", deterministic=False, coeff_fft="host"):
        if not isinstance(kernel, GaussianKernel):
            raise ValidationError("kernel must be a GaussianKernel")
        profile = resolve_profile(profile)
        X = _as_matrix(sources, "sources")
        d = X.shape[1]
        if not 1 <= d <= 3:
            raise ValidationError(f"fast summation supports 1..3 dimensions, got {d}")
        if config is None:
            config = PeriodizationConfig.for_profile(profile)
        Z = None
        if targets is not None:
            Z = _as_matrix(targets, "targets")
            if Z.shape[1] != d:
                raise ShapeError(f"targets have {Z.shape[1]} columns, sources {d}")
        self.kernel = kernel
        self.config = config
        self.profile = profile
        self.dims = d
        self._plan = _Plan(X, Z, [tuple(range(d))], [1.0], kernel, config, profile, device, max_rhs,
                           window_eval, coeff_fft=coeff_fft)
        self._nodes = (X, Z)             # for the lazily built NfftPlan views
        self._nfft = {}
        self._device = device
        self._window_eval = window_eval
        if deterministic:
            self._plan.set_deterministic(True)
        w = self._plan.windows[0]
        self.scale = w.scale
        self.center = w.center
        self.scaled_kernel = w.scaled_kernel
        self.coeffs = w.coeffs

    @property
    def n_sources(self):
        return self._plan.N

    @property
    def n_targets(self):
        return self._plan.Nt

    def apply(self, alpha):
        a = alpha if hasattr(alpha, "is_cuda") else np.asarray(alpha, dtype=np.float64)
        if a.shape[0] != self.n_sources or len(a.shape) not in (1, 2):
            raise ShapeError(f"alpha must have length {self.n_sources}, got shape {tuple(a.shape)}")
        return self._plan.apply(a)

    # -- the reference's NFFT-level view of the operator (fastsum.py:228-252) ----------
    def _nfft_plan(self, side):
        """GPU NfftPlan on the scaled sources / targets, built on first use: the nodes are
        (x - center) * scale exactly as fastsum.py:228-232 forms them."""
        if side not in self._nfft:
            from .nfft import NfftPlan
            from .params import GridSpec

            A = self._nodes[0 if side == "source" else 1]
            if A is None:
                self._nfft[side] = None
            else:
                A = A.cpu().numpy() if hasattr(A, "is_cuda") else A
                grid = GridSpec((self.config.coeff_grid,) * self.dims)
                self._nfft[side] = NfftPlan(grid, (A - self.center) * self.scale, self.profile,
                                            device=self._device, window_eval=self._window_eval)
        return self._nfft[side]

    @property
    def source_plan(self):
        return self._nfft_plan("source")

    @property
    def target_plan(self):
        return self._nfft_plan("target")

    def apply_complex(self, alpha):
        """forward_Z(c_hat * adjoint_X(alpha)) for real or complex alpha, without taking the
        real part (fastsum.py:243-252): the NFFT stages run on the GPU, the M^d spectrum
        product and the Hermitian folding on the host.  ``apply`` is the fused real path."""
        a = np.asarray(alpha)
        if a.ndim != 1 or a.shape[0] != self.n_sources:
            raise ShapeError(f"alpha must have length {self.n_sources}, got shape {a.shape}")
        spectrum = self.source_plan.adjoint(a.astype(np.complex128, copy=False))
        out_plan = self.target_plan if self.target_plan is not None else self.source_plan
        return out_plan.forward(self.coeffs.ravel() * spectrum)


def fastsum_build(kernel, config, sources, targets=None, profile="default", **kw):
    return FastsumOperator(kernel, config, sources, targets, profile, **kw)


def fastsum_apply(op, alpha):
    return op.apply(alpha)


def anova_build(X, windows, sigma, profile="default", targets=None, config=None, **kw):
    return AnovaKernelOperator(X, windows, sigma, profile, targets, config, **kw)


def anova_apply(op, alpha):
    return op.apply(alpha)
