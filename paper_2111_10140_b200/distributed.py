"""Multi-GPU ANOVA matvec: one process per GPU, torch.distributed (NCCL) plumbing.

The reference has no parallelism.  The path shards naturally
in one exchange step per matvec:

* ``WindowSharded`` (C3/C5: many windows) — windows are dealt to ranks by
  LPT on their modelled spread+gather time (``window_costs``); every rank holds all
  points and alpha, computes ``sum_{l in S_rank} eta_l K_l alpha`` and one
  all-reduce sums the N-vector partials.  The terms are independent
  (anova.py:179-183), so the result equals the single-GPU sum up to the
  order of the cross-window additions.
* ``PointSharded`` (C4: one window, huge N) — every rank owns N/p points and
  their alpha; the bbox (hence center/scale) is all-reduced first so every
  rank builds the same multiplier; each rank spreads its points onto a full
  grid, the grids are all-reduced (the spread is linear in the node set,
  nfft.py:241-245), every rank runs the spectral stage and gathers its own
  points.  The output stays row-sharded.

Both classes take the local compute as injectable backends so the
orchestration is testable on CPU (gloo) without a GPU (tests/test_distributed.py);
the default backends are the CUDA operators of this package.

``sharded_cg`` runs the reference's CG (krr.py:76-110) over either operator
(SURVEY §8(e)): window-sharded with replicated vectors (the matvec already
all-reduces Ap, so every rank runs identical vector updates), point-sharded
with row-sharded vectors and scalar all-reduces (b.b once, then per iteration
p.Ap with the non-finite flag, and r.r).  The control loop is ``cg.run_cg``;
the vector updates run as the fused device kernels of the C ABI
(``afs_cg_vec_*``), or their torch CPU mirror in the gloo tests.
"""

from __future__ import annotations

import numpy as np

from .params import AccuracyProfile, PeriodizationConfig


def lpt_assign(costs, world):
    """Longest-processing-time deal: returns owner rank per item (ties -> lowest rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    owner = [0] * len(costs)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += costs[i]
    return owner


def window_costs(windows, N, m):
    """Modelled spread+gather time of each window on one B200.

    At m = 4 the measured per-node times of the kernels each window gets:
    3-D 155 ps (tensor-core kernels), 2-D 25 ps when the window is dense enough for the sub-cell
    kernels (about N >= 5e6) and 73 ps on the half-cell kernels, 1-D 20 ps (batched / fused).  C3
    prices a 3-D window at 6.2 2-D windows (1.55 vs 0.248 ms at N = 1e7); the bare touch count
    N (2m)^d would say 8.  Other cutoffs: fp64 work per node and pass -- touches (2m)^d + window
    values 2m d 12 + line products (2m)^(d-1) -- over the FMA kernels' pipe efficiency 0.58."""
    costs = []
    for w in windows:
        d = len(w)
        if m == 4:
            ps = {1: 20.0, 2: 25.0 if N >= 5_000_000 else 73.0, 3: 155.0}[d]
            costs.append(float(N) * ps)
        else:
            work = (2 * m) ** d + 2 * m * d * 12 + (2 * m) ** (d - 1)
            costs.append(float(N) * work / 0.58)
    return costs


class WindowSharded:
    """Window-sharded ANOVA operator.

    ``make_local(windows, weights)`` returns, for this rank's windows, an object with
    ``apply(alpha) -> partial`` or such a callable (default: a CUDA
    ``AnovaKernelOperator``, kept as ``self.local``).  ``apply`` returns the full sum on
    every rank.
    """

    def __init__(self, X, windows, sigma, *, M=64, m=4, oversampling=2.0, group=None,
                 make_local=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.windows = [tuple(w) for w in windows]
        P = len(self.windows)
        self.N = X.shape[0]
        self.owner = lpt_assign(window_costs(self.windows, self.N, m), self.world)
        self.mine = [l for l in range(P) if self.owner[l] == self.rank]
        weights = [1.0 / P] * len(self.mine)
        if make_local is None:
            make_local = _cuda_window_backend(X, sigma, M, m, oversampling, device)
        self.local = make_local([self.windows[l] for l in self.mine], weights) if self.mine else None

    def apply(self, alpha):
        import torch

        if self.local is not None:
            part = getattr(self.local, "apply", self.local)(alpha)
        else:
            part = torch.zeros_like(alpha)
        part = part.contiguous()
        self.dist.all_reduce(part, group=self.group)
        return part

    @property
    def n_sources(self):
        return self.N

    n_targets = n_sources
    rows_sharded = False


def _cuda_window_backend(X, sigma, M, m, oversampling, device):
    from .operators import AnovaKernelOperator

    def make(windows, weights):
        return AnovaKernelOperator(X, windows, sigma, AccuracyProfile("sharded", oversampling, m),
                                   None, PeriodizationConfig(coeff_grid=M), strict=False,
                                   weights=weights, device=device)
    return make


def global_bbox(X_local, windows, group=None):
    """Per-window (min, max) over all ranks' points (all-reduce MIN / MAX)."""
    import torch
    import torch.distributed as dist

    out = []
    for w in windows:
        sub = X_local[:, list(w)]
        if isinstance(sub, np.ndarray):
            lo = torch.from_numpy(sub.min(axis=0).copy())
            hi = torch.from_numpy(sub.max(axis=0).copy())
        else:
            lo, hi = sub.amin(dim=0).clone(), sub.amax(dim=0).clone()
        dev = torch.device("cuda", torch.cuda.current_device()) if (
            dist.get_backend(group) == "nccl") else torch.device("cpu")
        lo, hi = lo.to(dev), hi.to(dev)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
        out.append((lo.cpu().numpy(), hi.cpu().numpy()))
    return out


class PointSharded:
    """Point-sharded fast summation (one or more windows, all ranks share the grids).

    ``backend`` must provide ``spread(alpha) -> grids`` (a tensor this class
    all-reduces in place), ``spectral(grids)`` and ``gather(grids) -> out``.
    """

    def __init__(self, backend, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.backend = backend

    def apply(self, alpha_local):
        grids = self.backend.spread(alpha_local)
        self.dist.all_reduce(grids, group=self.group)
        self.backend.spectral(grids)
        out = self.backend.gather(grids)
        if alpha_local.dim() == 1 and out.dim() == 2:
            out = out[0]
        return out

    rows_sharded = True


class CudaPointBackend:
    """Stage backend over a CUDA plan whose exchange buffer is a torch tensor (NCCL-visible).

    exchange="spectrum" (default): spread + forward transform locally, all-reduce
    the pruned spectra E (.) F(g) -- K^(d-1)(M/2+1) complex values per window, 17 MB per rhs
    for C4 -- then inverse transform + gather.  exchange="grid": all-reduce the real
    oversampled grids (n^d values, 134 MB per rhs for C4) and run the fused spectral stage."""

    def __init__(self, X_local, windows, sigma, *, M, m, oversampling=2.0, weights=None,
                 max_rhs=1, group=None, device=None, exchange="spectrum"):
        import torch

        from .operators import AnovaKernelOperator, bbox_scaling

        cfg = PeriodizationConfig(coeff_grid=M)
        boxes = global_bbox(X_local, windows, group)
        scaling = [bbox_scaling(lo, hi, cfg) for lo, hi in boxes]
        P = len(windows)
        self.op = AnovaKernelOperator(X_local, windows, sigma, AccuracyProfile("pts", oversampling, m),
                                      None, cfg, strict=False,
                                      weights=weights if weights is not None else [1.0 / P] * P,
                                      device=device, max_rhs=max_rhs, scaling=scaling)
        self.plan = self.op._plan
        if exchange not in ("spectrum", "grid"):
            raise ValueError(f"exchange must be 'spectrum' or 'grid', got {exchange!r}")
        self.exchange = exchange
        if exchange == "grid":
            self.per = self.plan.grid_doubles_per_rhs()
            self.buf = torch.zeros(self.per * self.plan.max_rhs, dtype=torch.float64,
                                   device=self.plan.device)
            self.plan.bind_grids(self.buf)
        else:
            self.per = self.plan.spectrum_doubles_per_rhs()
            self.buf = torch.zeros(self.per * self.plan.max_rhs, dtype=torch.float64,
                                   device=self.plan.device)
            self.plan.bind_spectra(self.buf)
        self.R = 1

    def spread(self, alpha):
        """Local spread (+ forward transform): returns the buffer to all-reduce."""
        a = alpha if alpha.dim() == 2 else alpha[None, :]
        self.R = a.shape[0]
        self.plan.spread_device(a.contiguous(), self.R)
        if self.exchange == "spectrum":
            self.plan.spectral_forward_device(self.R)
        return self.buf[: self.per * self.R]

    def spectral(self, exchanged):
        if self.exchange == "spectrum":
            self.plan.spectral_inverse_device(self.R)
        else:
            self.plan.spectral_device(self.R)

    def gather(self, grids):
        import torch

        out = torch.empty((self.R, self.plan.Nt), dtype=torch.float64, device=self.plan.device)
        self.plan.gather_device(out, self.R)
        return out


# --------------------------------------------------------------------------- sharded CG
def sharded_cg(operator, b, beta, tol=1e-3, maxiter=1000, *, vectors=None, group=None):
    """CG for (K + beta I) x = b over a sharded operator (krr.py:76-110).

    ``operator.apply(p) -> K p``: a ``WindowSharded`` returns the full, all-reduced
    vector and the CG vectors are replicated; a ``PointSharded`` returns this rank's rows,
    the vectors are row-sharded and the three scalars are all-reduced.  ``b`` is the full
    vector or this rank's rows accordingly.  Every rank takes the same decisions.
    Returns a ``CgResult`` whose x is shaped like b."""
    import torch.distributed as dist

    from .cg import CudaCgVectors, run_cg

    reduce = None
    if getattr(operator, "rows_sharded", False):
        def reduce(ws, lo, hi):
            dist.all_reduce(ws[lo:hi], group=group)
    if vectors is None:
        vectors = CudaCgVectors(b.device)
    return run_cg(operator.apply, b, beta, tol, maxiter, vectors, reduce)
