"""The reference's accuracy oracles and its matvec benchmark, on the GPU.

- ``direct_sum``: dense ``s(z_i) = sum_j alpha_j kappa(z_i, x_j)`` (fastsum.py:162-179), the
  exact kernel the fast summation approximates.  Chunked fp64 on the device: the pairwise
  distances use the same ``|z|^2 + |x|^2 - 2 z.x`` expansion and clamp as the reference.
- ``ndft_direct`` / ``ndft_adjoint_direct``: O(N |I_M|) direct transforms (nfft.py:263-300),
  the oracles of ``NfftPlan``.
- ``bench_mvm``: the reference's only benchmark, ``nfftkrr bench-mvm`` (cli.py:295-369): per
  N, X ~ U[0,1]^d and alpha ~ N(0,1) from PCG64, one warm-up apply, the mean of ``runs``
  timed applies, the direct sum and the relative error below the size guard (20000,
  oracle.py:13); the same CSV columns and ``run-report/1`` JSON.

These are dense O(N^2) / O(N |I_M|) checkers, not the product path; they use torch on the
given device (cuda by default, cpu allowed for small checks).
"""

from __future__ import annotations

import csv
import json
import time

import numpy as np

from .errors import ShapeError, ValidationError
from .params import GaussianKernel, GridSpec

SIZE_GUARD = 20000          # oracle.py:13
REPORT_FORMAT = "run-report/1"   # cli.py:40
RNG_NAME = "numpy-pcg64"    # data.py:16


def _torch():
    import torch

    return torch


def _device(device):
    torch = _torch()
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    return torch.device(device)


def direct_sum(kernel: GaussianKernel, sources, targets, alpha, chunk: int = 4096, device=None):
    """Exact dense evaluation of s(z_i) = sum_j alpha_j kappa(z_i, x_j) (fastsum.py:162-179)."""
    torch = _torch()
    X = np.atleast_2d(np.asarray(sources, dtype=np.float64))
    Z = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    a = np.asarray(alpha, dtype=np.float64)
    if X.ndim != 2 or Z.ndim != 2 or X.shape[1] != Z.shape[1]:
        raise ShapeError("sources and targets must be (N, d) matrices with equal d")
    if a.shape != (X.shape[0],):
        raise ShapeError(f"alpha must have length {X.shape[0]}, got {a.shape}")
    dev = _device(device)
    Xd = torch.from_numpy(X).to(dev)
    ad = torch.from_numpy(a).to(dev)
    sq_x = (Xd * Xd).sum(dim=1)
    sigma = float(kernel.sigma)
    out = np.empty(Z.shape[0])
    for lo in range(0, Z.shape[0], chunk):
        zc = torch.from_numpy(Z[lo:lo + chunk]).to(dev)
        d2 = (zc * zc).sum(dim=1)[:, None] + sq_x[None, :] - 2.0 * (zc @ Xd.T)
        d2.clamp_(min=0.0)
        r = torch.sqrt(d2)
        out[lo:lo + chunk] = (torch.exp(-(r / sigma) ** 2) @ ad).cpu().numpy()
    return out


def _grid_and_nodes(grid, nodes):
    from .nfft import validate_nodes

    if not isinstance(grid, GridSpec):
        grid = GridSpec(tuple(grid))
    return grid, validate_nodes(nodes, grid.dims)


def _modes(grid: GridSpec):
    axes = [np.arange(-b // 2, b // 2) for b in grid.bandwidths]
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([x.ravel() for x in g], axis=1).astype(np.float64)


def ndft_direct(grid, nodes, f_hat, chunk: int = 4096, device=None):
    """Direct O(N |I_M|) forward transform f_j = sum_k f_hat_k e^{2 pi i k.x_j} (nfft.py:263-281)."""
    torch = _torch()
    grid, coords = _grid_and_nodes(grid, nodes)
    f_hat = np.asarray(f_hat)
    if f_hat.shape == tuple(grid.bandwidths):
        f_hat = f_hat.ravel()
    if f_hat.ndim != 1 or f_hat.shape[0] != grid.n_modes:
        raise ShapeError(f"coefficient vector must have length {grid.n_modes}, got shape {f_hat.shape}")
    dev = _device(device)
    K = torch.from_numpy(_modes(grid)).to(dev)
    fh = torch.from_numpy(np.asarray(f_hat, dtype=np.complex128)).to(dev)
    out = np.empty(coords.shape[0], dtype=np.complex128)
    for lo in range(0, coords.shape[0], chunk):
        phase = torch.from_numpy(coords[lo:lo + chunk]).to(dev) @ K.T
        out[lo:lo + chunk] = (torch.exp(2j * np.pi * phase) @ fh).cpu().numpy()
    return out


def ndft_adjoint_direct(grid, nodes, c, chunk: int = 4096, device=None):
    """Direct O(N |I_M|) adjoint f_hat_k = sum_j c_j e^{-2 pi i k.x_j} (nfft.py:284-300)."""
    torch = _torch()
    grid, coords = _grid_and_nodes(grid, nodes)
    c = np.asarray(c)
    if c.ndim != 1 or c.shape[0] != coords.shape[0]:
        raise ShapeError(f"node vector must have length {coords.shape[0]}, got shape {c.shape}")
    dev = _device(device)
    K = torch.from_numpy(_modes(grid)).to(dev)
    cd = torch.from_numpy(np.asarray(c, dtype=np.complex128)).to(dev)
    out = torch.zeros(grid.n_modes, dtype=torch.complex128, device=dev)
    for lo in range(0, coords.shape[0], chunk):
        phase = torch.from_numpy(coords[lo:lo + chunk]).to(dev) @ K.T
        out += torch.exp(-2j * np.pi * phase).T @ cd[lo:lo + chunk]
    return out.cpu().numpy()


def bench_mvm(n_list, d: int = 3, sigma: float = 1.0, profile="default", runs: int = 3, seed: int = 0,
              out: str | None = None, report_out: str | None = None, verbose: bool = True):
    """``nfftkrr bench-mvm`` (cli.py:295-369) on the GPU operator; returns the table rows.

    Times are host wall clock around the synchronous ``FastsumOperator.apply`` (numpy in and
    out, as the reference's), so they include the host<->device copies of alpha and the result.
    """
    from . import __version__
    from .operators import fastsum_build

    n_list = [int(n) for n in n_list]
    if any(n <= 0 for n in n_list) or n_list != sorted(n_list):
        raise ValidationError(f"--n-list must be ascending positive integers, got {n_list}")
    kernel = GaussianKernel(sigma)
    rng = np.random.default_rng(seed)
    rows = []
    for n in n_list:
        X = rng.uniform(0.0, 1.0, size=(n, d))
        alpha = rng.standard_normal(n)
        op = fastsum_build(kernel, None, X, profile=profile)
        op.apply(alpha)   # warm-up, excludes one-time allocations from timing
        t_fast = []
        for _ in range(runs):
            t0 = time.perf_counter()
            fast = op.apply(alpha)
            t_fast.append(time.perf_counter() - t0)
        row = {"n": n, "t_fast": float(np.mean(t_fast))}
        if n <= SIZE_GUARD:
            t_direct = []
            for _ in range(runs):
                t0 = time.perf_counter()
                dense = direct_sum(kernel, X, X, alpha)
                t_direct.append(time.perf_counter() - t0)
            row["t_direct"] = float(np.mean(t_direct))
            row["rel_error"] = float(np.linalg.norm(fast - dense) / np.linalg.norm(dense))
            row["direct_ran"] = True
        else:
            row["t_direct"] = None
            row["rel_error"] = None
            row["direct_ran"] = False
        rows.append(row)
        if verbose:
            direct_txt = f"{row['t_direct']:.4f}s" if row["direct_ran"] else "skipped (size guard)"
            err_txt = f"{row['rel_error']:.3e}" if row["direct_ran"] else "-"
            print(f"N={n}: fast {row['t_fast']:.4f}s, direct {direct_txt}, rel_error {err_txt}")
    if out is not None:
        with open(out, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(["n", "t_direct", "t_fast", "rel_error", "direct_ran"])
            for row in rows:
                w.writerow([row["n"], "" if row["t_direct"] is None else repr(row["t_direct"]),
                            repr(row["t_fast"]), "" if row["rel_error"] is None else repr(row["rel_error"]),
                            row["direct_ran"]])
    if report_out is not None:
        payload = {
            "format": REPORT_FORMAT,
            "command": "bench-mvm",
            "config": {"d": d, "sigma": sigma, "profile": profile if isinstance(profile, str) else profile.name,
                       "runs": runs},
            "timings": {str(r["n"]): {"t_fast": r["t_fast"], "t_direct": r["t_direct"]} for r in rows},
            "mvm_relative_errors": {str(r["n"]): r["rel_error"] for r in rows if r["direct_ran"]},
            "seed": seed,
            "rng": RNG_NAME,
            "versions": {"paper_2111_10140_b200": __version__},
        }
        with open(report_out, "w", encoding="utf-8") as fh:
            json.dump(payload, fh, indent=1)
            fh.write("\n")
    return rows


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser(description="bench-mvm (cli.py:295-369) on the GPU operator")
    ap.add_argument("--n-list", type=int, nargs="+", default=[1000, 10000, 100000])
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--profile", default="default")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="bench_mvm.csv")
    ap.add_argument("--report-out", default=None)
    a = ap.parse_args()
    bench_mvm(a.n_list, a.d, a.sigma, a.profile, a.runs, a.seed, a.out, a.report_out)
