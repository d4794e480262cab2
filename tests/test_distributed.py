"""Multi-rank orchestration on CPU (gloo, world_size 2): window sharding and point
sharding must reproduce the single-process ANOVA sum.  The local compute is the
CPU oracle / a numpy model of the device stages (test infrastructure); the
CUDA backends of the same classes run on the GPU box."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from paper_2111_10140_b200.distributed import lpt_assign, window_costs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _free_port()
    mp.spawn(fn, args=(world, port) + args, nprocs=world, join=True)


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def test_lpt_balances_c3_windows():
    w = synthetic.C3_WINDOWS
    costs = window_costs(w, 10_000_000, 4)
    for world in (1, 2, 4, 8):
        owner = lpt_assign(costs, world)
        loads = [sum(c for c, o in zip(costs, owner) if o == r) for r in range(world)]
        assert sorted(set(owner)) == list(range(world))
        # LPT bound: max load <= 4/3 optimum (and >= the mean)
        assert max(loads) <= 4.0 / 3.0 * max(sum(costs) / world, max(costs)) + 1e-6
        assert owner == lpt_assign(costs, world)   # deterministic


# --------------------------------------------------------------------------- window sharding
def _window_worker(rank, world, port, out_path):
    _init(rank, world, port)
    from oracle import fastsum_oracle as orc
    from paper_2111_10140_b200.distributed import WindowSharded

    w = synthetic.c3(N=400)

    def make_local(windows, weights):
        def apply(alpha):
            a = alpha.numpy()
            s = np.zeros(w.N)
            for eta, win in zip(weights, windows):
                s += eta * orc.fastsum_apply(w.X[:, list(win)], a, w.sigma, w.M, w.m)
            return torch.from_numpy(s)
        return apply

    op = WindowSharded(w.X, w.windows, w.sigma, M=w.M, m=w.m, make_local=make_local)
    res = op.apply(torch.from_numpy(w.alpha.copy())).numpy()
    np.save(out_path + f".{rank}.npy", res)
    dist.destroy_process_group()


def test_window_sharded_matches_single_process(tmp_path):
    from oracle import fastsum_oracle as orc

    out = str(tmp_path / "ws")
    _run(_window_worker, 2, out)
    w = synthetic.c3(N=400)
    ref = orc.anova_apply(w.X, w.windows, w.alpha, w.sigma, w.M, w.m)
    for r in range(2):
        got = np.load(out + f".{r}.npy")
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13


# --------------------------------------------------------------------------- point sharding
class NumpyPointBackend:
    """numpy model of the device stages for one window (spread / spectral / gather)."""

    def __init__(self, X_local, win, sigma, M, m, group=None, exchange="grid"):
        from oracle import fastsum_oracle as orc
        from paper_2111_10140_b200 import GaussianKernel, PeriodizationConfig, regularize_kernel
        from paper_2111_10140_b200.distributed import global_bbox
        from paper_2111_10140_b200.operators import bbox_scaling
        from paper_2111_10140_b200.spectrum import window_multiplier

        self.orc = orc
        self.exchange = exchange
        cfg = PeriodizationConfig(coeff_grid=M)
        (lo, hi), = global_bbox(X_local, [win], group)
        center, scale = bbox_scaling(lo, hi, cfg)
        self.d = len(win)
        self.n = 2 * M
        self.M, self.m = M, m
        self.b = np.pi * (2.0 - M / self.n)
        self.E = window_multiplier(regularize_kernel(GaussianKernel(sigma * scale), cfg, self.d),
                                   M, self.n, m)
        self.xs = (X_local[:, list(win)] - center) * scale

    def _tensor(self):
        n, m = self.n, self.m
        flat, w = None, None
        for t in range(self.d):
            nx = n * self.xs[:, t]
            c = np.floor(nx)[:, None] + np.arange(1 - m, m + 1)[None, :]
            idx = np.mod(c, n).astype(np.int64)
            val = self.orc.kb_window(nx[:, None] - c, m, self.b)
            if flat is None:
                flat, w = idx, val
            else:
                flat = (flat[:, :, None] * n + idx[:, None, :]).reshape(len(nx), -1)
                w = (w[:, :, None] * val[:, None, :]).reshape(len(nx), -1)
        return flat, w

    def spread(self, alpha):
        """Local spread; with exchange="spectrum" also the forward half of the spectral stage,
        so the returned buffer (what PointSharded all-reduces) is the pruned spectrum."""
        flat, w = self._tensor()
        g = np.bincount(flat.ravel(), (alpha.numpy()[:, None] * w).ravel(), minlength=self.n ** self.d)
        if self.exchange == "grid":
            self.buf = torch.from_numpy(g)
        else:
            S = self._forward(g)
            self.shape = S.shape
            self.buf = torch.from_numpy(np.ascontiguousarray(S).view(np.float64).ravel().copy())
        return self.buf

    def _forward(self, g):
        n, M, d = self.n, self.M, self.d
        H = M // 2 + 1
        sym = (np.arange(M + 1) - M // 2) % n
        A = np.fft.fft(g.reshape((n,) * d), axis=-1)[..., :H]
        if d == 3:
            A = np.fft.fft(A, axis=1)[:, sym, :]
        if d >= 2:
            A = np.fft.fft(A, axis=0)[sym]
        return A * self.E

    def _inverse(self, S):
        n, M, d = self.n, self.M, self.d
        H = M // 2 + 1
        sym = (np.arange(M + 1) - M // 2) % n
        A = S
        if d >= 2:
            Y = np.zeros((n,) + S.shape[1:], dtype=complex)
            Y[sym] = S
            A = n * np.fft.ifft(Y, axis=0)
        if d == 3:
            full = np.zeros((n, n, H), dtype=complex)
            full[:, sym, :] = A
            A = n * np.fft.ifft(full, axis=1)
        line = np.zeros(A.shape[:-1] + (n,), dtype=complex)
        line[..., :H] = A
        return (n * np.fft.ifft(line, axis=-1)).real.ravel()

    def spectral(self, buf):
        if self.exchange == "grid":
            self.grid = self._inverse(self._forward(buf.numpy()))
        else:
            self.grid = self._inverse(buf.numpy().view(np.complex128).reshape(self.shape))

    def gather(self, buf):
        flat, w = self._tensor()
        return torch.from_numpy((self.grid[flat] * w).sum(1))


def _point_worker(rank, world, port, out_path):
    _init(rank, world, port)
    from paper_2111_10140_b200.distributed import PointSharded

    exchange = out_path.rsplit("_", 1)[-1]
    wl = synthetic.c4(N=600, R=1)
    shard = np.array_split(np.arange(wl.N), world)[rank]
    be = NumpyPointBackend(wl.X[shard], (0, 1, 2), wl.sigma, wl.M, wl.m, exchange=exchange)
    res = PointSharded(be).apply(torch.from_numpy(wl.alpha[shard, 0].copy())).numpy()
    np.save(out_path + f".{rank}.npy", res)
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["grid", "spectrum"])
def test_point_sharded_matches_single_process(tmp_path, exchange):
    """world 2 over gloo: all-reducing either the grids or the pruned spectra (linear in the
    node set) reproduces the single-process fast sum."""
    from oracle import fastsum_oracle as orc

    out = str(tmp_path / f"ps_{exchange}")
    _run(_point_worker, 2, out)
    wl = synthetic.c4(N=600, R=1)
    ref = orc.fastsum_apply(wl.X, wl.alpha[:, 0], wl.sigma, wl.M, wl.m)
    got = np.concatenate([np.load(out + f".{r}.npy") for r in range(2)])
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


# --------------------------------------------------------------------------- sharded CG
def _oracle_windows_local(w):
    from oracle import fastsum_oracle as orc

    def make_local(windows, weights):
        def apply(alpha):
            a = alpha.numpy()
            s = np.zeros(w.N)
            for eta, win in zip(weights, windows):
                s += eta * orc.fastsum_apply(w.X[:, list(win)], a, w.sigma, w.M, w.m)
            return torch.from_numpy(s)
        return apply
    return make_local


def _cg_window_worker(rank, world, port, out_path):
    _init(rank, world, port)
    from paper_2111_10140_b200.cg import TorchCgVectors
    from paper_2111_10140_b200.distributed import WindowSharded, sharded_cg

    w = synthetic.c5(N=300)
    op = WindowSharded(w.X, w.windows, w.sigma, M=w.M, m=w.m, make_local=_oracle_windows_local(w))
    res = sharded_cg(op, torch.from_numpy(w.y.copy()), w.beta, 1e-6, 400, vectors=TorchCgVectors())
    np.save(out_path + f".{rank}.npy", np.concatenate([[res.iterations, res.residual],
                                                       res.x.numpy()]))
    dist.destroy_process_group()


def test_window_sharded_cg_matches_single_process(tmp_path):
    """CG with replicated vectors over window shards (one all-reduce of Ap per iteration):
    every rank ends with the single-process solution at the same iteration count."""
    from oracle import fastsum_oracle as orc

    out = str(tmp_path / "wcg")
    _run(_cg_window_worker, 2, out)
    w = synthetic.c5(N=300)
    rx, rit, _, _ = orc.cg_solve(
        lambda v: orc.anova_apply(w.X, w.windows, v, w.sigma, w.M, w.m) + w.beta * v,
        w.y, tol=1e-6, maxiter=400)
    for r in range(2):
        got = np.load(out + f".{r}.npy")
        assert abs(int(got[0]) - rit) <= 1
        assert np.linalg.norm(got[2:] - rx) / np.linalg.norm(rx) < 1e-8


def _cg_point_worker(rank, world, port, out_path):
    _init(rank, world, port)
    from paper_2111_10140_b200.cg import TorchCgVectors
    from paper_2111_10140_b200.distributed import PointSharded, sharded_cg

    wl = synthetic.c4(N=500, R=1)
    y = np.sin(7.0 * wl.X).sum(axis=1)
    shard = np.array_split(np.arange(wl.N), world)[rank]
    be = NumpyPointBackend(wl.X[shard], (0, 1, 2), wl.sigma, 16, wl.m, exchange="spectrum")
    res = sharded_cg(PointSharded(be), torch.from_numpy(y[shard].copy()), 0.5, 1e-8, 300,
                     vectors=TorchCgVectors())
    np.save(out_path + f".{rank}.npy", np.concatenate([[res.iterations, res.residual],
                                                       res.x.numpy()]))
    dist.destroy_process_group()


def test_point_sharded_cg_matches_single_process(tmp_path):
    """CG with row-sharded vectors and scalar all-reduces: the stacked shards
    equal the single-process solution, with the same iteration count and residual."""
    from oracle import fastsum_oracle as orc

    out = str(tmp_path / "pcg")
    _run(_cg_point_worker, 2, out)
    wl = synthetic.c4(N=500, R=1)
    y = np.sin(7.0 * wl.X).sum(axis=1)
    rx, rit, _, _ = orc.cg_solve(lambda v: orc.fastsum_apply(wl.X, v, wl.sigma, 16, wl.m) + 0.5 * v,
                                 y, tol=1e-8, maxiter=300)
    parts = [np.load(out + f".{r}.npy") for r in range(2)]
    for p in parts:
        assert abs(int(p[0]) - rit) <= 1
    assert parts[0][1] == parts[1][1]           # identical decisions on every rank
    x = np.concatenate([p[2:] for p in parts])
    assert np.linalg.norm(x - rx) / np.linalg.norm(rx) < 1e-8


def test_host_cg_path_is_bitwise_the_reference_loop():
    """cg_solve on a plain callable runs the shared control loop on numpy vectors with the
    reference's elementwise expressions (krr.py:86-109): bit-identical to the oracle loop."""
    from oracle import fastsum_oracle as orc
    from paper_2111_10140_b200.krr import cg_solve

    rng = np.random.default_rng(7)
    A = rng.standard_normal((60, 60))
    A = A @ A.T + 60 * np.eye(60)
    b = rng.standard_normal(60)
    got = cg_solve(lambda v: A @ v, b, tol=1e-10, maxiter=200)
    rx, rit, rres, rconv = orc.cg_solve(lambda v: A @ v, b, tol=1e-10, maxiter=200)
    assert got.iterations == rit and got.converged == rconv
    np.testing.assert_array_equal(got.x, rx)
    assert got.residual == rres
    with pytest.raises(Exception, match="non-positive curvature"):
        cg_solve(lambda v: -v, b, tol=1e-10, maxiter=5)
    with pytest.raises(Exception, match="non-finite operator output at iteration 1"):
        cg_solve(lambda v: v * np.nan, b, tol=1e-10, maxiter=5)
