"""Two ranks sharing the one GPU of the box, over gloo (host-staged all-reduce, so no
rank's kernels wait on another's): the CUDA backends of window sharding, point sharding
(grid and spectrum exchange) and the sharded CG drivers must reproduce the single-rank
operator / solve.  The collectives are NCCL in production (bench.py)."""

import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, *args):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    mp.spawn(fn, args=(2, _free_port()) + args, nprocs=2, join=True)


def _init(rank, world, port):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return torch, dist


def _c3_small():
    from paper_2111_10140_b200 import synthetic

    return synthetic.c3(N=20_000)


def _window_worker(rank, world, port, out):
    torch, dist = _init(rank, world, port)
    from paper_2111_10140_b200.distributed import WindowSharded

    w = _c3_small()
    op = WindowSharded(w.X, w.windows, w.sigma, M=w.M, m=w.m, device=0)
    res = op.apply(torch.from_numpy(w.alpha).cuda())
    np.save(f"{out}.{rank}.npy", res.cpu().numpy())
    dist.destroy_process_group()


def test_window_sharded_cuda_two_ranks(tmp_path):
    import paper_2111_10140_b200 as afs

    out = str(tmp_path / "ws")
    _run(_window_worker, out)
    w = _c3_small()
    ref = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                                  afs.PeriodizationConfig(coeff_grid=w.M), strict=False).apply(w.alpha)
    for r in range(2):
        got = np.load(f"{out}.{r}.npy")
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"window-sharded rank {r}: rel l2 {err:.2e}")
        assert err < 1e-13


def _c4_small():
    from paper_2111_10140_b200 import synthetic

    return synthetic.c4(N=40_000, R=2)


def _point_worker(rank, world, port, out, exchange):
    torch, dist = _init(rank, world, port)
    from paper_2111_10140_b200.distributed import CudaPointBackend, PointSharded

    w = _c4_small()
    shard = np.array_split(np.arange(w.N), world)[rank]
    be = CudaPointBackend(w.X[shard], [(0, 1, 2)], w.sigma, M=w.M, m=w.m, max_rhs=2, device=0,
                          exchange=exchange)
    a = torch.from_numpy(np.ascontiguousarray(w.alpha[shard].T)).cuda()
    res = PointSharded(be).apply(a)
    np.save(f"{out}.{rank}.npy", res.cpu().numpy().T)
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["grid", "spectrum"])
def test_point_sharded_cuda_two_ranks(tmp_path, exchange):
    import paper_2111_10140_b200 as afs

    out = str(tmp_path / f"ps_{exchange}")
    _run(_point_worker, out, exchange)
    w = _c4_small()
    ref = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                                  afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                  max_rhs=2).apply(w.alpha)
    got = np.concatenate([np.load(f"{out}.{r}.npy") for r in range(2)])
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print(f"point-sharded [{exchange}]: rel l2 {err:.2e}")
    assert err < 1e-13


def _c2_small():
    """The C2 recipe (3 windows, beta=1): well conditioned, so single- and two-rank solves
    that differ only by the order of cross-window additions stay within roundoff."""
    from paper_2111_10140_b200 import synthetic

    return synthetic.c2(N=20_000, n_test=10)


def _cg_window_worker(rank, world, port, out):
    torch, dist = _init(rank, world, port)
    import paper_2111_10140_b200 as afs

    w = _c2_small()
    op = afs.WindowSharded(w.X, w.windows, w.sigma, M=w.M, m=w.m, device=0)
    res = afs.cg_solve(afs.KernelSystem(op, w.beta), torch.from_numpy(w.y).cuda(), 1e-6, 1000)
    np.save(f"{out}.{rank}.npy", np.concatenate([[res.iterations, res.residual],
                                                 res.x.cpu().numpy()]))
    dist.destroy_process_group()


def test_window_sharded_cg_two_ranks(tmp_path):
    """Replicated-vector CG over window shards: same iteration count as the single-rank
    whole-solve graph, and both ranks hold the same x."""
    import paper_2111_10140_b200 as afs

    out = str(tmp_path / "wcg")
    _run(_cg_window_worker, out)
    w = _c2_small()
    op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                                 afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                 deterministic=True)
    ref = afs.cg_solve(afs.KernelSystem(op, w.beta), w.y, 1e-6, 1000)
    got = [np.load(f"{out}.{r}.npy") for r in range(2)]
    np.testing.assert_array_equal(got[0], got[1])
    err = np.linalg.norm(got[0][2:] - ref.x) / np.linalg.norm(ref.x)
    print(f"window-sharded CG: it {int(got[0][0])} vs {ref.iterations}; |x - x_1rank| {err:.2e}")
    assert abs(int(got[0][0]) - ref.iterations) <= 1
    assert err < 1e-8


def _cg_point_worker(rank, world, port, out):
    torch, dist = _init(rank, world, port)
    import paper_2111_10140_b200 as afs
    from paper_2111_10140_b200.distributed import CudaPointBackend

    w = _c4_small()
    y = np.sin(7.0 * w.X).sum(axis=1)
    shard = np.array_split(np.arange(w.N), world)[rank]
    be = CudaPointBackend(w.X[shard], [(0, 1, 2)], w.sigma, M=w.M, m=w.m, device=0)
    sys_ = afs.KernelSystem(afs.PointSharded(be), 50.0)
    res = afs.cg_solve(sys_, torch.from_numpy(y[shard].copy()).cuda(), 1e-8, 500)
    np.save(f"{out}.{rank}.npy", np.concatenate([[res.iterations, res.residual],
                                                 res.x.cpu().numpy()]))
    dist.destroy_process_group()


def test_point_sharded_cg_two_ranks(tmp_path):
    """Row-sharded CG with scalar all-reduces: the stacked shards equal the single-rank
    solve at the same iteration count (beta = 50 keeps the clustered C4 system well
    conditioned, so roundoff-level differences are not amplified)."""
    import paper_2111_10140_b200 as afs

    out = str(tmp_path / "pcg")
    _run(_cg_point_worker, out)
    w = _c4_small()
    y = np.sin(7.0 * w.X).sum(axis=1)
    op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                                 afs.PeriodizationConfig(coeff_grid=w.M), strict=False)
    ref = afs.cg_solve(afs.KernelSystem(op, 50.0), y, 1e-8, 500)
    parts = [np.load(f"{out}.{r}.npy") for r in range(2)]
    assert parts[0][0] == parts[1][0] and parts[0][1] == parts[1][1]
    x = np.concatenate([p[2:] for p in parts])
    err = np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
    print(f"point-sharded CG: it {int(parts[0][0])} vs {ref.iterations}; |x - x_1rank| {err:.2e}")
    assert abs(int(parts[0][0]) - ref.iterations) <= 1
    assert err < 1e-8
