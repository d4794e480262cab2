"""Dense oracles and bench-mvm (paper_2111_10140_b200/harness.py) against the reference's
formulas (fastsum.py:162-179, nfft.py:263-300, cli.py:295-369): CPU runs use torch on the
host; the bench-mvm run is a GPU test."""

import csv
import json
import os

import numpy as np
import pytest

import paper_2111_10140_b200 as afs
from paper_2111_10140_b200 import harness


def _numpy_direct_sum(sigma, X, Z, a):
    # fastsum.py:162-179, restated
    sq_x = (X * X).sum(axis=1)
    d2 = (Z * Z).sum(axis=1)[:, None] + sq_x[None, :] - 2.0 * (Z @ X.T)
    np.maximum(d2, 0.0, out=d2)
    return np.exp(-(np.sqrt(d2) / sigma) ** 2) @ a


def test_direct_sum_matches_restatement():
    rng = np.random.default_rng(5)
    X, Z, a = rng.normal(size=(700, 3)), rng.normal(size=(300, 3)), rng.normal(size=700)
    got = afs.direct_sum(afs.GaussianKernel(0.7), X, Z, a, chunk=128, device="cpu")
    want = _numpy_direct_sum(0.7, X, Z, a)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
    with pytest.raises(afs.ShapeError):
        afs.direct_sum(afs.GaussianKernel(0.7), X, Z[:, :2], a, device="cpu")
    with pytest.raises(afs.ShapeError):
        afs.direct_sum(afs.GaussianKernel(0.7), X, Z, a[:-1], device="cpu")


def test_ndft_direct_known_answers_and_adjointness():
    # test_nfft.py:44-54 style: constant coefficients, a single mode
    rng = np.random.default_rng(9)
    x = rng.uniform(-0.5, 0.5, size=(50, 2))
    f = afs.ndft_direct((2, 2), x, np.ones(4), device="cpu")   # modes {-1, 0}^2
    np.testing.assert_allclose(f, np.prod(1.0 + np.exp(-2j * np.pi * x), axis=1), atol=1e-13)
    fh = np.zeros((4, 4), dtype=complex)
    fh[2 + 1, 2 - 2] = 1j                       # mode k = (1, -2)
    got = afs.ndft_direct((4, 4), x, fh, device="cpu")
    want = 1j * np.exp(2j * np.pi * (x[:, 0] * 1 - 2 * x[:, 1]))
    np.testing.assert_allclose(got, want, atol=1e-14)
    # adjointness <A f, c> = <f, A^H c>
    M = (8, 6)
    fh = rng.normal(size=48) + 1j * rng.normal(size=48)
    c = rng.normal(size=50) + 1j * rng.normal(size=50)
    lhs = np.vdot(c, afs.ndft_direct(M, x, fh, device="cpu"))
    rhs = np.vdot(afs.ndft_adjoint_direct(M, x, c, device="cpu"), fh)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(fh) * np.linalg.norm(c) * 48
    with pytest.raises(afs.ShapeError):
        afs.ndft_direct(M, x, fh[:-1], device="cpu")
    with pytest.raises(afs.ValidationError):
        afs.ndft_direct(M, x + 1.0, fh, device="cpu")


def test_bench_mvm_validates_n_list(tmp_path):
    with pytest.raises(afs.ValidationError):
        afs.bench_mvm([100, 50], out=str(tmp_path / "x.csv"))
    with pytest.raises(afs.ValidationError):
        afs.bench_mvm([0], out=str(tmp_path / "x.csv"))


@pytest.mark.gpu
def test_bench_mvm_on_gpu(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out, rep = tmp_path / "b.csv", tmp_path / "r.json"
    rows = afs.bench_mvm([300, 3000], d=3, sigma=1.0, profile="default", runs=2, seed=0,
                         out=str(out), report_out=str(rep), verbose=False)
    assert [r["direct_ran"] for r in rows] == [True, True]
    # the fast summation approximates the dense kernel to the profile's accuracy
    assert all(r["rel_error"] < 1e-4 for r in rows)
    with open(out) as fh:
        table = list(csv.reader(fh))
    assert table[0] == ["n", "t_direct", "t_fast", "rel_error", "direct_ran"]
    assert [int(t[0]) for t in table[1:]] == [300, 3000]
    payload = json.load(open(rep))
    assert payload["format"] == "run-report/1" and payload["command"] == "bench-mvm"
    assert set(payload["mvm_relative_errors"]) == {"300", "3000"}
