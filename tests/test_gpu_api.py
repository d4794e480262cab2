"""Boundary features of the reference API on the GPU:
FastsumOperator.apply_complex / .source_plan / .target_plan against the reference's
own outputs (tests/golden/golden_complex.npz, make_golden_full.py `complex`), and
reentrant apply: concurrent callers on one plan (workspace clones, api.cu) get the
results of serial calls."""

import os
import sys
import threading

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from cases import FASTSUM_CASES, fastsum_inputs  # noqa: E402


@pytest.fixture(scope="module")
def afs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_10140_b200 as afs_mod

    return afs_mod


@pytest.fixture(scope="module")
def gc():
    with np.load(os.path.join(HERE, "golden", "golden_complex.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", FASTSUM_CASES[:7], ids=[c[0] for c in FASTSUM_CASES[:7]])
def test_apply_complex_matches_reference(afs, gc, case):
    tag, d, M, m, os_, sigma, N, n_tgt = case
    X, Z, alpha = fastsum_inputs(tag, d, N, n_tgt)
    op = afs.FastsumOperator(afs.GaussianKernel(sigma), afs.PeriodizationConfig(coeff_grid=M), X, Z,
                             afs.AccuracyProfile("t", os_, m))
    calpha = alpha + 1j * np.random.default_rng(len(tag)).standard_normal(N)
    got_r = op.apply_complex(alpha)
    got_c = op.apply_complex(calpha)
    e_r = rel_l2(got_r, gc[tag + "_real"])
    e_c = rel_l2(got_c, gc[tag + "_cplx"])
    # the real part is the fused apply path's result
    e_apply = rel_l2(op.apply(alpha), gc[tag + "_real"].real)
    print(f"{tag}: apply_complex real {e_r:.2e} complex {e_c:.2e}; apply vs Re {e_apply:.2e}")
    assert e_r < 1e-10 and e_c < 1e-10 and e_apply < 1e-10
    assert op.source_plan.node_count == N
    assert (op.target_plan is None) == (Z is None)
    if Z is not None:
        assert op.target_plan.node_count == n_tgt


def test_apply_complex_rejects_bad_shape(afs):
    X, _, alpha = fastsum_inputs("fs_d1_M32_m4", 1, 50, 0)
    op = afs.FastsumOperator(afs.GaussianKernel(0.3), afs.PeriodizationConfig(coeff_grid=16), X)
    with pytest.raises(afs.ShapeError):
        op.apply_complex(np.ones(49))


@pytest.mark.parametrize("deterministic", [False, True], ids=["atomic", "deterministic"])
def test_concurrent_applies_match_serial(afs, deterministic):
    """8 host threads, each on its own CUDA stream, share one plan; every result equals
    the serial apply of the same alpha (bitwise in deterministic mode)."""
    import torch
    from paper_2111_10140_b200 import synthetic

    w = synthetic.c3(N=200_000)
    op = afs.AnovaKernelOperator(w.X, w.windows[:6], w.sigma, afs.AccuracyProfile("b", 2.0, w.m),
                                 None, afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                 deterministic=deterministic)
    rng = np.random.default_rng(3)
    alphas = [torch.from_numpy(rng.standard_normal(w.N)).cuda() for _ in range(8)]
    serial = [op.apply(a).cpu().numpy() for a in alphas]
    results = [None] * 8
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    out = op.apply(alphas[k])
                s.synchronize()
                results[k] = out.cpu().numpy()
        except Exception as e:   # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k in range(8):
        if deterministic:
            np.testing.assert_array_equal(results[k], serial[k])
        else:
            assert rel_l2(results[k], serial[k]) < 1e-14


@pytest.mark.parametrize("sigma,M,d", [(0.05, 32, 2), (0.3, 16, 3), (0.1, 128, 3)])
def test_device_coefficient_fft_matches_pocketfft(afs, sigma, M, d):
    """c_hat with the plan-time transform on cuFFT (coeff_fft="device", row f2) against the
    reference-identical pocketfft path: roundoff-level agreement."""
    from paper_2111_10140_b200.spectrum import regularize_kernel

    cfg = afs.PeriodizationConfig(coeff_grid=M)
    host = regularize_kernel(afs.GaussianKernel(sigma), cfg, d)
    dev = regularize_kernel(afs.GaussianKernel(sigma), cfg, d, fft="device")
    err = rel_l2(dev, host)
    print(f"c_hat sigma={sigma} M={M} d={d}: device vs pocketfft rel l2 {err:.2e}")
    assert err < 1e-14


def test_device_coefficient_fft_operator_matches_reference(afs, golden):
    from paper_2111_10140_b200 import synthetic

    w = synthetic.c3(N=1500)
    op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                                 afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                 coeff_fft="device")
    err = rel_l2(op.apply(w.alpha), golden["c3s_out"])
    print(f"C3s with device c_hat: rel l2 {err:.2e}")
    assert err < 1e-10


def test_anova_operators_are_per_window_fastsum_operators(afs):
    """operators[l] of an ANOVA operator behaves like the reference's FastsumOperator on the
    window's columns (anova.py:163-172): same scaling, and apply equals the oracle's
    single-window fast sum; the weighted sum of the terms equals the ANOVA apply."""
    from oracle import fastsum_oracle as orc
    from paper_2111_10140_b200 import synthetic

    w = synthetic.c1(N=2000)
    Z = np.random.default_rng(2).standard_normal((500, 9))
    op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("c1", 2.0, 2),
                                 targets=Z, config=afs.PeriodizationConfig(coeff_grid=32))
    total = np.zeros(500)
    for eta, win, term in zip(op.windows.weights, w.windows, op.operators):
        got = term.apply(w.alpha)
        ref = orc.fastsum_apply(w.X[:, list(win)], w.alpha, w.sigma, 32, 2, 2.0,
                                Z=Z[:, list(win)])
        assert rel_l2(got, ref) < 1e-10
        assert term.source_plan.node_count == 2000 and term.target_plan.node_count == 500
        total += eta * got
    assert rel_l2(op.apply(w.alpha), total) < 1e-14
