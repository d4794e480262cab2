"""CPU checks of the host plan layer: the pruned real multiplier E and the
pass structure of the device spectral stage (csrc/spectral.cu), emulated in
numpy, must reproduce the reference's Re(forward(c_hat * adjoint(alpha))).
No GPU needed."""

import os
import sys

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fastsum_oracle as orc
from paper_2111_10140_b200 import (AccuracyProfile, GaussianKernel, PeriodizationConfig,
                                   ValidationError, WindowSet, regularize_kernel)
from paper_2111_10140_b200.spectrum import window_multiplier

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from cases import FASTSUM_CASES, fastsum_inputs  # noqa: E402


def _stencil(xs, n, m, b):
    nx = n * xs
    u = np.floor(nx)
    cells = u[:, None] + np.arange(1 - m, m + 1)[None, :]
    return np.mod(cells, n).astype(np.int64), orc.kb_window(nx[:, None] - cells, m, b)


def emulate_device(X, alpha, sigma, M, m, oversampling, Z=None):
    """numpy model of spread -> spectral passes -> gather as the kernels run them."""
    X = np.asarray(X, dtype=np.float64)
    d = X.shape[1]
    pts = X if Z is None else np.vstack([X, Z])
    lo, hi = pts.min(0), pts.max(0)
    diam = float(np.linalg.norm(hi - lo))
    scale = PeriodizationConfig().ball_radius / diam
    center = (lo + hi) / 2
    prof = AccuracyProfile("t", oversampling, m)
    n = prof.grid_size(M)
    b = np.pi * (2.0 - M / n)
    E = window_multiplier(regularize_kernel(GaussianKernel(sigma * scale),
                                            PeriodizationConfig(coeff_grid=M), d), M, n, m)
    H = M // 2 + 1

    def tensor(P):
        st = [_stencil((P[:, t] - center[t]) * scale, n, m, b) for t in range(d)]
        flat, w = st[0]
        for t in range(1, d):
            flat = (flat[:, :, None] * n + st[t][0][:, None, :]).reshape(len(P), -1)
            w = (w[:, :, None] * st[t][1][:, None, :]).reshape(len(P), -1)
        return flat, w

    flat, w = tensor(X)
    g = np.bincount(flat.ravel(), (alpha[:, None] * w).ravel(), minlength=n ** d)
    g = g.reshape((n,) * d)
    sym = (np.arange(M + 1) - M // 2) % n
    A = np.fft.fft(g, axis=-1)[..., :H]                     # real last axis -> half spectrum
    if d == 3:
        A = np.fft.fft(A, axis=1)[:, sym, :]                # middle axis, keep j in 0..M
    if d >= 2:
        F = np.fft.fft(A, axis=0)
        Y = np.zeros_like(F)
        Y[sym] = F[sym] * E                                 # fused first-axis multiply
        A = n * np.fft.ifft(Y, axis=0)
    else:
        A = A * E
    if d == 3:
        full = np.zeros((n, n, H), dtype=complex)
        full[:, sym, :] = A
        A = n * np.fft.ifft(full, axis=1)
    line = np.zeros(A.shape[:-1] + (n,), dtype=complex)
    line[..., :H] = A
    h = (n * np.fft.ifft(line, axis=-1)).real
    tflat, tw = tensor(X if Z is None else Z)
    return (h.ravel()[tflat] * tw).sum(1)


@pytest.mark.parametrize("case", FASTSUM_CASES, ids=[c[0] for c in FASTSUM_CASES])
def test_real_pipeline_matches_reference_golden(golden, case):
    tag, d, M, m, os_, sigma, N, n_tgt = case
    X, Z, alpha = fastsum_inputs(tag, d, N, n_tgt)
    got = emulate_device(X, alpha, sigma, M, m, os_, Z)
    assert rel_l2(got, golden[tag + "_out"]) < 1e-13


def test_multiplier_layout_shapes():
    c = np.ones((8, 8, 8))
    E = window_multiplier(c, 8, 16, 2)
    assert E.shape == (9, 9, 5)
    assert window_multiplier(np.ones((8, 8)), 8, 16, 2).shape == (9, 5)
    assert window_multiplier(np.ones(8), 8, 16, 2).shape == (5,)


def test_multiplier_is_centrally_symmetric():
    rng = np.random.default_rng(0)
    c = rng.random((8, 8))
    c = c + c[::-1, ::-1]  # interior symmetry does not matter; faces are what D_sym fixes
    E = window_multiplier(c, 8, 18, 3)
    # k_last = 0 column is symmetric in k0 (E(k0,0) = E(-k0,0))
    np.testing.assert_allclose(E[:, 0], E[::-1, 0], rtol=0, atol=1e-300)


def test_coefficients_match_reference_golden(golden):
    for sigma, M, d in ((0.1, 16, 1), (0.05, 32, 2), (0.3, 16, 3), (2.0, 8, 3)):
        ref = golden[f"coef_s{sigma}_M{M}_d{d}"]
        got = regularize_kernel(GaussianKernel(sigma), PeriodizationConfig(coeff_grid=M), d)
        # same profile samples and the same pocketfft transform (scipy.fft): bit-identical
        np.testing.assert_array_equal(got, ref)


def test_profile_grid_size_rule():
    assert AccuracyProfile("x", 2.0, 4).grid_size(64) == 128
    assert AccuracyProfile("x", 1.5, 3).grid_size(16) == 24
    assert AccuracyProfile("x", 1.5, 3).grid_size(2) == 6      # max(2m, ...)
    with pytest.raises(ValidationError):
        AccuracyProfile("x", 1.0, 4)
    with pytest.raises(ValidationError):
        AccuracyProfile("x", 2.0, 0)


def test_windowset_rules():
    WindowSet([(0, 1, 2), (3, 4)])
    with pytest.raises(ValidationError):
        WindowSet([(0, 1, 2), (2, 3, 4)])
    with pytest.raises(ValidationError):
        WindowSet([(0, 1), (2, 3, 4)])
    with pytest.raises(ValidationError):
        WindowSet([])
    assert WindowSet([(0, 1, 2), (3,)]).weights == (0.5, 0.5)


def _parse_inc_tables(path, shape):
    """Arrays of a generated csrc/*.inc table file, in file order."""
    import re

    text = open(path).read()
    tables = []
    for body in re.findall(r"AFS_KB_INIT\(\{(.*?)\}\)\);", text, flags=re.S):
        vals = [float(v) for v in re.findall(r"[-+]?\d+\.?\d*(?:[eE][-+]?\d+)?", body)]
        tables.append(np.array(vals).reshape(shape))
    return tables


def test_sub_cell_tables_reproduce_the_reference_window():
    """csrc/kb_sub.inc (tools/gen_kb_sub.py): on every sub-interval f in [s/16, (s+1)/16) the
    8-term Chebyshev series in t = 32 f - 2 s - 1 gives the reference's window value
    phi(f + 3 - o) (nfft.py:118-122) for every stencil offset, for both compile-time ratios
    n/M = 2 and 3/2; the reference formula itself carries ~3.5e-15 of the peak in fp64."""
    from oracle import fastsum_oracle as orc

    here = os.path.dirname(os.path.abspath(__file__))
    inc = os.path.join(os.path.dirname(here), "paper_2111_10140_b200", "csrc", "kb_sub.inc")
    tabs = _parse_inc_tables(inc, (16, 8, 8))
    assert len(tabs) == 2
    rng = np.random.default_rng(0)
    for tab, (M, n) in zip(tabs, ((64, 128), (64, 96))):
        b = orc.kb_shape(M, n)
        peak = float(orc.kb_window(np.array([0.0]), 4, b)[0])
        worst = 0.0
        for s in range(16):
            t = rng.uniform(-1.0, 1.0, size=64)
            f = (s + (t + 1.0) / 2.0) / 16.0
            T = np.cos(np.arange(8)[:, None] * np.arccos(t)[None, :])     # T_k(t)
            for o in range(8):
                got = tab[s, o] @ T
                want = orc.kb_window(f + 3 - o, 4, b)
                worst = max(worst, float(np.abs(got - want).max()) / peak)
        assert worst < 2e-14, worst
