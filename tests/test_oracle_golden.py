"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py runs /root/reference's nfftkrr)."""

import json
import sys
import os

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fastsum_oracle as orc
from paper_2111_10140_b200 import synthetic

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from cases import FASTSUM_CASES, fastsum_inputs  # noqa: E402

PROFILES = {"rough": (1.5, 3), "default": (2.0, 4), "fine": (2.0, 6)}


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("prof", ["rough", "default", "fine"])
def test_nfft_forward_adjoint_match_reference(golden, d, prof):
    key = f"nfft_d{d}_{prof}"
    M = 16 if d < 3 else 8
    os_, m = PROFILES[prof]
    geo = orc.NodeGeometry(golden[key + "_x"], M, m, os_)
    assert rel_l2(geo.forward(golden[key + "_fhat"]), golden[key + "_fwd"]) < 1e-13
    assert rel_l2(geo.adjoint(golden[key + "_c"]), golden[key + "_adj"]) < 1e-13


@pytest.mark.parametrize("sigma,M,d", [(0.1, 16, 1), (0.05, 32, 2), (0.3, 16, 3), (2.0, 8, 3)])
def test_kernel_coefficients_match_reference(golden, sigma, M, d):
    ref = golden[f"coef_s{sigma}_M{M}_d{d}"]
    got = orc.kernel_coefficients(sigma, M, d)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("case", FASTSUM_CASES, ids=[c[0] for c in FASTSUM_CASES])
def test_fastsum_matches_reference(golden, case):
    tag, d, M, m, os_, sigma, N, n_tgt = case
    X, Z, alpha = fastsum_inputs(tag, d, N, n_tgt)
    np.testing.assert_array_equal(X, golden[tag + "_X"])
    got = orc.fastsum_apply(X, alpha, sigma, M, m, os_, Z)
    assert rel_l2(got, golden[tag + "_out"]) < 1e-12


def test_c1_anova_matches_reference(golden):
    w = synthetic.c1()
    got = orc.anova_apply(w.X, w.windows, w.alpha, w.sigma, w.M, w.m)
    assert rel_l2(got, golden["c1_out"]) < 1e-12


def test_c3_c4_c5_small_match_reference(golden):
    w3 = synthetic.c3(N=1500)
    assert rel_l2(orc.anova_apply(w3.X, w3.windows, w3.alpha, w3.sigma, w3.M, w3.m),
                  golden["c3s_out"]) < 1e-12
    w4 = synthetic.c4(N=2000, R=3)
    for r in range(3):
        got = orc.anova_apply(w4.X, w4.windows, w4.alpha[:, r], w4.sigma, w4.M, w4.m)
        assert rel_l2(got, golden["c4s_out"][:, r]) < 1e-12
    w5 = synthetic.c5(N=2000)
    assert rel_l2(orc.anova_apply(w5.X, w5.windows, w5.alpha, w5.sigma, w5.M, w5.m),
                  golden["c5s_out"]) < 1e-12


def test_c2_cg_matches_reference(golden):
    w = synthetic.c2(N=1200, n_test=400)
    apply = lambda v: orc.anova_apply(w.X, w.windows, v, w.sigma, w.M, w.m) + w.beta * v
    assert rel_l2(apply(w.y) - w.beta * w.y, golden["c2s_apply_y"]) < 1e-12
    x, it, res, conv = orc.cg_solve(apply, w.y, tol=1e-6, maxiter=200)
    assert abs(it - int(golden["c2s_iters"])) <= 1
    assert rel_l2(x, golden["c2s_x"]) < 1e-8
    dec = orc.anova_apply(w.X, w.windows, x, w.sigma, w.M, w.m, Z=w.Z)
    assert rel_l2(dec, golden["c2s_decision"]) < 1e-8


def test_golden_meta_records_versions(golden):
    meta = json.loads(str(golden["meta_json"]))
    assert "numpy" in meta and "scipy" in meta
