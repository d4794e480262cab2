"""The GPU NfftPlan against the contract the reference's own NFFT suite pins
(pkg/tests/test_nfft.py): known answers, exact zeros, fast vs direct
sums per accuracy profile, the accuracy ladder, linearity, and cost growth.
The direct sums are the oracle's (oracle/fastsum_oracle.py, numpy), so these
checks are independent of the GPU code."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def afs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_10140_b200 as afs_mod

    return afs_mod


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_forward_constant_coefficients_known_answer(afs):
    """f_hat = 1 on I_4 at x = 0 sums to 4 (test_nfft.py:66-69 kind)."""
    plan = afs.NfftPlan((4,), np.array([[0.0]]), "fine")
    assert abs(plan.forward(np.ones(4))[0] - 4.0) < 1e-8


def test_adjoint_single_node_at_origin_known_answer(afs):
    """c = 1 at x = 0 gives f_hat_k = 1 for every k (test_nfft.py:89-92 kind)."""
    plan = afs.NfftPlan((8,), np.array([[0.0]]), "fine")
    np.testing.assert_allclose(plan.adjoint(np.ones(1)), np.ones(8), atol=1e-9)


def test_zero_inputs_give_exact_zeros(afs):
    rng = np.random.default_rng(4)
    plan = afs.NfftPlan((8, 8), rng.uniform(-0.5, 0.5, (30, 2)))
    assert np.all(plan.forward(np.zeros(64)) == 0.0)
    assert np.all(plan.adjoint(np.zeros(30)) == 0.0)


@pytest.mark.parametrize("profile,bar", [("rough", 1e-3), ("default", 1e-6), ("fine", 1e-9)])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_profiles_meet_their_error_targets(afs, profile, bar, d):
    """Fast vs direct transforms per profile (test_nfft.py:79-86, 101-107, 137-145)."""
    from oracle import fastsum_oracle as orc

    rng = np.random.default_rng(10 * d + len(profile))
    M = 16 if d < 3 else 8
    X = rng.uniform(-0.5, 0.5, size=(200, d))
    f = rng.standard_normal(M ** d) + 1j * rng.standard_normal(M ** d)
    c = rng.standard_normal(200) + 1j * rng.standard_normal(200)
    plan = afs.NfftPlan((M,) * d, X, profile)
    ef = _rel(plan.forward(f), orc.ndft_forward([M] * d, X, f))
    ea = _rel(plan.adjoint(c), orc.ndft_adjoint([M] * d, X, c))
    print(f"d={d} {profile}: forward {ef:.2e} adjoint {ea:.2e} (target {bar:g})")
    assert ef < bar and ea < bar


def test_accuracy_ladder_is_monotone(afs):
    """rough > default > fine error (test_nfft.py:124-134)."""
    from oracle import fastsum_oracle as orc

    rng = np.random.default_rng(12)
    X = rng.uniform(-0.5, 0.5, size=(300, 2))
    f = rng.standard_normal(256) + 1j * rng.standard_normal(256)
    ref = orc.ndft_forward([16, 16], X, f)
    errs = [_rel(afs.NfftPlan((16, 16), X, p).forward(f), ref) for p in ("rough", "default", "fine")]
    print("ladder", errs)
    assert errs[0] > errs[1] > errs[2]


def test_linearity(afs):
    """forward(a f + b g) = a forward(f) + b forward(g) (test_nfft.py:148-158)."""
    rng = np.random.default_rng(13)
    plan = afs.NfftPlan((16, 16, 16), rng.uniform(-0.5, 0.5, (500, 3)))
    f, g = (rng.standard_normal(16 ** 3) + 1j * rng.standard_normal(16 ** 3) for _ in range(2))
    a, b = 0.7 - 0.2j, -1.3 + 0.5j
    lhs = plan.forward(a * f + b * g)
    rhs = a * plan.forward(f) + b * plan.forward(g)
    assert _rel(lhs, rhs) < 1e-12


def test_forward_cost_grows_at_most_linearly(afs):
    """Wall time vs N over 2^14 .. 2^20 nodes: log-log slope <= 1.15 (test_nfft.py:220-237)."""
    rng = np.random.default_rng(14)
    f = rng.standard_normal(32 ** 2) + 1j * rng.standard_normal(32 ** 2)
    Ns, ts = [], []
    for e in range(14, 21, 2):
        N = 1 << e
        plan = afs.NfftPlan((32, 32), rng.uniform(-0.5, 0.5, (N, 2)))
        plan.forward(f)
        t0 = time.perf_counter()
        for _ in range(3):
            plan.forward(f)
        ts.append((time.perf_counter() - t0) / 3)
        Ns.append(N)
    slope = np.polyfit(np.log(Ns), np.log(ts), 1)[0]
    print("times", dict(zip(Ns, ts)), "slope", slope)
    assert slope <= 1.15


@pytest.mark.parametrize("bw", [(16, 8), (6, 12, 8), (4, 16)])
def test_unequal_bandwidths_match_direct_sums(afs, bw):
    """Unequal bandwidths (nfft.py:72-99 allows them) are embedded in the largest one; both
    transforms against the oracle's direct sums at the profile's accuracy, and the adjoint
    identity <forward(f), c> = <f, adjoint(c)> to roundoff of that accuracy."""
    from oracle import fastsum_oracle as orc

    rng = np.random.default_rng(sum(bw))
    d = len(bw)
    n_modes = int(np.prod(bw))
    X = rng.uniform(-0.5, 0.5, size=(150, d))
    f = rng.standard_normal(n_modes) + 1j * rng.standard_normal(n_modes)
    c = rng.standard_normal(150) + 1j * rng.standard_normal(150)
    plan = afs.NfftPlan(bw, X, "fine")
    fwd, adj = plan.forward(f), plan.adjoint(c)
    assert adj.shape == (n_modes,)
    e_f = _rel(fwd, orc.ndft_forward(list(bw), X, f))
    e_a = _rel(adj, orc.ndft_adjoint(list(bw), X, c))
    print(f"bandwidths {bw}: forward {e_f:.2e}, adjoint {e_a:.2e}")
    assert e_f < 1e-9 and e_a < 1e-9
    lhs, rhs = np.vdot(c, fwd), np.vdot(adj, f)
    assert abs(lhs - rhs) < 1e-8 * abs(lhs)
