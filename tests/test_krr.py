"""KRR wrappers around the hot path (fit / decision_values / predict / model JSON) against
the reference's own outputs (tests/golden/make_golden_krr.py)."""
import json
import os
import sys

import numpy as np
import pytest

from conftest import rel_l2

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from cases import krr_inputs  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_krr.npz")


@pytest.fixture(scope="module")
def gk():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def test_mis_and_windows_match_reference(gk):
    X, y, _, _ = krr_inputs()
    Xs = afs.zscore_apply(afs.zscore_fit(X), X)
    rep = afs.mis_scores(Xs, y)
    np.testing.assert_allclose(rep.scores, gk["mis_scores"], rtol=1e-12, atol=1e-15)
    ws = afs.build_windows(rep)
    assert ws.to_dict() == json.loads(str(gk["windows_json"]))


def test_model_json_roundtrip(gk):
    doc = json.loads(str(gk["model_json"]))
    model = afs.model_from_dict(doc)
    assert afs.model_to_dict(model) == doc
    with pytest.raises(afs.ValidationError):
        afs.model_from_dict(dict(doc, format="krr-model/0"))


def test_config_validation():
    with pytest.raises(afs.ValidationError):
        afs.KrrConfig(sigma=0)
    with pytest.raises(afs.ValidationError):
        afs.KrrConfig(cg_tol=1.5)


@pytest.mark.gpu
def test_fit_predict_match_reference(gk):
    X, y, Xt, yt = krr_inputs()
    cfg = afs.KrrConfig(sigma=1.5, lam=0.5, cg_tol=1e-10, cg_maxiter=300)
    model = afs.fit(X, y, cfg)
    assert abs(model.cg_iterations - int(gk["iterations"])) <= 1
    err = rel_l2(model.alpha, gk["alpha"])
    print(f"fit alpha rel {err:.2e}, iterations {model.cg_iterations} vs {int(gk['iterations'])}")
    assert err < 1e-8
    dec = afs.decision_values(model, Xt)
    assert rel_l2(dec, gk["decision"]) < 1e-8
    np.testing.assert_array_equal(afs.predict(model, Xt), gk["predict"])
    # the reference's own model file, evaluated on the GPU: matvec-level parity
    ref_model = afs.model_from_dict(json.loads(str(gk["model_json"])))
    assert rel_l2(afs.decision_values(ref_model, Xt), gk["decision"]) < 1e-10
