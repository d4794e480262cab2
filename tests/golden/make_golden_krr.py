"""Golden vectors for the KRR wrappers (fit / decision_values / predict / model JSON) from the
REFERENCE itself.  Run here (needs /root/reference):  python tests/golden/make_golden_krr.py"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import nfftkrr  # noqa: E402  (the reference)
from nfftkrr import KrrConfig, decision_values, fit, mis_scores, predict  # noqa: E402
from nfftkrr.krr import model_to_dict  # noqa: E402

sys.path.insert(0, HERE)
from cases import krr_inputs  # noqa: E402




def main():
    X, y, Xt, yt = krr_inputs()
    cfg = KrrConfig(sigma=1.5, lam=0.5, cg_tol=1e-10, cg_maxiter=300)
    model = fit(X, y, cfg)
    doc = model_to_dict(model)
    g = {
        "mis_scores": mis_scores((X - X.mean(0)) / X.std(0), y).scores,
        "alpha": model.alpha,
        "iterations": np.array(model.cg_iterations),
        "windows_json": np.array(json.dumps(doc["windows"])),
        "decision": decision_values(model, Xt),
        "predict": predict(model, Xt),
        "model_json": np.array(json.dumps(doc)),
        "meta_json": np.array(json.dumps({"numpy": np.__version__,
                                          "reference": getattr(nfftkrr, "__version__", "?")})),
    }
    np.savez_compressed(os.path.join(HERE, "golden_krr.npz"), **g)
    print("iterations", model.cg_iterations, "windows", doc["windows"])


if __name__ == "__main__":
    main()
