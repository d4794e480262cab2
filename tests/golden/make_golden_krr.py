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


def krr_inputs(seed=31, n=700, n_test=300, d=7):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n + n_test, d)) * rng.uniform(0.5, 3.0, size=d) + rng.normal(size=d)
    w = rng.normal(size=d)
    y = np.where(np.sin(X) @ w + 0.2 * rng.normal(size=n + n_test) >= 0, 1, -1)
    return X[:n], y[:n], X[n:], y[n:]


def main():
    X, y, Xt, yt = krr_inputs()
    cfg = KrrConfig(sigma=1.5, lam=0.5, cg_tol=1e-8, cg_maxiter=300)
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
