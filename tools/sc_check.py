"""GPU check of the sub-cell 2-D kernels: every 2-D m = 4 golden case with the layout forced
(AFS_SC=2), the default choice and the half-cell kernels (AFS_SC=0), multi-RHS, targets,
deterministic mode.   python tools/sc_check.py"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(REPO, "tests", "golden")
CODE = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2111_10140_b200 as afs
from paper_2111_10140_b200 import synthetic
from cases import FASTSUM_CASES, fastsum_inputs
g = dict(np.load(os.path.join(%r, "golden.npz")))
res = {}
for tag, d, M, m, os_, sigma, N, n_tgt in FASTSUM_CASES:
    if d != 2 or m != 4:
        continue
    X, Z, alpha = fastsum_inputs(tag, d, N, n_tgt)
    op = afs.FastsumOperator(afs.GaussianKernel(sigma), afs.PeriodizationConfig(coeff_grid=M), X, Z,
                             afs.AccuracyProfile("t", os_, m))
    got = op.apply(alpha)
    res[tag] = float(np.linalg.norm(got - g[tag + "_out"]) / np.linalg.norm(g[tag + "_out"]))
w = synthetic.c3(N=1500)
op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False)
got = op.apply(w.alpha)
res["c3s"] = float(np.linalg.norm(got - g["c3s_out"]) / np.linalg.norm(g["c3s_out"]))
# multi-RHS, targets, determinism on a dense window
rng = np.random.default_rng(5)
N = 200_000
X = rng.uniform(-1, 1, size=(N, 2)); Z = rng.uniform(-1, 1, size=(50_000, 2))
A = rng.standard_normal((N, 3))
op = afs.AnovaKernelOperator(X, [(0, 1)], 0.4, afs.AccuracyProfile("t", 2.0, 4), Z,
                             afs.PeriodizationConfig(coeff_grid=32), strict=False, max_rhs=3)
out3 = op.apply(A)
one = op.apply(A[:, 1])
res["rhs"] = float(np.abs(one - out3[:, 1]).max() / np.abs(one).max())
res["_out3_sum"] = float(np.abs(out3).sum())
opd = afs.AnovaKernelOperator(X, [(0, 1)], 0.4, afs.AccuracyProfile("t", 2.0, 4), Z,
                              afs.PeriodizationConfig(coeff_grid=32), strict=False, max_rhs=3,
                              deterministic=True)
d1 = opd.apply(A[:, 0]); d2 = opd.apply(A[:, 0])
res["det_equal"] = float(np.array_equal(d1, d2))
res["det_vs_atomic"] = float(np.linalg.norm(d1 - out3[:, 0]) / np.linalg.norm(d1))
print(json.dumps(res))
""" % (REPO, GOLD, GOLD)

ref = None
for mode in ("2", "0", None):
    env = dict(os.environ)
    env.pop("AFS_SC", None)
    if mode is not None:
        env["AFS_SC"] = mode
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    if out.returncode != 0:
        print("AFS_SC=%s FAILED\n%s" % (mode, out.stderr[-3000:]))
        continue
    res = json.loads(out.stdout.strip().splitlines()[-1])
    print("AFS_SC=%s" % mode, json.dumps(res))
