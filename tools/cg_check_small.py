import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2111_10140_b200 as afs
from paper_2111_10140_b200 import synthetic
from oracle import fastsum_oracle as orc
w2 = synthetic.c2(N=800, n_test=10)
op = afs.AnovaKernelOperator(w2.X, w2.windows, w2.sigma, "default", deterministic=True)
v = np.random.default_rng(0).standard_normal(800)
y = op.apply(v)
ref = orc.anova_apply(w2.X, w2.windows, v, w2.sigma, w2.M, w2.m)
print("matvec rel err", np.linalg.norm(y-ref)/np.linalg.norm(ref), "checksum", repr(float(y.sum())))
for tol in (1e-6, 2e-6):
    res = afs.cg_solve(afs.KernelSystem(op, w2.beta), w2.y, tol=tol, maxiter=50)
    print(tol, res.iterations, res.residual)
