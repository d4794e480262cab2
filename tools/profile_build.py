"""Plan-build breakdown (host validation, bbox, c_hat/multipliers, upload, native plan):

    python tools/profile_build.py [--config C3|C2|C4] [--n N]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import operators, spectrum, synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--n", type=int, default=None)
a = ap.parse_args()
kw = {} if a.n is None else {"N": a.n}
w = {"C3": synthetic.c3, "C2": synthetic.c2, "C4": synthetic.c4}[a.config](**kw)
X = w.X
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
T = {}
t = time.perf_counter()
Xm = operators._as_matrix(X, "X")
T["validate"] = time.perf_counter() - t
t = time.perf_counter()
lo, hi = operators._all_columns_minmax(Xm)
T["minmax"] = time.perf_counter() - t
cfg = afs.PeriodizationConfig(coeff_grid=w.M)
prof = afs.AccuracyProfile("p", 2.0, w.m)
t = time.perf_counter()
for win in w.windows:
    c, s = operators.bbox_scaling(lo[list(win)], hi[list(win)], cfg)
    co = spectrum.regularize_kernel(afs.GaussianKernel(w.sigma).rescaled(s), cfg, len(win))
    spectrum.window_multiplier(co, w.M, prof.grid_size(w.M), w.m)
T["chat+mult"] = time.perf_counter() - t
t = time.perf_counter()
Xd = torch.from_numpy(Xm).to("cuda")
torch.cuda.synchronize()
T["upload"] = time.perf_counter() - t
del Xd
t = time.perf_counter()
op = afs.AnovaKernelOperator(X, w.windows, w.sigma, prof, None, cfg, strict=False,
                             weights=[1.0 / w.P] * w.P, max_rhs=getattr(w, "R", 1))
torch.cuda.synchronize()
T["operator_total"] = time.perf_counter() - t
print({k: round(v, 4) for k, v in T.items()}, "N", w.N, "P", w.P)
