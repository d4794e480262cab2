"""A/B of per-window kernel times on the C3 recipe (profiling mode), for library variants:
    AFS_LIB=build_variants/libanovafs_X.so python tools/ab_windows.py --windows 0,3 --applies 5
prints mean spread / gather ms per window."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--windows", default="0,3,4")
ap.add_argument("--applies", type=int, default=5)
ap.add_argument("--config", default="C3")
a = ap.parse_args()
w = synthetic.c3(N=a.n) if a.config == "C3" else synthetic.c5(N=a.n)
idx = [int(x) for x in a.windows.split(",")]
wins = [w.windows[i] for i in idx]
op = afs.AnovaKernelOperator(w.X, wins, w.sigma, afs.AccuracyProfile("p", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                             weights=[1.0 / w.P] * len(wins))
alpha = torch.from_numpy(w.alpha).cuda()[None, :].contiguous()
out = torch.empty_like(alpha)
plan = op._plan
plan.apply_device(alpha, out, 1)
torch.cuda.synchronize()
plan.set_profiling(True)
for _ in range(a.applies):
    plan.apply_device(alpha, out, 1)
torch.cuda.synchronize()
sp, ga = plan.window_times(reset=True)
print(json.dumps({"lib": os.environ.get("AFS_LIB", "main"), "windows": wins,
                  "spread_ms": [t / a.applies for t in sp], "gather_ms": [t / a.applies for t in ga],
                  "checksum": float(out.double().abs().sum())}))
