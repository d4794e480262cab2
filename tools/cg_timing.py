"""CG timing on the C2 / C5 recipes (whole-solve graph), for A/B of the CG epilogue:
    python tools/cg_timing.py --config c2 --iters 200 [--det]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--det", action="store_true")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
w = synthetic.c2() if a.config == "c2" else synthetic.c5()
op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                             deterministic=a.det)
b = torch.from_numpy(w.y).cuda()
sysm = afs.KernelSystem(op, w.beta)
res = afs.cg_solve(sysm, b, 1e-6, a.iters)   # captures the graph
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    res = afs.cg_solve(sysm, b, 1e-6, a.iters)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
al = b[None, :].contiguous()
out = torch.empty_like(al)
for _ in range(3):
    op._plan.apply_device(al, out, 1)
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    op._plan.apply_device(al, out, 1)
e1.record()
torch.cuda.synchronize()
mv = e0.elapsed_time(e1) / 20
print(json.dumps({"config": a.config, "fused": os.environ.get("AFS_CG_FUSED", "1"), "det": a.det,
                  "iterations": res.iterations, "residual": res.residual,
                  "ms_per_solve": ms, "ms_per_iteration": ms / res.iterations, "ms_per_matvec": mv,
                  "x_checksum": float(res.x.abs().sum())}))
