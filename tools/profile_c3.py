"""Small driver for ncu captures: C3-recipe operator over a window subset.

    python tools/profile_c3.py --n 10000000 --windows 0,3 --applies 2
windows are indices into the C3 list (0-2 triples, 3-38 pairs)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--windows", default="all")
ap.add_argument("--applies", type=int, default=2)
ap.add_argument("--mode", default="poly")
ap.add_argument("--config", default="C3")
ap.add_argument("--rhs", type=int, default=1)
a = ap.parse_args()

if a.config == "C4":
    w = synthetic.c4(N=a.n, R=a.rhs)
else:
    w = synthetic.c3(N=a.n)
idx = list(range(w.P)) if a.windows == "all" else [int(x) for x in a.windows.split(",")]
wins = [w.windows[i] for i in idx]
op = afs.AnovaKernelOperator(w.X, wins, w.sigma, afs.AccuracyProfile("p", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                             weights=[1.0 / w.P] * len(wins), window_eval=a.mode, max_rhs=a.rhs)
alpha = torch.from_numpy(w.alpha.reshape(w.N, -1).T.copy()).cuda()
out = torch.empty((a.rhs, w.N), dtype=torch.float64, device="cuda")
plan = op._plan
torch.cuda.synchronize()
plan.set_profiling(True)
for _ in range(a.applies):
    t0 = time.perf_counter()
    plan.apply_device(alpha, out, a.rhs)
    torch.cuda.synchronize()
    print(f"apply {1e3 * (time.perf_counter() - t0):.2f} ms", plan.stage_times(reset=True))
