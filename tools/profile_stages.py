"""Per-stage device times (profiling mode) of one config's apply:
    python tools/profile_stages.py --config c2"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--applies", type=int, default=10)
a = ap.parse_args()
gen = {"c2": synthetic.c2, "c3": synthetic.c3, "c5": synthetic.c5}[a.config]
w = gen(N=a.n) if a.n else gen()
op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False)
al = torch.from_numpy(w.y if w.y is not None else w.alpha).cuda()[None, :].contiguous()
out = torch.empty_like(al)
plan = op._plan
for _ in range(3):
    plan.apply_device(al, out, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.applies):
    plan.apply_device(al, out, 1)
e1.record()
torch.cuda.synchronize()
plan.set_profiling(True)
for _ in range(a.applies):
    plan.apply_device(al, out, 1)
torch.cuda.synchronize()
st = plan.stage_times(reset=True)
print(json.dumps({"config": a.config, "N": w.N, "ms_per_apply_graph": e0.elapsed_time(e1) / a.applies,
                  "stages_ms": {k: v / st["applies"] for k, v in st.items() if k != "applies"},
                  "info": plan.info()}))
