"""Stage and per-window breakdown of the C5 matvec (20 singles + 10 pairs, N=1M)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

w = synthetic.c5()
op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False)
p = op._plan
a = torch.from_numpy(w.y).cuda()[None, :].contiguous()
o = torch.empty_like(a)
for _ in range(3):
    p.apply_device(a, o, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    p.apply_device(a, o, 1)
e1.record()
torch.cuda.synchronize()
print("graph apply ms", e0.elapsed_time(e1) / 10)
p.set_profiling(True)
for _ in range(5):
    p.apply_device(a, o, 1)
st = p.stage_times()
sp, ga = p.window_times()
print({k: v / 5 for k, v in st.items()})
for i, win in enumerate(w.windows):
    print(win, round(sp[i] / 5, 4), round(ga[i] / 5, 4))
