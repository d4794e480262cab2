"""C4 spectral stage alone (n=256, 3-D window, R=8) for ncu: one plan at N=200k, a few
applies.  The spectral cost does not depend on N."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

w = synthetic.c4(N=200_000, R=8)
op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                             afs.PeriodizationConfig(coeff_grid=w.M), strict=False, max_rhs=8)
p = op._plan
a = torch.from_numpy(w.alpha.T.copy()).cuda().contiguous()
o = torch.empty_like(a)
for _ in range(3):
    p.apply_device(a, o, 8)
torch.cuda.synchronize()
p.set_profiling(True)
for _ in range(3):
    p.apply_device(a, o, 8)
print({k: v / 3 for k, v in p.stage_times().items()})
