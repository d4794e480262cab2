"""Stage breakdown for small configs (launch-bound regime): C1 and C2 matvecs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_10140_b200 as afs  # noqa: E402
from paper_2111_10140_b200 import synthetic  # noqa: E402

for name in ("C1", "C2"):
    if name == "C1":
        w = synthetic.c1()
        op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("c1", 2.0, 2),
                                     config=afs.PeriodizationConfig(coeff_grid=32))
        vec = w.alpha
    else:
        w = synthetic.c2(N=100_000, n_test=10)
        op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, "default")
        vec = w.y
    p = op._plan
    a = torch.from_numpy(vec).cuda()[None, :].contiguous()
    o = torch.empty_like(a)
    for _ in range(3):
        p.apply_device(a, o, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        p.apply_device(a, o, 1)
    torch.cuda.synchronize()
    graph_ms = (time.perf_counter() - t0) / 20 * 1e3
    p.set_profiling(True)
    for _ in range(5):
        p.apply_device(a, o, 1)
    st = p.stage_times()
    p.set_profiling(False)
    print(name, f"graph apply {graph_ms:.3f} ms wall;", {k: (v / 5 if k != "applies" else v) for k, v in st.items()},
          "info", p.info())
