"""C2 matvec loop for ncu captures of the spectral line passes (3-D windows, n=128)."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2111_10140_b200 as afs
from paper_2111_10140_b200 import synthetic
w = synthetic.c2(N=100_000, n_test=10)
op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, "default")
p = op._plan
a = torch.from_numpy(w.y).cuda()[None, :].contiguous()
o = torch.empty_like(a)
for _ in range(3):
    p.apply_device(a, o, 1)
torch.cuda.synchronize()
