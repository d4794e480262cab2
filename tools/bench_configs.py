"""Secondary measurements for the other BASELINE configs (not the headline bench line):
C1 matvec, C2 CG fit (device-resident) + predict, C4 multi-RHS matvec, C5 matvec + CG.
Prints one JSON object per config.   python tools/bench_configs.py [--c4-n 10000000]"""
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


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def free_op(w, max_rhs=1):
    return afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("b", 2.0, w.m), None,
                                   afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                   max_rhs=max_rhs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4-n", type=int, default=10_000_000)
    ap.add_argument("--c2-n", type=int, default=100_000)
    ap.add_argument("--skip", default="")
    a = ap.parse_args()
    skip = set(a.skip.split(","))
    dev = torch.device("cuda", 0)

    if "C1" not in skip:
        w = synthetic.c1()
        op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, afs.AccuracyProfile("c1", 2.0, 2),
                                     config=afs.PeriodizationConfig(coeff_grid=32))
        al = torch.from_numpy(w.alpha).to(dev)[None, :].contiguous()
        out = torch.empty_like(al)
        ms = timed(lambda: op._plan.apply_device(al, out, 1), reps=50, warm=5)
        print(json.dumps({"config": "C1", "N": w.N, "P": w.P, "ms_per_matvec": ms,
                          "matvec_per_s": 1e3 / ms, "updates_per_s": w.N * w.P * 1e3 / ms}), flush=True)

    if "C2" not in skip:
        w = synthetic.c2(N=a.c2_n, n_test=20_000)
        t0 = time.perf_counter()
        op = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, "default")
        t_build = time.perf_counter() - t0
        al = torch.from_numpy(w.y).to(dev)[None, :].contiguous()
        out = torch.empty_like(al)
        ms = timed(lambda: op._plan.apply_device(al, out, 1), reps=20, warm=3)
        yd = torch.from_numpy(w.y).to(dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = afs.cg_solve(afs.KernelSystem(op, w.beta), yd, tol=1e-6, maxiter=200)
        torch.cuda.synchronize()
        t_cg = time.perf_counter() - t0
        t0 = time.perf_counter()
        pred = afs.AnovaKernelOperator(w.X, w.windows, w.sigma, "default", targets=w.Z)
        dec = pred.apply(res.x.cpu().numpy())
        t_pred = time.perf_counter() - t0
        print(json.dumps({"config": "C2", "N": w.N, "P": w.P, "ms_per_matvec": ms,
                          "plan_build_s": t_build, "cg_iterations": res.iterations,
                          "cg_converged": res.converged, "cg_residual": res.residual,
                          "cg_wall_s": t_cg, "ms_per_cg_iteration": 1e3 * t_cg / max(1, res.iterations),
                          "predict_wall_s_incl_build": t_pred, "n_test": w.Z.shape[0],
                          "decision_abs_mean": float(np.mean(np.abs(dec)))}),
              flush=True)

    if "C4" not in skip:
        w = synthetic.c4(N=a.c4_n, R=8)
        t0 = time.perf_counter()
        op = free_op(w, max_rhs=8)
        t_build = time.perf_counter() - t0
        al = torch.from_numpy(np.ascontiguousarray(w.alpha.T)).to(dev)
        out = torch.empty_like(al)
        ms = timed(lambda: op._plan.apply_device(al, out, 8), reps=3, warm=2)   # 2nd call captures the graph
        op._plan.set_profiling(True)
        op._plan.apply_device(al, out, 8)
        st = op._plan.stage_times()
        op._plan.set_profiling(False)
        # size-independent checks at full N: linearity (rhs 2 = rhs 0 + rhs 1) and symmetry
        # <K a0, a1> = <a0, K a1>
        al[2] = al[0] + al[1]
        op._plan.apply_device(al, out, 8)
        lin = float((out[2] - out[0] - out[1]).norm() / out[2].norm())
        sym = float(abs(torch.dot(out[0], al[1]) - torch.dot(al[0], out[1]))
                    / (out[0].norm() * al[1].norm()))
        print(json.dumps({"config": "C4", "N": w.N, "R": 8, "ms_per_matvec": ms,
                          "matvec_per_s": 1e3 / ms, "updates_per_s": w.N * 8 * 1e3 / ms,
                          "plan_build_s": t_build, "stages": st,
                          "linearity_rel": lin, "symmetry_rel": sym,
                          "device_peak_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
        del op, al, out

    if "C5" not in skip:
        w = synthetic.c5()
        op = free_op(w)
        al = torch.from_numpy(w.y).to(dev)[None, :].contiguous()
        out = torch.empty_like(al)
        ms = timed(lambda: op._plan.apply_device(al, out, 1), reps=10, warm=2)
        yd = torch.from_numpy(w.y).to(dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = afs.cg_solve(afs.KernelSystem(op, w.beta), yd, tol=1e-6, maxiter=200)
        torch.cuda.synchronize()
        t_cg = time.perf_counter() - t0
        print(json.dumps({"config": "C5", "N": w.N, "P": w.P, "ms_per_matvec": ms,
                          "matvec_per_s": 1e3 / ms, "updates_per_s": w.N * w.P * 1e3 / ms,
                          "cg_iterations": res.iterations, "cg_converged": res.converged,
                          "cg_residual": res.residual, "cg_wall_s": t_cg}), flush=True)


if __name__ == "__main__":
    main()
