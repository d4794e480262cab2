#!/usr/bin/env python
"""Benchmark: ANOVA fast-summation matvecs/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the config the metric's roofline target is
quoted on): C3 — N=10,000,000 points, d=9 features U[-1/4,1/4), 3 triple
windows + 36 pair windows (P=39, eta=1/39), Gaussian sigma=0.5, M=64 (grid
n=128), m=4, one right-hand side, fp64.  One "step" = one full ANOVA matvec.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs one process per GPU (torchrun); windows are dealt to ranks by LPT on
their spread+gather cost and the N-vector partial results are summed with one
NCCL all-reduce per matvec.  Rank 0 prints ONE JSON line.

``--impl reference`` times the CPU oracle port of the reference path
(oracle/fastsum_oracle.py; the reference itself is pure Python and cannot be
built into oracle/_ref) on the host cores of this box, on a bounded sample
of the same workload (first-N rows recipe at N=--cpu-n), all host cores via a
process pool over windows; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ANOVA fast-sum matvecs/s"
UNIT = "matvec/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=10_000_000, help="points (C3 default 10M)")
    ap.add_argument("--cpu-n", type=int, default=50_000, help="CPU baseline sample size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--deterministic", action="store_true",
                    help="bit-reproducible fixed-point spread (afs_plan_set_deterministic)")
    return ap.parse_args()


def workload_config(N, P, m, M, n, extra=None):
    cfg = {
        "workload": f"C3: N={N:,} d=9 U[-1/4,1/4), 3 triples + 36 pairs (P={P}), sigma=0.5, "
                    f"M={M} (grid n={n}), m={m}, R=1, fp64",
        "N": N, "P": P, "M": M, "n": n, "m": m, "R": 1,
        "l2": "inputs larger than L2 (720 MB coordinates + 80 MB alpha + 80 MB out per matvec)",
    }
    if extra:
        cfg.update(extra)
    return cfg


def algorithmic_bytes(N, windows, n, R=1):
    """B = sum_l [(Nx+Nz)*8*d_l + Nx*8*R + Nz*8*R] + sum_l 32*R*n^d_l (Z=X)."""
    tot = 0
    spread = 0
    gather = 0
    for w in windows:
        d = len(w)
        sp = N * 8 * d + N * 8 * R + 8 * R * n ** d
        ga = N * 8 * d + N * 8 * R + 8 * R * n ** d
        spread += sp
        gather += ga
        tot += sp + ga + 16 * R * n ** d
    return tot, spread, gather


def lpt_assign(windows, N, m, world):
    """Longest-processing-time deal of windows to ranks on the modelled kernel time
    (distributed.window_costs)."""
    from paper_2111_10140_b200.distributed import lpt_assign as lpt, window_costs

    return lpt(window_costs(windows, N, m), world)


class ClockSampler:
    """SM clocks / power / clock-event (throttle) reasons sampled during the timed region:
    NVML every 10 ms in a thread (nvidia_ml_py), else nvidia-smi every 200 ms."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.thread = None
        self.rows = []
        self.source = None

    def _nvml_loop(self, nv, h):
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((float(sm), pw, int(rs)))
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        try:
            import threading

            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.stop = False
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            self.source = "nvml"
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.thread is not None:
            self.stop = True
            self.thread.join(timeout=2)
        elif self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.thread is not None and self.rows:
            reasons = sorted({k for _, _, rs in self.rows for k, bit in self.REASONS.items() if rs & bit})
            return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_sm,
                    "power_w_max": max(r[1] for r in self.rows), "samples": len(self.rows),
                    "source": "nvml, 10 ms", "reasons": reasons}
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None,
                "samples": len(rows), "source": "nvidia-smi, 200 ms", "reasons": reasons}


def measured_peak_hbm():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_fp64_peak():
    """Peak of the fp64 pipe on this pool: the larger of the DFMA microbenchmark
    (tools/fp64_peak.cu, profiles/r01_fp64_peak.txt) and the DMMA one (tools/dmma_peak.cu,
    profiles/r01_dmma_peak.txt; DFMA and DMMA share the pipe, DMMA issues 256 MACs at once)."""
    vals = []
    try:
        with open(os.path.join(REPO, "profiles", "r01_fp64_peak.txt")) as fh:
            vals += [(float(l.split("=")[1].split("TFLOP")[0]), "DFMA") for l in fh if "TFLOP/s" in l]
        with open(os.path.join(REPO, "profiles", "r01_dmma_peak.txt")) as fh:
            vals += [(float(l.split("total")[1].split("TFLOP")[0]), "DMMA m8n8k4")
                     for l in fh if "total" in l and "+DFMA" not in l]
    except Exception:
        pass
    if not vals:
        return 37.0, "nominal (B200 fp64 spec)"
    v, src = max(vals)
    return v, f"measured ({src} microbenchmark, profiles/r01_{'dmma' if 'DMMA' in src else 'fp64'}_peak.txt)"


def ncu_traffic(key):
    """dram read+write bytes per launch from a committed ncu --set full capture."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU side: oracle port timed on the host (never the product path)
# ---------------------------------------------------------------------------
_POOL_STATE = {}


def _cpu_window(i):
    from oracle import fastsum_oracle as orc

    st = _POOL_STATE
    w = st["windows"][i]
    return orc.fastsum_apply(st["X"][:, list(w)], st["alpha"], st["sigma"], st["M"], st["m"], 2.0)


def cpu_matvec_seconds(w, workers):
    """One oracle matvec of the sampled workload; windows summed in reference order."""
    from oracle import fastsum_oracle as orc

    t0 = time.perf_counter()
    if workers <= 1:
        out = orc.anova_apply(w.X, w.windows, w.alpha, w.sigma, w.M, w.m)
    else:
        import multiprocessing as mp

        _POOL_STATE.update(X=w.X, alpha=w.alpha, windows=w.windows, sigma=w.sigma, M=w.M, m=w.m)
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            parts = pool.map(_cpu_window, range(len(w.windows)))
        out = np.zeros(w.N)
        for s in parts:
            out += (1.0 / len(w.windows)) * s
    return time.perf_counter() - t0, out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2111_10140_b200 import synthetic

    w = synthetic.c3(N=args.cpu_n)
    cores = os.cpu_count() or 1
    workers = min(cores, len(w.windows))
    for _ in range(args.warmup):
        cpu_matvec_seconds(w, workers)
    times = [cpu_matvec_seconds(w, workers)[0] for _ in range(args.steps)]
    t = float(np.mean(times))
    scale = args.n / args.cpu_n
    value = 1.0 / (t * scale)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * scale * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.n, len(w.windows), w.m, w.M, 2 * w.M),
        "updates_per_s": w.N * len(w.windows) / t,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"C3 recipe at N={args.cpu_n:,} (all 39 windows), one matvec "
                                   f"per step, windows dealt over {workers} processes; matvecs/s "
                                   f"extrapolated linearly to N={args.n:,}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        # test hook for the multi-rank code path on a single-GPU box: AFS_BENCH_SHARE_GPU=1
        # maps every rank onto the visible devices round-robin and uses gloo (host-staged
        # all-reduce; no rank's kernels wait on another's).  Never used for reported numbers.
        share = os.environ.get("AFS_BENCH_SHARE_GPU") == "1"
        if share:
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_2111_10140_b200 as afs
    from paper_2111_10140_b200 import synthetic

    w = synthetic.c3(N=args.n)
    owner = lpt_assign(w.windows, w.N, w.m, world)
    mine = [i for i in range(w.P) if owner[i] == rank]
    my_windows = [w.windows[i] for i in mine]
    torch.cuda.synchronize()
    t_build0 = time.perf_counter()
    op = afs.AnovaKernelOperator(w.X, my_windows, w.sigma, afs.AccuracyProfile("c3", 2.0, w.m),
                                 None, afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                 weights=[1.0 / w.P] * len(mine), deterministic=args.deterministic)
    plan = op._plan
    torch.cuda.synchronize()
    plan_build_s = time.perf_counter() - t_build0
    alpha_host = w.alpha
    alpha = torch.from_numpy(alpha_host).to(dev)[None, :].contiguous()
    out = torch.empty((1, w.N), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.apply_device(alpha, out, 1)
        if dist is not None:
            dist.all_reduce(out)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # --- headline: K matvecs, device-timed with CUDA events on the launching stream
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = 1000.0 / ms_step

    # --- stage shares (separate profiled pass; one sync per apply)
    plan.set_profiling(True)
    for _ in range(max(2, min(args.steps, 5))):
        plan.apply_device(alpha, out, 1)
    torch.cuda.synchronize()
    st = plan.stage_times(reset=True)
    win_sp, win_ga = plan.window_times(reset=True)
    plan.set_profiling(False)
    napp = max(1, st["applies"])
    stage = {k: st[k] / napp for k in ("spread_ms", "spectral_ms", "gather_ms")}
    win_sp = [t / napp for t in win_sp]
    win_ga = [t / napp for t in win_ga]

    # --- e2e through the public API with host buffers: alpha in pinned host memory (torch CPU
    # tensor) -> AnovaKernelOperator.apply -> result in pinned host memory; the pageable numpy
    # path (the reference's own call style) is reported beside it
    alpha_pinned = torch.from_numpy(alpha_host).pin_memory()

    def e2e_time(x):
        times = []
        warm = 2   # first use allocates staging, the second captures the CUDA graph
        for i in range(max(1, args.e2e_steps) + warm):
            barrier()
            t0 = time.perf_counter()
            if dist is None:
                res = op.apply(x)                      # H2D alpha, matvec, D2H result
            else:
                # H2D alpha, this rank's windows on the device, all-reduce, D2H of the sum
                xt = x if torch.is_tensor(x) else torch.from_numpy(x)
                part = op.apply(xt.to(dev, non_blocking=True))
                dist.all_reduce(part)
                res = part.cpu()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if i >= warm:
                times.append(dt)
        t_s = float(np.mean(times))
        if dist is not None:
            t = torch.tensor([t_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_s = float(t.item())
        return t_s

    e2e_s = e2e_time(alpha_pinned)
    e2e_pageable_s = e2e_time(alpha_host)

    # roofline of the dominant kernel: group the per-window launches by (stage, window dim),
    # take the group with the largest total time, report algorithmic bytes per launch over
    # its mean launch time (and its fp64 rate against the measured fp64 peak)
    peak, peak_src = measured_peak_hbm()
    groups = {}
    for l, win in enumerate(my_windows):
        d = len(win)
        for kind, t in (("spread", win_sp[l]), ("gather", win_ga[l])):
            groups.setdefault((kind, d), []).append(t)
    (kind, d), times = max(groups.items(), key=lambda kv: sum(kv[1]))
    t_launch = float(np.mean(times)) * 1e-3
    n = plan.n
    dom_bytes = w.N * 8 * d + w.N * 8 + 8 * n ** d      # coordinates + alpha/out + grid
    achieved = dom_bytes / t_launch / 1e9
    # Horner degree of the compile-time window table (kb_tables.inc kb_terms - 1; n = 2M)
    deg = {1: 13, 2: 12, 3: 12}.get(w.m, 11) if plan.n == 2 * w.M else 13
    fma_per_node = (2 * w.m) ** d + 2 * w.m * d * deg + (2 * w.m) ** (d - 1)   # touches + Horner
    fp64_tflops = 2.0 * fma_per_node * w.N / t_launch / 1e12
    fp64_peak, fp64_src = measured_fp64_peak()
    traffic = ncu_traffic(f"{kind}_d{d}")
    info = plan.info()
    Btot, _, _ = algorithmic_bytes(w.N, w.windows, plan.n)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        wc = synthetic.c3(N=args.cpu_n)
        tcpu, _ = cpu_matvec_seconds(wc, 1)
        scale = args.n / args.cpu_n
        cpu = {"value": 1.0 / (tcpu * scale), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"oracle port (numpy restatement of the reference) on the C3 recipe at "
                         f"N={args.cpu_n:,}, all 39 windows, one matvec in {tcpu:.2f} s on 1 core; "
                         f"matvecs/s extrapolated linearly to N={args.n:,}",
               "updates_per_s": args.cpu_n * w.P / tcpu}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(w.N, w.P, w.m, w.M, plan.n,
                                      {"parallelism": f"windows dealt by LPT over {world} GPU(s)"
                                                      + ("; NCCL all-reduce of the N-vector" if world > 1 else ""),
                                       "spread_accumulation": "fixed-point limbs (deterministic)"
                                                              if args.deterministic else "fp64 atomics"}),
            "updates_per_s": w.N * w.P * value,
            "hbm_fraction_matvec": {"bytes_per_matvec": Btot,
                                    "achieved_gbs": Btot / (ms_step * 1e-3) / 1e9,
                                    "frac_of_measured": Btot / (ms_step * 1e-3) / 1e9 / peak,
                                    "frac_of_8tbs": Btot / (ms_step * 1e-3) / 8e12},
            "stage_ms": stage,
            "plan_build_s": plan_build_s,
            "roofline": {"bound": "hbm", "kernel": f"{kind} ({d}-D windows)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": dom_bytes,
                         "mean_launch_ms": t_launch * 1e3, "launches_per_step": len(times),
                         "fp64": {"achieved_tflops": fp64_tflops, "peak_tflops": fp64_peak,
                                  "frac": fp64_tflops / fp64_peak, "peak_source": fp64_src,
                                  "fma_per_node": fma_per_node},
                         "note": "m=4 makes the kernel fp64-pipe-bound (DESIGN.md §5); 2-D windows at "
                                 "m=4 run on the fp64 tensor cores (DMMA: the spread executes 256 "
                                 "MACs/node, the gather 192 plus 1024 per half-cell, vs the 248 "
                                 "algorithmic FMAs counted here); traffic = ncu dram "
                                 "read+write per launch (profiles/)"},
            "window_ms": {"spread": win_sp, "gather": win_ga},
            "cpu_baseline": cpu,
            "e2e": {"value": 1.0 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * w.N,
                    "d2h_bytes_per_step": 8 * w.N,
                    "path": ("AnovaKernelOperator.apply(pinned torch CPU alpha) -> pinned CPU result"
                             if world == 1 else
                             "pinned alpha -> device; AnovaKernelOperator.apply on this rank's windows; "
                             "NCCL all-reduce; D2H of the sum"),
                    "pageable_numpy_value": 1.0 / e2e_pageable_s},
            "clocks": clk.summary(),
            "gpu_launches": info["kernel_launches_per_apply"] * args.steps,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
