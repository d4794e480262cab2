#!/usr/bin/env python
"""Benchmark: ANOVA fast-summation matvecs/s on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[2], the config the metric's roofline target is
quoted on): C3 -- N=10,000,000 points, d=9 features U[-1/4,1/4), 3 triple windows + 36
pair windows (P=39, eta=1/39), Gaussian sigma=0.5, M=64 (grid n=128), m=4, one
right-hand side, fp64.  One "step" = one full ANOVA matvec.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c4|c5]

--gpus N > 1 runs one process per GPU: launched under torchrun by the driver, or, when
WORLD_SIZE is unset, bench.py re-executes itself under torch.distributed.run with N
ranks.  Multi-GPU paths:
  c3  windows dealt to ranks by LPT, one NCCL all-reduce of the N-vector per matvec
  c5  (BASELINE configs[4]) 200-iteration CG on window shards, replicated vectors
  c4  (BASELINE configs[3]) N=1e8, R=8, points sharded, NCCL all-reduce of the pruned
      spectra per matvec, output row-sharded
Rank 0 prints ONE JSON line.

``--impl reference`` times the UNMODIFIED reference package (``nfftkrr``, byte-compiled
into oracle/_ref by oracle/build_ref.py) through its own public API on this box's host
cores: per step one matvec of the same config on a bounded first-rows sample, windows
(c3/c5) or right-hand sides (c4) dealt over a process pool of all cores; the per-matvec
time is extrapolated linearly to the full N and both numbers are reported.  Rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ANOVA fast-sum matvecs/s"
UNIT = "matvec/s"
FULL_N = {"c3": 10_000_000, "c4": 100_000_000, "c5": 1_000_000}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c3", "c4", "c5"], default="c3")
    ap.add_argument("--n", type=int, default=None, help="points (default: the config's N)")
    ap.add_argument("--cpu-n", type=int, default=None, help="cpu_baseline sample size")
    ap.add_argument("--ref-n", type=int, default=None,
                    help="reference-arm sample size (default: sized to --ref-budget-s)")
    ap.add_argument("--ref-budget-s", type=float, default=240.0)
    ap.add_argument("--cg-iters", type=int, default=200, help="c5: CG iterations per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--deterministic", action="store_true",
                    help="bit-reproducible fixed-point spread (afs_plan_set_deterministic)")
    if argv is None and os.environ.get("AFS_BENCH_ARGV"):
        argv = json.loads(os.environ["AFS_BENCH_ARGV"])   # set by relaunch_under_torchrun
    a = ap.parse_args(argv)
    if a.n is None:
        a.n = FULL_N[a.config]
    return a


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` without a launcher: re-exec with N ranks (127.0.0.1)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)]
    # the ranks get this command line through the environment: torchrun's own argument parser
    # would otherwise see (and reject as ambiguous) options such as --n after the script
    env = dict(os.environ, AFS_BENCH_ARGV=json.dumps(sys.argv[1:]))
    return subprocess.call(cmd, env=env)


def algorithmic_bytes(N, windows, n, R=1):
    """B = sum_l [(Nx+Nz)*8*d_l + Nx*8*R + Nz*8*R] + sum_l 32*R*n^d_l (Z=X)."""
    tot = 0
    for w in windows:
        d = len(w)
        tot += 2 * (N * 8 * d + N * 8 * R + 8 * R * n ** d) + 16 * R * n ** d
    return tot


def fma_per_node(d, m, M, n):
    """fp64 FMAs per node and pass: touches (2m)^d + Horner window values 2m d deg + line
    products (2m)^(d-1); deg from the compile-time tables (kb_tables.inc kb_terms - 1)."""
    deg = {1: 13, 2: 12, 3: 12}.get(m, 11) if n == 2 * M else 13
    return (2 * m) ** d + 2 * m * d * deg + (2 * m) ** (d - 1)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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

    def _nvml_handle(self, nv):
        """NVML handle of CUDA device self.idx, matched by UUID (CUDA and NVML orders can
        differ, e.g. under CUDA_VISIBLE_DEVICES); the NVML index as a fallback."""
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.idx).uuid)
            for i in range(nv.nvmlDeviceGetCount()):
                h = nv.nvmlDeviceGetHandleByIndex(i)
                u = nv.nvmlDeviceGetUUID(h)
                u = u.decode() if isinstance(u, bytes) else u
                if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                    return h
        except Exception:
            pass
        return nv.nvmlDeviceGetHandleByIndex(self.idx)

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
            h = self._nvml_handle(nv)
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
# CPU side: the UNMODIFIED reference (oracle/_ref) -- a checker/baseline, never the product
# ---------------------------------------------------------------------------
REF_ZIP = os.path.join(REPO, "oracle", "_ref", "nfftkrr_ref.zip")
_POOL = {}


def import_reference():
    """The reference package byte-compiled by oracle/build_ref.py (prebuilt on the GPU box)."""
    if not os.path.exists(REF_ZIP):
        from oracle import build_ref

        if build_ref.build() is None:
            raise RuntimeError("oracle/_ref/nfftkrr_ref.zip missing: run oracle/build_ref.py "
                               "where /root/reference exists")
    if REF_ZIP not in sys.path:
        sys.path.insert(0, REF_ZIP)
    import nfftkrr

    if not hasattr(nfftkrr, "FastsumOperator") or REF_ZIP not in (nfftkrr.__file__ or ""):
        raise RuntimeError(f"imported {nfftkrr!r}, not the reference build in {REF_ZIP}")
    return nfftkrr


def reference_workload(config, N):
    from paper_2111_10140_b200 import synthetic

    if config == "c3":
        return synthetic.c3(N=N)
    if config == "c5":
        return synthetic.c5(N=N)
    return synthetic.c4(N=N, R=8)


def reference_ops(nk, w):
    """One reference FastsumOperator per window: the SURVEY §8(c) composed recipe (the
    reference's WindowSet rejects the overlapping C3/C5 window lists)."""
    prof = nk.AccuracyProfile("bench", 2.0, w.m)
    cfg = nk.PeriodizationConfig(coeff_grid=w.M)
    return [nk.FastsumOperator(nk.GaussianKernel(w.sigma), cfg, w.X[:, list(win)], None, prof)
            for win in w.windows]


def _ref_task(i):
    st = _POOL
    t0 = time.perf_counter()
    if st["per_rhs"]:
        s = st["ops"][0].apply(st["alpha"][:, i])
    else:
        s = st["ops"][i].apply(st["alpha"])
    return i, s, time.perf_counter() - t0


class ReferenceMatvec:
    """One matvec of the reference on `workers` processes (fork after the operators are
    built, so they are shared copy-on-write); tasks are windows (c3/c5, summed with
    eta = 1/P in window order, anova.py:179-183) or right-hand sides (c4)."""

    def __init__(self, config, N, workers):
        import multiprocessing as mp

        nk = import_reference()
        self.w = reference_workload(config, N)
        t0 = time.perf_counter()
        self.ops = reference_ops(nk, self.w)
        self.build_s = time.perf_counter() - t0
        self.per_rhs = config == "c4"
        ntask = self.w.R if self.per_rhs else self.w.P
        self.tasks = list(range(ntask))
        _POOL.update(ops=self.ops, alpha=self.w.alpha, per_rhs=self.per_rhs)
        self.workers = max(1, min(workers, ntask))
        self.pool = mp.get_context("fork").Pool(self.workers) if self.workers > 1 else None
        self.task_s = {}

    def __call__(self):
        t0 = time.perf_counter()
        if self.pool is None:
            res = [_ref_task(i) for i in self.tasks]
        else:
            res = self.pool.map(_ref_task, self.tasks, chunksize=1)
        parts = {i: s for i, s, _ in res}
        self.task_s = {i: t for i, _, t in res}
        if self.per_rhs:
            out = np.stack([parts[i] for i in self.tasks], axis=1)
        else:
            out = np.zeros(self.w.N)
            for i in self.tasks:
                out += (1.0 / self.w.P) * parts[i]
        return time.perf_counter() - t0, out

    def order_by_cost(self):
        """Longest tasks first (the pool takes them in order: LPT-like dealing)."""
        if self.task_s:
            self.tasks = sorted(self.tasks, key=lambda i: -self.task_s[i])

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def plan_reference_sample(config, steps, budget_s, workers):
    """Largest first-rows sample N (<= the config's reference-sample cap) whose build +
    steps matvecs fit the budget, from a probe at N=20k (times scaled linearly in N,
    which over-estimates the fixed FFT costs, so the choice is conservative)."""
    cap = {"c3": 1_000_000, "c5": 1_000_000, "c4": 1_000_000}[config]
    probe = ReferenceMatvec(config, 20_000, workers)
    probe()                                   # per-task times at the probe size
    task = sorted(probe.task_s.values(), reverse=True)
    build = probe.build_s
    probe.close()
    loads = [0.0] * probe.workers
    for t in task:                            # LPT makespan of one matvec at the probe size
        k = loads.index(min(loads))
        loads[k] += t
    per_pt = max(loads) / 20_000
    per_pt_build = build / 20_000
    n = int(budget_s / (steps * per_pt + per_pt_build))
    return max(20_000, min(cap, n // 10_000 * 10_000))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    steps_total = args.steps + args.warmup
    N = args.ref_n or plan_reference_sample(args.config, steps_total, args.ref_budget_s, cores)
    rm = ReferenceMatvec(args.config, N, cores)
    for k in range(args.warmup):
        rm()
        if k == 0:
            rm.order_by_cost()
    times = [rm()[0] for _ in range(args.steps)]
    rm.close()
    t = float(np.mean(times))
    full = FULL_N[args.config]
    factor = full / N
    value = 1.0 / (t * factor)
    w = rm.w
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, full, w, 2 * w.M),
        "reference": {"package": "nfftkrr (unmodified; oracle/_ref built by oracle/build_ref.py)",
                      "api": "FastsumOperator(...).apply per window, composed with eta=1/P "
                             "(SURVEY §8(c))" if args.config != "c4" else
                             "FastsumOperator(...).apply per right-hand side",
                      "sample_n": N, "measured_s_per_matvec": t,
                      "extrapolation_factor": factor,
                      "extrapolated_s_per_matvec_full_n": t * factor,
                      "plan_build_s": rm.build_s, "cpu_model": cpu_model(),
                      "processes": rm.workers, "host_cores": cores},
        "updates_per_s": N * w.P * w.R / t,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": rm.workers, "kind": "reference",
                         "sample": f"first-rows sample N={N:,} of the {args.config.upper()} recipe, "
                                   f"one matvec per step ({t:.2f} s measured), "
                                   f"{'RHS' if args.config == 'c4' else 'windows'} dealt over "
                                   f"{rm.workers} processes; matvecs/s extrapolated x{factor:g} "
                                   f"to N={full:,}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(config, n_sample):
    """Reference on ONE core, one matvec of a bounded sample (10-30 s of CPU work)."""
    rm = ReferenceMatvec(config, n_sample, 1)
    if config == "c4":
        rm.tasks = [0]                       # one right-hand side, scaled by R below
    t, _ = rm()
    t_full = t * (8 if config == "c4" else 1) * FULL_N[config] / n_sample
    return {"value": 1.0 / t_full, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"unmodified reference (oracle/_ref) on 1 core, {config.upper()} recipe at "
                      f"N={n_sample:,}" + (", one of the 8 right-hand sides" if config == "c4" else "")
                      + f": {t:.2f} s; matvecs/s extrapolated linearly to N={FULL_N[config]:,}",
            "cpu_model": cpu_model()}


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
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


def workload_config(config, N, w, n, extra=None):
    if config == "c3":
        cfg = {"workload": f"C3: N={N:,} d=9 U[-1/4,1/4), 3 triples + 36 pairs (P=39), sigma=0.5, "
                           f"M={w.M} (grid n={n}), m={w.m}, R=1, fp64",
               "l2": "inputs larger than L2 (720 MB coordinates + 80 MB alpha + 80 MB out per matvec)"}
    elif config == "c5":
        cfg = {"workload": f"C5: N={N:,} d=20 (5 blocks rho=0.7), 20 singles + 10 pairs (P=30), "
                           f"sigma=1, beta=0.1, M={w.M} (grid n={n}), m={w.m}; one step = a "
                           f"CG solve at tol 1e-6 capped at the iteration count below (x0=0); "
                           f"metric counts matvecs (one per CG iteration), fp64",
               "l2": "inputs larger than L2 (160 MB coordinates + 8 MB vectors, 30 windows)"}
    else:
        cfg = {"workload": f"C4: N={N:,} d=3, 16-cluster Gaussian mixture (std 0.02), one 3-D window, "
                           f"sigma=0.1, M={w.M} (grid n={n}), m={w.m}, R=8 right-hand sides, fp64",
               "l2": "inputs larger than L2 (2.4 GB coordinates + 6.4 GB alpha + 6.4 GB out)"}
    cfg.update({"N": N, "P": w.P, "M": w.M, "n": n, "m": w.m, "R": w.R})
    if extra:
        cfg.update(extra)
    return cfg


def init_dist(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # test hook for the multi-rank code path on a single-GPU box: AFS_BENCH_SHARE_GPU=1
    # maps every rank onto the visible devices round-robin and uses gloo (host-staged
    # all-reduce; no rank's kernels wait on another's).  Never used for reported numbers.
    share = os.environ.get("AFS_BENCH_SHARE_GPU") == "1"
    if world > 1:
        import torch.distributed as dist

        if share:
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but {world} rank(s) started")
    return torch, dist, rank, world, torch.device("cuda", torch.cuda.current_device())


def max_over_ranks(v, dist, dev):
    if dist is None:
        return v
    import torch

    t = torch.tensor([float(v)], dtype=torch.float64, device=dev if dist.get_backend() == "nccl"
                     else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def device_timed(torch, step, steps, dev, dist):
    """K steps between barrier + synchronize, CUDA events on the launching stream, clocks
    sampled during the region; returns (ms per step, max over ranks; clock summary)."""
    stream = torch.cuda.current_stream(dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    return max_over_ranks(e0.elapsed_time(e1), dist, dev) / steps, clk.summary()


def wall_timed(torch, fn, reps, warm, dist, dev):
    """Mean wall seconds of fn() (host buffers in and out), max over ranks."""
    times = []
    for i in range(reps + warm):
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        if i >= warm:
            times.append(time.perf_counter() - t0)
    return max_over_ranks(float(np.mean(times)), dist, dev)


def stage_profile(plan, alpha, out, R, reps):
    """Per-stage and per-window device times (profiling mode: one sync per apply)."""
    plan.set_profiling(True)
    for _ in range(reps):
        plan.apply_device(alpha, out, R)
    st = plan.stage_times(reset=True)
    sp, ga = plan.window_times(reset=True)
    plan.set_profiling(False)
    k = max(1, st["applies"])
    return ({key: st[key] / k for key in ("spread_ms", "spectral_ms", "gather_ms")},
            [t / k for t in sp], [t / k for t in ga])


def roofline(windows, win_sp, win_ga, N, R, M, m, n):
    """The dominant kernel = the (stage, window dim) group with the largest total time;
    achieved = its algorithmic bytes per launch / mean launch time."""
    groups = {}
    for l, win in enumerate(windows):
        for kind, t in (("spread", win_sp[l]), ("gather", win_ga[l])):
            groups.setdefault((kind, len(win)), []).append(t)
    (kind, d), times = max(groups.items(), key=lambda kv: sum(kv[1]))
    t_launch = float(np.mean(times)) * 1e-3
    dom_bytes = N * 8 * d + N * 8 * R + 8 * R * n ** d       # coordinates + alpha/out + grid
    achieved = dom_bytes / t_launch / 1e9
    fpn = fma_per_node(d, m, M, n) + (R - 1) * (2 * m) ** d
    fp64 = 2.0 * fpn * N / t_launch / 1e12
    peak, peak_src = measured_peak_hbm()
    fpk, fpk_src = measured_fp64_peak()
    return {"bound": "hbm", "kernel": f"{kind} ({d}-D windows)", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic(f"{kind}_d{d}"),
            "peak_source": peak_src, "algorithmic_bytes_per_launch": dom_bytes,
            "mean_launch_ms": t_launch * 1e3, "launches_per_step": len(times),
            "fp64": {"achieved_tflops": fp64, "peak_tflops": fpk, "frac": fp64 / fpk,
                     "peak_source": fpk_src, "fma_per_node": fpn},
            "note": "fp64 figures use the reference's tensor-product operation count (fma_per_node); "
                    "the sub-cell 2-D kernels (sc2d.cuh) execute 62 (gather) / 78 (spread) per node and "
                    "are bound by the SM load/store pipe: one l1tex cycle per randomly indexed 8-byte "
                    "access plus the shared-memory tables (ncu, profiles/r02_ncu_sc_2d.txt); the 3-D "
                    "kernels run on the fp64 tensor cores at ~71% of the pipe; traffic = ncu dram "
                    "read+write per launch (profiles/ncu_traffic.json)"}


def free_operator(afs, w, windows, weights, max_rhs=1, deterministic=False, device=None):
    return afs.AnovaKernelOperator(w.X, windows, w.sigma, afs.AccuracyProfile("bench", 2.0, w.m),
                                   None, afs.PeriodizationConfig(coeff_grid=w.M), strict=False,
                                   weights=weights, max_rhs=max_rhs, deterministic=deterministic,
                                   device=device)


def run_ours(args):
    torch, dist, rank, world, dev = init_dist(args)
    import paper_2111_10140_b200 as afs
    from paper_2111_10140_b200 import synthetic
    from paper_2111_10140_b200.distributed import lpt_assign, window_costs

    warm = max(3, args.warmup)
    cfg = args.config
    extra = {}
    if cfg == "c4":
        w = synthetic.c4_shard(args.n, 8, rank, world)
        N_total = args.n
        mine = [0]
    else:
        w = synthetic.c3(N=args.n) if cfg == "c3" else synthetic.c5(N=args.n)
        N_total = w.N
        owner = lpt_assign(window_costs(w.windows, w.N, w.m), world)
        mine = [i for i in range(w.P) if owner[i] == rank]
    my_windows = [w.windows[i] for i in mine]
    torch.cuda.synchronize()
    t_build0 = time.perf_counter()
    R = w.R
    if cfg == "c4" and world > 1:
        from paper_2111_10140_b200.distributed import CudaPointBackend, PointSharded

        backend = CudaPointBackend(w.X, w.windows, w.sigma, M=w.M, m=w.m, max_rhs=R,
                                   device=dev.index, exchange="spectrum")
        op, plan = PointSharded(backend), backend.plan
    elif cfg == "c5" and world > 1:   # WindowSharded makes the same LPT deal, owns the plan
        sharded = afs.WindowSharded(w.X, w.windows, w.sigma, M=w.M, m=w.m, device=dev.index)
        op = sharded.local
        plan = op._plan if op is not None else None
    else:
        op = free_operator(afs, w, my_windows, [1.0 / w.P] * len(mine), max_rhs=R,
                           deterministic=args.deterministic, device=dev.index) if mine else None
        plan = op._plan if op is not None else None
    torch.cuda.synchronize()
    plan_build_s = time.perf_counter() - t_build0
    Nloc = w.N
    alpha_host = np.ascontiguousarray(w.alpha.reshape(Nloc, R).T)     # (R, N) rows
    alpha = torch.from_numpy(alpha_host).to(dev)
    out = torch.zeros((R, Nloc), dtype=torch.float64, device=dev)
    gpu_launches_step = (plan.info()["kernel_launches_per_apply"] if plan is not None else 0)

    if cfg == "c3":
        def step():
            if plan is not None:
                plan.apply_device(alpha, out, 1)
            if dist is not None:
                dist.all_reduce(out)
        h2d, d2h = 8 * w.N, 8 * w.N
    elif cfg == "c4":
        if world > 1:
            def step():
                res = op.apply(alpha)
                out.copy_(res)
        else:
            def step():
                plan.apply_device(alpha, out, R)
        h2d, d2h = 8 * Nloc * R * world, 8 * Nloc * R * world
    else:   # c5: whole CG solves, maxiter = --cg-iters
        system = afs.KernelSystem(sharded if world > 1 else op, w.beta)
        b_dev = torch.from_numpy(w.y).to(dev)
        iters = []

        def step():
            res = afs.cg_solve(system, b_dev, tol=1e-6, maxiter=args.cg_iters)
            iters.append(res.iterations)
        h2d, d2h = 8 * w.N, 8 * w.N

    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    ms_step, clocks = device_timed(torch, step, args.steps, dev, dist)
    if cfg == "c5":
        its = iters[-args.steps:]
        matvecs_per_step = float(np.mean(its))
        value = matvecs_per_step * 1000.0 / ms_step
        extra.update({"cg_iterations_per_step": its[-1], "cg_solve_ms": ms_step,
                      "cg_tol": 1e-6, "cg_maxiter": args.cg_iters})
    else:
        matvecs_per_step = 1.0
        value = 1000.0 / ms_step

    # --- stage shares and per-window kernel times (profiling pass on this rank's plan)
    stage, win_sp, win_ga = ({}, [], [])
    if plan is not None:
        a1 = alpha if cfg != "c5" else torch.from_numpy(w.y).to(dev)[None, :].contiguous()
        stage, win_sp, win_ga = stage_profile(plan, a1, out, R, max(2, min(args.steps, 5)))

    # --- e2e through the public API with host buffers (H2D in, D2H out inside the region)
    if cfg == "c3":
        alpha_pinned = torch.from_numpy(w.alpha).pin_memory()

        def e2e_call(x):
            if dist is None:
                return op.apply(x)                       # AnovaKernelOperator.apply
            xt = x if torch.is_tensor(x) else torch.from_numpy(x)
            part = op.apply(xt.to(dev, non_blocking=True)) if op is not None else \
                torch.zeros(w.N, dtype=torch.float64, device=dev)
            dist.all_reduce(part)
            return part.cpu()
        e2e_s = wall_timed(torch, lambda: e2e_call(alpha_pinned), args.e2e_steps, 2, dist, dev)
        e2e_np_s = wall_timed(torch, lambda: e2e_call(w.alpha), args.e2e_steps, 2, dist, dev)
        e2e_path = ("AnovaKernelOperator.apply(pinned torch CPU alpha) -> pinned CPU result"
                    if world == 1 else "pinned alpha -> device; AnovaKernelOperator.apply on this "
                    "rank's windows; NCCL all-reduce; D2H of the sum")
        e2e_value = 1.0 / e2e_s
    elif cfg == "c4":
        a_host = torch.from_numpy(np.ascontiguousarray(w.alpha)).pin_memory()   # (N_loc, R)

        def e2e_call():
            if world == 1:
                return op.apply(a_host)                 # AnovaKernelOperator.apply, (N, R)
            res = op.apply(a_host.to(dev, non_blocking=True).t().contiguous())
            return res.t().cpu()
        e2e_s = wall_timed(torch, e2e_call, max(2, args.e2e_steps // 2), 1, dist, dev)
        e2e_np_s = None
        e2e_path = ("AnovaKernelOperator.apply(pinned (N, 8) alpha) -> (N, 8) host result" if world == 1
                    else "PointSharded.apply: pinned row shard -> device, spread + spectral forward, "
                         "NCCL all-reduce of the pruned spectra, inverse + gather, D2H of the rows")
        e2e_value = 1.0 / e2e_s
    else:
        def e2e_call():
            res = afs.cg_solve(system, w.y, tol=1e-6, maxiter=args.cg_iters)   # numpy in/out
            return res
        e2e_s = wall_timed(torch, e2e_call, max(2, args.e2e_steps // 2), 1, dist, dev)
        e2e_np_s = None
        e2e_path = ("cg_solve(KernelSystem(op, beta), numpy y) -> numpy x "
                    + ("(whole-solve CUDA graph)" if world == 1 else
                       "(window-sharded CG: NCCL all-reduce of Ap per iteration)"))
        e2e_value = matvecs_per_step / e2e_s

    roof = roofline(my_windows, win_sp, win_ga, Nloc, R, w.M, w.m, 2 * w.M) if win_sp else None
    Btot = algorithmic_bytes(N_total, w.windows, 2 * w.M, R)
    peak, _ = measured_peak_hbm()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_cpu = args.cpu_n or {"c3": 50_000, "c4": 50_000, "c5": 100_000}[cfg]
        try:
            cpu = cpu_baseline(cfg, n_cpu)
        except Exception as e:   # the checker is absent: report it instead of failing the bench
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        mv_s = value
        par = {"c3": f"windows dealt by LPT over {world} GPU(s)" + (
                   "; NCCL all-reduce of the N-vector per matvec" if world > 1 else ""),
               "c5": f"windows dealt by LPT over {world} GPU(s)" + (
                   "; replicated CG vectors, NCCL all-reduce of Ap per iteration" if world > 1
                   else "; whole-solve CUDA graph (device-side loop)"),
               "c4": f"points sharded over {world} GPU(s)" + (
                   "; NCCL all-reduce of the pruned spectra per matvec" if world > 1 else "")}[cfg]
        line = {
            "metric": METRIC, "value": mv_s, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded numpy PCG64, BASELINE shapes)",
            "config": workload_config(cfg, N_total, w, 2 * w.M, dict(
                parallelism=par, **({"spread_accumulation": "fixed-point limbs (deterministic)"
                                     if args.deterministic else "fp64 atomics"}), **extra)),
            "updates_per_s": N_total * w.P * R * mv_s,
            "hbm_fraction_matvec": {"bytes_per_matvec": Btot,
                                    "achieved_gbs": Btot * mv_s / 1e9,
                                    "frac_of_measured": Btot * mv_s / 1e9 / peak,
                                    "frac_of_8tbs": Btot * mv_s / 8e12},
            "stage_ms_rank0": stage, "plan_build_s": plan_build_s,
            "roofline": roof,
            "window_ms_rank0": {"spread": win_sp, "gather": win_ga},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "path": e2e_path,
                    **({"pageable_numpy_value": 1.0 / e2e_np_s} if e2e_np_s else {})},
            "clocks": clocks,
            "gpu_launches": int(gpu_launches_step * matvecs_per_step * args.steps),
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
