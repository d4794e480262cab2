"""Summarise gpurun_out/NAME_raw.csv (+ _src.csv) from tools/ncu_box.sh: key metrics, top stall
reasons, and the SASS opcode mix with shared-memory wavefronts.   python tools/ncu_read.py NAME"""
import collections
import csv
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_red.sum", "sm__inst_executed_pipe_fp64.sum"]


def main(name):
    rows = list(csv.reader(open(f"gpurun_out/{name}_raw.csv")))
    h, u = rows[0], rows[1]
    ki = h.index("Kernel Name")
    stalls = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        print("##", r[ki][:100])
        for k in KEYS:
            if k in h:
                print(f"   {k:80s} {r[h.index(k)]:>14s} {u[h.index(k)]}")
        st = sorted(((float(r[h.index(k)] or 0), k) for k in stalls), reverse=True)[:7]
        print("   stalls:", ", ".join(f"{k[34:-23]} {v:.2f}" for v, k in st))
    try:
        src = list(csv.reader(open(f"gpurun_out/{name}_src.csv")))
    except OSError:
        return
    kernels = []
    cur = None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            kernels.append(cur)
        elif cur is not None and r and r[0] == "Address":
            cur["h"] = {k: i for i, k in enumerate(r)}
        elif cur is not None and r and r[0].startswith("0x"):
            cur["rows"].append(r)
    seen = set()
    for kz in kernels:
        if kz["name"] in seen or "h" not in kz:
            continue
        seen.add(kz["name"])
        H = kz["h"]
        ops, wf, smp = collections.Counter(), collections.Counter(), collections.Counter()

        def num(x):
            try:
                return int(x)
            except ValueError:
                return 0
        for r in kz["rows"]:
            t = r[H["Source"]].split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] += num(r[H["Instructions Executed"]])
            wf[op] += num(r[H.get("L1 Wavefronts Shared", 0)])
            smp[op] += num(r[H["# Samples"]])
        tot = sum(ops.values())
        print(f"\n## SASS mix {kz['name'][:90]}: {tot} warp-instructions")
        print("   " + ", ".join(f"{o}:{100 * c / tot:.1f}%" + (f"(wf {wf[o]})" if wf[o] else "")
                               for o, c in ops.most_common(14)))


if __name__ == "__main__":
    main(sys.argv[1])
