"""Summarise an ncu --page source --csv (SASS) dump: top instructions by stall samples
and executed-instruction histogram by opcode.  usage: sass_hot.py dump.csv [topN]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1], encoding='utf-8', errors='replace')))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kernels = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r and r[0].startswith("0x"):
        cur["rows"].append(r)
for k in kernels:
    h = k["hdr"]
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    tot_s = sum(int(r[si]) for r in k["rows"])
    tot_e = sum(int(r[ei]) for r in k["rows"])
    print("=" * 100)
    print(k["name"][:120], f"samples={tot_s} warp-insts={tot_e}")
    ops = collections.Counter()
    for r in k["rows"]:
        toks = r[1].split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        ops[op.split(".")[0]] += int(r[ei])
    print("  opcode mix:", ", ".join(f"{o}:{c/tot_e:.1%}" for o, c in ops.most_common(16)))
    for r in sorted(k["rows"], key=lambda r: -int(r[si]))[:top]:
        print(f"  {int(r[si]):7d} {int(r[ei]):10d}  {r[1].strip()[:90]}")
