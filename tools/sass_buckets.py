"""Bucket the SASS instructions of an ncu --page source --csv dump by execution count (loop nesting
shows up as distinct counts): instruction mix, share of executed instructions and stall samples
per bucket.   python tools/sass_buckets.py gpurun_out/NAME_src.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1], encoding='utf-8', errors='replace')))
kern=None; K=[]
for r in rows:
    if r and r[0]=="Kernel Name": kern={"name":r[1],"rows":[]}; K.append(kern)
    elif r and r[0]=="Address": kern["h"]=r
    elif kern is not None and r and r[0].startswith("0x"): kern["rows"].append(r)
seen=set()
for k in K:
    if k["name"] in seen: continue
    seen.add(k["name"])
    h=k["h"]; ei=h.index("Instructions Executed"); si=h.index("Warp Stall Sampling (All Samples)")
    buckets=collections.defaultdict(lambda: [0,0,collections.Counter()])
    for r in k["rows"]:
        e=int(r[ei]); 
        if e==0: continue
        toks=r[1].split(); op=(toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        b=buckets[e]; b[0]+=1; b[1]+=int(r[si]); b[2][op]+=1
    print(k["name"][:60])
    tot=sum(e*b[0] for e,b in buckets.items())
    for e,b in sorted(buckets.items(), key=lambda x:-x[0]*x[1][0])[:12]:
        print(f"  exec={e:>10} n_instr={b[0]:4d} share={e*b[0]/tot:.1%} samples={b[1]:6d}  ", ", ".join(f"{o}:{c}" for o,c in b[2].most_common(12)))
