"""Summarise an ncu --page source --csv export (SASS): instructions per
mma step by execution-frequency bucket, hot opcode mix, top stall sites.
    ncu -i rep --page source --csv --print-source sass > src.csv
    python scripts/ncu_src_summary.py src.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
for d in data:
    d["n"] = int(d["Instructions Executed"] or 0)
    d["s"] = int(d["Warp Stall Sampling (All Samples)"] or 0)
    toks = d["Source"].strip().split()
    d["op"] = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else ""))
step = max(d["n"] for d in data if d["op"].startswith("HMMA"))
tot = sum(d["n"] for d in data)
S = sum(d["s"] for d in data)
print("instructions per mma step: %.1f (steps %d)" % (tot / step, step))
b, bs = collections.Counter(), collections.Counter()
for d in data:
    r = d["n"] / step
    k = "hot" if r >= 0.9 else ("warm" if r >= 0.02 else "cold")
    b[k] += d["n"] / step
    bs[k] += d["s"] / S
print("per step by bucket", {k: round(v, 1) for k, v in b.items()}, "stall share", {k: round(v, 3) for k, v in bs.items()})
ops = collections.Counter()
for d in data:
    if d["n"] >= 0.9 * step:
        ops[d["op"].split(".")[0]] += d["n"] / step
print("hot opcodes per step", [(k, round(v, 1)) for k, v in ops.most_common(20)])
ops = collections.Counter()
for d in data:
    if 0.02 * step <= d["n"] < 0.9 * step:
        ops[d["op"].split(".")[0]] += d["n"] / step
print("warm opcodes per step", [(k, round(v, 1)) for k, v in ops.most_common(20)])
for d in sorted(data, key=lambda d: -d["s"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print("%.3f  x%.3f  %s  %s" % (d["s"] / S, d["n"] / step, d["Address"][-5:], d["Source"].strip()[:70]))
