"""Stall hot spots of an ncu --page source --csv --print-source sass export:
python tools/sass_hot.py gpurun_out/<tag>_sass.csv [N]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("samples", tot, "instructions", len(data))
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = Counter()
for r in data:
    for k in stalls:
        agg[k] += int(r[ix[k]] or 0)
print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in agg.most_common(10)))
opc = Counter()
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    opc[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in opc.most_common(16)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in top:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    why = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    print(f"{100*s/tot:5.2f}% {r[ix['Address']]:>6} {r[ix['Source']][:60]:60s} {why}")
