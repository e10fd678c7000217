#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot = sum(float(r[si] or 0) for r in data)
tot_i = sum(float(r[ie] or 0) for r in data)
print(f"samples {tot:.0f}  warp-instructions {tot_i:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
idx = {id(r): k for k, r in enumerate(data)}
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    print(f"{float(r[si]) / tot * 100:5.1f}%  #{idx[id(r)]:5d} exec={r[ie]:>10}  {r[1].strip()[:90]}")
