#!/usr/bin/env python
"""Print the phases / per-kernel table of a bench.py JSON line."""
import json
import sys

line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(line)
print(f"ms/step {d['ms_per_step']:.3f}  value {d['value']:.4g} {d['unit']}")
for k, v in d.get("phases", {}).items():
    print(f"  {k:10s} {v}")
for k, v in sorted(d.get("kernels", {}).items(), key=lambda x: -x[1]["ms_per_step"]):
    print(f"  {k:22s} {v['ms_per_step']:8.3f} ms  {v['gbs'] or 0:8.1f} GB/s")
for key in ("roofline", "e2e", "clocks", "cpu_baseline"):
    if d.get(key):
        print(key, json.dumps(d[key])[:400])
