#!/usr/bin/env python
"""Write profiles/ncu_traffic.json from `ncu --set full` captures.

usage: python scripts/ncu_traffic.py <config> <phase> <kernel> <report.ncu-rep> [...]
(repeated groups of four). Records dram__bytes_read.sum + dram__bytes_write.sum
of the captured launch, which bench.py reports as roofline.traffic.
"""
import csv
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    tot = 0.0
    for k, un, x in zip(h, u, v):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(x.replace(",", "")) * UNIT[un]
    return int(tot)


def main():
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                        "ncu_traffic.json")
    data = {}
    if os.path.exists(path):
        data = json.load(open(path))
    args = sys.argv[1:]
    for i in range(0, len(args), 4):
        cfg, phase, kernel, rep = args[i:i + 4]
        data.setdefault(cfg, {})[phase] = {"kernel": kernel, "dram_bytes": dram_bytes(rep),
                                           "source": os.path.basename(rep)}
    with open(path, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
