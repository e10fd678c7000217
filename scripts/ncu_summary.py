#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

  ncu_summary.py launches <launches.csv>          per-kernel share of a launch list
  ncu_summary.py full <prof.ncu-rep> [...]        key --set full metrics per kernel
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
        a = agg.setdefault(k, [0.0, 0])
        a[0] += float(r["Metric Value"].replace(",", "")) * scale
        a[1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"{'kernel':40s} {'total ms':>10s} {'launches':>8s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k:40s} {v[0]:10.3f} {v[1]:8d} {100 * v[0] / tot:6.1f}%")
    print(f"{'TOTAL':40s} {tot:10.3f}")


def full(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(f"== {p}: no data")
            continue
        h, units = rows[0], rows[1]
        for v in rows[2:]:
            name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            print(f"== {p}: {name[:100]}")
            for i, n in enumerate(h):
                if n in FULL_METRICS:
                    print(f"   {n:60s} {v[i]:>16s} {units[i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
