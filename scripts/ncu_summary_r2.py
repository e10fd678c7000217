#!/usr/bin/env python
"""Round-2 ncu summaries (C4): kernel shares of the bench step from the launch
list, per-kernel DRAM bytes of the build and PageRank against their
algorithmic bytes, and profiles/ncu_traffic.json (bench.py's roofline.traffic).

usage: python scripts/ncu_summary_r2.py   (reads gpurun_out/r2n_*, writes profiles/)
"""
import csv
import io
import json
import subprocess
from collections import OrderedDict, defaultdict
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
G = REPO / "gpurun_out"
P = REPO / "profiles"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "usecond": 1e-6, "msecond": 1e-3, "second": 1}
# C4 graph (bench line): rows, nodes, distinct edges
R, N, E = 1_470_000_000, 35_431_536, 1_447_065_313


def rows(path):
    text = path.read_text()
    i = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[i:])))


def short(name):
    return name.split("(")[0].replace("void ", "").strip()


def per_launch(path):
    """[(kernel, {metric: value in base units})] in launch order."""
    out = OrderedDict()
    for r in rows(path):
        key = (int(r["ID"]), short(r["Kernel Name"]))
        out.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * \
            UNIT.get(r["Metric Unit"], 1)
    return [(k[1], v) for k, v in out.items()]


def launches_summary():
    launches = per_launch(G / "r2n_launches_c4.csv")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for k, v in launches:
        tot[k] += v["gpu__time_duration.sum"]
        cnt[k] += 1
    # the bench ran warmup 1 + steps 2 (+ generation): shares over all launches
    allt = sum(tot.values())
    lines = ["# C4 bench (python bench.py --steps 2 --warmup 1 --no-extras --no-e2e "
             "--no-cpu-baseline) under ncu --metrics gpu__time_duration.sum --clock-control none",
             "# cold-cache, serialised launches: compare SHARES, not absolute times",
             f"# {len(launches)} launches, {allt * 1e3:.1f} ms in total",
             f"{'kernel':44s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
    for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"{k:44s} {cnt[k]:8d} {t * 1e3:10.2f} {t / allt * 100:6.1f}%")
    (P / "r2_launches_c4.txt").write_text("\n".join(lines) + "\n")


def dram_summary():
    out = ["# per-launch DRAM traffic at C4 (ncu --metrics gpu__time_duration.sum,"
           "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none)",
           f"# graph: R={R} rows, N={N} nodes, E={E} edges; algorithmic bytes as in DESIGN.md §4",
           f"{'kernel':40s} {'ms':>8s} {'DRAM GB':>9s} {'DRAM GB/s':>10s}"]
    traffic = {}
    for src, label in (("r2n_build_dram_c4.csv", "ToGraph (scripts/prof_build.py c4 1)"),
                       ("r2n_pr_dram_c4.csv", "graph build + PageRank x20 (scripts/prof_pagerank.py c4 1)")):
        out.append(f"## {label}")
        agg = OrderedDict()
        for k, v in per_launch(G / src):
            if k in ("rmat_kernel", "uniform_kernel"):
                continue
            by = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
            t = v.get("gpu__time_duration.sum", 0)
            a = agg.setdefault(k, [0, 0.0, 0.0])
            a[0] += 1
            a[1] += t
            a[2] += by
            out.append(f"{k:40s} {t * 1e3:8.3f} {by / 1e9:9.3f} {by / t / 1e9 if t else 0:10.1f}")
        out.append(f"-- per kernel (sum over launches)")
        for k, (c, t, by) in agg.items():
            out.append(f"{k:40s} x{c:<3d} {t * 1e3:8.2f} ms {by / 1e9:9.2f} GB  "
                       f"{by / t / 1e9 if t else 0:8.1f} GB/s  {by / c / 1e9:8.3f} GB/launch")
            traffic[k] = by / c
    (P / "r2_ncu_dram_c4.txt").write_text("\n".join(out) + "\n")
    return traffic


def full_capture():
    rep = G / "r2n_full_c4_pr_spmv.ncu-rep"
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    keep = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct")
    lines = [f"== {rep.name}: {v[h.index('Kernel Name')][:100]}"]
    by = 0.0
    for k, un, x in zip(h, u, v):
        if k in keep:
            lines.append(f"   {k:60s} {x:>20s} {un}")
            if k.startswith("dram__bytes"):
                by += float(x.replace(",", "")) * UNIT[un]
    (P / "r2_ncu_full_c4_pr_spmv.txt").write_text("\n".join(lines) + "\n")
    return by


def main():
    launches_summary()
    t = dram_summary()
    spmv_full = full_capture()
    path = P / "ncu_traffic.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    c4 = {}
    m = {"build.minmax": "minmax_kernel", "build.presence": "presence_kernel",
         "build.pack": "pack_kernel", "build.out_sort": "onesweep",
         "build.dedupe": "segment_kernel", "pr.fixup": "pr_fixup_kernel"}
    for phase, k in m.items():
        hit = [v for kk, v in t.items() if kk.startswith(k)]
        if hit:
            c4[phase] = {"kernel": k, "dram_bytes": int(max(hit)),
                         "source": "profiles/r2_ncu_dram_c4.txt (ncu --metrics dram__bytes)"}
    c4["pr.spmv"] = {"kernel": "pr_spmv_kernel", "dram_bytes": int(spmv_full),
                     "source": "profiles/r2_ncu_full_c4_pr_spmv.txt (r2n_full_c4_pr_spmv.ncu-rep)"}
    data["c4"] = c4
    path.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(json.dumps(c4, indent=1))


if __name__ == "__main__":
    main()
