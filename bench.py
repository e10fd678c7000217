#!/usr/bin/env python
"""Benchmark of the hot path: ToGraph -> PageRank x20 -> triangle count.

One "step" = one pass of the path over one synthetic edge table, by default
BASELINE.json configs[3] = C4 (R-MAT scale 26, 1.47 B int64 rows, seed 3,
permuted ids; the north-star config), triangles on its symmetrised version:
    table_to_graph  ->  pagerank(d=0.85, 20 iterations, fp64)  ->  triangle_count
`--config c2` runs configs[1] (69 M rows, + configs[2] triangles), `c5` the
uniform 2.0 B-row contrast graph (ToGraph + PageRank only).

`value` = input rows per second through the whole step (table already in
HBM); `e2e` = the same through the public Python API with host (pinned)
columns, host->device copy and result readback inside the timed region;
`phases` break the step into the three rows of the metric, each in its own
unit (build rows/s, PageRank edge-iterations/s, triangles undirected edges/s);
`roofline` = HBM roofline of the north-star kernels (build, PageRank) against
the measured copy peak (MEASURED_PEAKS.json); the triangle count is issue-
bound and reported as informational only.

`--gpus N` runs N ranks (one process per GPU, NCCL): re-executed under
torchrun when WORLD_SIZE is unset. Strong scaling: rank r generates rows
[rR/N, (r+1)R/N) of the config's own table, the sharded pipeline
(distributed.py) builds, ranks and counts it, and `value` = R / step time
(max over ranks).

`--impl reference` times the reference's own implementation (the unmodified
`graphtables` package installed in baseline/_ref, all host cores) on a
bounded same-family sample of the workload (see `reference_sample`).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

METRIC = "edges/s: table->CSR build, PageRank iteration, triangle count (+% HBM roofline)"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=["c1", "c2", "c4", "c5"], default="c4")
    p.add_argument("--iterations", type=int, default=20)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-scale", type=int, default=14,
                   help="R-MAT scale of the reference-arm / cpu_baseline sample (same a/b/c, "
                        "edge factor and id permutation as the config)")
    p.add_argument("--no-tsv", action="store_true")
    p.add_argument("--lanes", action="store_true",
                   help="PageRank on lane 1 next to the triangle count on lane 0 (measured: "
                        "no faster than serial at C2, both saturate the SMs)")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the measured-apart extras (SURVEY 8f rows): step kernels only")
    p.add_argument("--tsv-rows", type=int, default=4_000_000)
    p.add_argument("--sharded", action="store_true",
                   help="use the multi-GPU (distributed.py) pipeline even on one GPU")
    p.add_argument("--dry-run", action="store_true",
                   help="harness check on CPU: gloo ranks, the CPU restatement of the per-rank "
                        "primitives (tests/dist_cpu_ops.py), a small prefix of the config's "
                        "table; prints the JSON line shape with dry_run set (not a measurement)")
    p.add_argument("--dry-run-rows", type=int, default=200_000)
    return p.parse_args()


def shard_range(rank: int, world: int, rows: int):
    """Rows [lo, hi) of the config's table that rank `rank` of `world` holds
    (strong scaling: the ranks split one table)."""
    return rows * rank // world, rows * (rank + 1) // world


def torchrun_argv(gpus: int, argv, port: int):
    """The re-exec command line for `--gpus N` without torchrun."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1",
            "--master-port", str(port), str(Path(__file__).resolve()), *argv]


def maybe_reexec(args):
    """`--gpus N > 1` launched as a plain process: re-exec under torchrun (one
    rank per GPU); fail loudly when fewer GPUs are visible."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    import socket

    if not args.dry_run:
        import torch

        visible = torch.cuda.device_count()
        if visible < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but only {visible} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.execv(sys.executable, torchrun_argv(args.gpus, sys.argv[1:], port))


def peaks():
    path = REPO / "MEASURED_PEAKS.json"
    if path.exists():
        d = json.loads(path.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return PEAKS_FALLBACK


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def dist_ready():
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized()


def spec_for(name):
    from paper_1503_07881_b200.synth import CONFIGS

    return CONFIGS[name]


def has_tc(spec):
    """C5 (uniform, BASELINE configs[4]) is ToGraph + PageRank only."""
    from paper_1503_07881_b200.synth import UniformSpec

    return not isinstance(spec, UniformSpec)


def spec_desc(name, spec, rows):
    from paper_1503_07881_b200.synth import UniformSpec

    if isinstance(spec, UniformSpec):
        return (f"{name}: uniform iid (Erdos-Renyi) {rows} rows over {spec.n_nodes} ids "
                f"seed {spec.seed} (counter-based stand-in for synth.random_edges)")
    perm = (f"ids Feistel-permuted over [0, 2^{spec.scale}) (stand-in for the dense "
            f"remap)" if spec.permute else "ids unpermuted")
    return f"{name}: R-MAT s{spec.scale} {rows} rows a/b/c={spec.a}/{spec.b}/{spec.c} " \
           f"seed {spec.seed}, {perm}"


def workload_desc(config, spec, iterations):
    return (f"{spec_desc(config, spec, spec.rows)}; ToGraph + PageRank x{iterations} fp64"
            f"{' + triangles on the symmetrised graph' if has_tc(spec) else ''}")


# ------------------------------------------------------------------ reference

REF_DIR = REPO / "baseline" / "_ref"


def reference_sample(config, scale_cap):
    """The bounded sample the reference is timed on: the config's own
    generator family at a smaller size — R-MAT with the same a/b/c, seed, id
    permutation and edge factor (rows / 2^scale) at scale `scale_cap`; for
    the uniform C5, the same edge factor over 2^scale_cap ids. The
    reference's per-row cost grows with graph size (its triangle count most),
    so a rate measured on the sample overstates its rate on the full table:
    the GPU/CPU ratio is a lower bound."""
    from paper_1503_07881_b200.synth import RmatSpec, UniformSpec

    spec = spec_for(config)
    if isinstance(spec, UniformSpec):
        n = min(spec.n_nodes, 1 << scale_cap)
        rows = int(round(spec.rows * n / spec.n_nodes))
        return UniformSpec(n_nodes=n, rows=rows, seed=spec.seed)
    scale = min(scale_cap, spec.scale)
    rows = int(round(spec.rows * (1 << scale) / (1 << spec.scale)))
    return RmatSpec(scale=scale, rows=rows, a=spec.a, b=spec.b, c=spec.c, seed=spec.seed,
                    permute=spec.permute)


def load_reference():
    """The unmodified reference package from baseline/_ref (pip --target
    install of /root/reference/pkg), or None when it is not installed."""
    if not (REF_DIR / "graphtables" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import graphtables

    return graphtables


def run_reference_step(spec, iterations, src=None, dst=None):
    """One step of the path through the reference's public API
    (convert.py:128, algorithms.py:36/90) with workers=None (all cores), or
    through the numpy port when the reference is not installed."""
    from paper_1503_07881_b200.synth import spec_edges

    if src is None:
        src, dst = spec_edges(spec)
    ref = load_reference()
    t0 = time.perf_counter()
    if ref is not None:
        table = ref.ColumnTable(ref.Schema([("src", "int"), ("dst", "int")]), [src, dst])
        g = ref.table_to_graph(table, ref.EdgeSpec("src", "dst"))
        t1 = time.perf_counter()
        ref.pagerank(g, 0.85, iterations)
        t2 = time.perf_counter()
        tc = ref.triangle_count(g) if has_tc(spec) else None
        n, e, kind = g.node_count, g.edge_count, "reference"
    else:
        from oracle import reference_port as port

        g = port.build_csr(src, dst)
        t1 = time.perf_counter()
        port.pagerank_csr(g, 0.85, iterations)
        t2 = time.perf_counter()
        tc = port.triangle_count_csr(g) if has_tc(spec) else None
        n, e, kind = g.n, g.e, "port"
    t3 = time.perf_counter()
    return {"rows": int(src.shape[0]), "n": n, "e": e, "tc": tc, "kind": kind,
            "build_s": t1 - t0, "pr_s": t2 - t1, "tc_s": t3 - t2, "total_s": t3 - t0}


def cpu_info():
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cores": os.cpu_count() or 1, "model": model, "numpy": np.__version__}


def sample_desc(config, sample, r, iterations):
    what = ("graphtables (unmodified reference, baseline/_ref) table_to_graph + pagerank"
            if r["kind"] == "reference" else "oracle/reference_port.py (numpy port) build + pagerank")
    return (f"{spec_desc(config + '-family sample', sample, sample.rows)}: {what} x{iterations}"
            f"{' + triangle_count' if has_tc(sample) else ''}, workers=None (all cores); "
            f"N={r['n']} E={r['e']} triangles={r['tc']}")


def config_dict(args, spec, world):
    """The `config` object both arms print (identical: same workload, same
    keys; the graph's measured sizes go to `graph` in our arm's line)."""
    return {"workload": workload_desc(args.config, spec, args.iterations),
            "rows": spec.rows, "pagerank_iterations": args.iterations,
            "parallelism": f"sharded x{world} (NCCL)" if world > 1 else "single",
            "l2": "inputs larger than L2 (16*rows bytes >> 126 MB)"}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    spec = spec_for(args.config)
    sample = reference_sample(args.config, args.cpu_sample_scale)
    from paper_1503_07881_b200.synth import spec_edges

    src, dst = spec_edges(sample)
    for _ in range(args.warmup):
        run_reference_step(sample, args.iterations, src, dst)
    times = []
    last = None
    for _ in range(args.steps):
        last = run_reference_step(sample, args.iterations, src, dst)
        times.append(last["total_s"])
    mean = sum(times) / len(times)
    value = sample.rows / mean
    info = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic (seeded, host numpy)",
        "config": config_dict(args, spec, max(world, args.gpus)),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": info["cores"],
                         "kind": last["kind"], "sample": sample_desc(args.config, sample, last,
                                                                     args.iterations),
                         "cpu": info["model"], "numpy": info["numpy"],
                         "phases_s": {k: last[k] for k in ("build_s", "pr_s", "tc_s")}},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------- ours

def relational_extras(table, rows, args, pk):
    """device Select and Join on the bench's edge table
    (select src < median id: ~half the rows; join the edge table (probe) with
    a node-attribute table of up to 1M distinct src ids (build) on src). Wall time of the public
    call (device-resident result) and kernel time from the library phases."""
    import torch

    import paper_1503_07881_b200 as gt
    from paper_1503_07881_b200 import _native

    out = {}
    src = table.column("src")
    thr = int(torch.median(src[: 1 << 20]).item())
    n_attr = 1 << 20
    nodes = torch.unique(src[:: max(1, rows // (4 * n_attr))])[:n_attr]  # distinct keys
    attr = gt.ColumnTable(gt.Schema([("node", "int"), ("score", "int")]),
                          [nodes, torch.arange(nodes.shape[0], dtype=torch.int64,
                                               device=src.device)])
    cases = (("select", lambda: gt.select(table, gt.Predicate("src", "<", thr))),
             ("join", lambda: gt.join(attr, table, "node", "src")))
    for name, call in cases:
        res = call()  # warm-up
        n_out = res.n_rows
        del res
        _native.profile_reset()
        _native.profile_enable(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = call()
            del res
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
        ph = _native.profile_read()
        _native.profile_enable(False)
        kern = sum(v[0] for v in ph.values()) / args.steps
        kb = sum(v[2] for v in ph.values()) / args.steps
        out[name] = {"ms": wall * 1e3, "kernel_ms": kern, "rows_in": rows, "rows_out": n_out,
                     "value": rows / wall, "unit": "input rows/s (call time)",
                     "kernel_gbs": kb / (kern / 1e3) / 1e9 if kern > 0 else None,
                     "kernel_hbm_frac": (kb / (kern / 1e3) / 1e9 / pk["hbm_gbs"]
                                         if kern > 0 else None)}
    if not args.no_cpu_baseline:  # the oracle port (reference algorithm) on a 1M-row sample
        from oracle import reference_port as ref_port

        m = min(rows, 1_000_000)
        h_src = src[:m].cpu().numpy()
        h_nodes = attr.column("node").cpu().numpy()
        t0 = time.perf_counter()
        ref_port.select_indices(h_src, "int", [], "<", thr)
        t_sel = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref_port.join_indices(h_nodes.tolist(), h_src.tolist())
        t_join = time.perf_counter() - t0
        for name, t in (("select", t_sel), ("join", t_join)):
            out[name]["cpu_port"] = {"rows": m, "s": t, "value": m / t,
                                     "unit": "input rows/s", "cores": 1,
                                     "kind": "port (oracle/reference_port.py)"}
    return out


def tsv_extra(src, dst, args, pk):
    """§8f next #2: LoadTableTSV of an int64 edge TSV on the GPU (file read +
    H2D + parse, wall clock) and the parse kernels alone, on the first
    args.tsv_rows rows of the table; the host (reference-semantics) parser on
    a 10x smaller prefix as the CPU baseline."""
    import torch

    from paper_1503_07881_b200 import _native
    from paper_1503_07881_b200.tables import INT, Schema, load_tsv

    n = min(args.tsv_rows, int(src.shape[0]))
    a = src[:n].cpu().numpy()
    b = dst[:n].cpu().numpy()
    text = ("\n".join(f"{x}\t{y}" for x, y in zip(a.tolist(), b.tolist())) + "\n").encode()
    schema = Schema([("src", INT), ("dst", INT)])
    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / "edges.tsv"
        path.write_bytes(text)
        load_tsv(path, schema, device="cuda")  # warm
        _native.profile_reset()
        _native.profile_enable(True)
        reps = 3
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            t = load_tsv(path, schema, device="cuda")
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps
        ph = _native.profile_read()
        _native.profile_enable(False)
        assert t.n_rows == n
        k_ms = sum(v[0] for k, v in ph.items() if k.startswith("tsv.")) / reps
        k_bytes = sum(v[2] for k, v in ph.items() if k.startswith("tsv.")) / reps
        small = Path(tmp) / "small.tsv"
        m = max(1, n // 10)
        small.write_bytes(b"".join(text.splitlines(keepends=True)[:m]))
        t0 = time.perf_counter()
        load_tsv(small, schema)
        host_s = time.perf_counter() - t0
    return {"rows": n, "bytes": len(text), "e2e_ms": wall * 1e3,
            "value": n / wall, "unit": "rows/s (file -> HBM columns)",
            "kernel_ms": k_ms, "kernel_gbs": k_bytes / (k_ms / 1e3) / 1e9 if k_ms else None,
            "kernel_hbm_frac": (k_bytes / (k_ms / 1e3) / 1e9 / pk["hbm_gbs"]) if k_ms else None,
            "cpu_host_parser": {"rows": m, "value": m / host_s, "unit": "rows/s", "cores": 1}}


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    polled every 2 ms from a thread (nvidia-smi -lms as the fallback)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = None
        self.thread = None
        self.samples = []  # (sm_mhz, max_mhz, reasons)

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.dev)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def __enter__(self):
        import threading

        try:
            nv, h = self._nvml_handle()
            bits = [getattr(nv, "nvmlClocksEventReason" + n, None) for n in
                    ("HwSlowdown", "HwThermalSlowdown", "SwThermalSlowdown", "SwPowerCap")]
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        break
                    self.samples.append((sm, mx, {n for n, b in zip(self.NAMES, bits)
                                                  if b is not None and rs & b}))
                    self.stop.wait(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.thread is None and self.path and os.path.exists(self.path):
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm, mx = float(parts[0]), float(parts[1])
                except ValueError:
                    continue
                self.samples.append((sm, mx, {n for n, v in zip(self.NAMES, parts[2:6])
                                              if v.lower().startswith("active")}))
            os.unlink(self.path)
        if not self.samples:
            return None
        reasons = set().union(*(r for _, _, r in self.samples))
        return {"sm_mhz": float(np.median([s for s, _, _ in self.samples])),
                "sm_max_mhz": float(max(m for _, m, _ in self.samples)),
                "reasons": sorted(reasons), "samples": len(self.samples),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


def roofline_block(args, phases, steps, rows, n, e, world, pk, elapsed_ms):
    """HBM roofline of the north-star kernels, per GPU.

    * build: B_kern = the element-count bytes each build kernel is credited
      with (its contract I/O: DESIGN.md §4.1), and B_min = 16R + 8N +
      2(8(N+1) + 4E) (read both columns once, write ids and both CSRs);
    * PageRank: B_PR = 12E + 32N per iteration (int32 in-adjacency + fp64
      gather per edge; offsets, 1/outdeg, score and contrib per node),
      over the iteration kernels' time and over the whole call;
    * the top-level kernel fields are the longest-running HBM-bound kernel of
      those phases; its `traffic` is ncu dram__bytes per launch from the
      committed C4 capture (profiles/ncu_traffic.json) when one matches;
    * triangles: issue-bound (bitmap / hash probes in shared memory), no HBM
      fraction is claimed; see `phases.triangles`.
    At N > 1 the bytes are per GPU (R/N rows, E/N edges, N/N rows of PR)."""
    peak = pk["hbm_gbs"]

    def grp(prefixes, exclude=()):
        ms = sum(v[0] for k, v in phases.items()
                 if k.startswith(prefixes) and not k.startswith(exclude)) / steps
        by = sum(v[2] for k, v in phases.items()
                 if k.startswith(prefixes) and not k.startswith(exclude)) / steps
        return ms, by

    g = max(world, 1)
    b_ms, b_kern = grp(("build.", "sort.", "dist."), exclude=("build.h2d",))
    b_min = (16.0 * rows + 8.0 * n + 2 * (8.0 * (n + 1) + 4.0 * e)) / g
    pr_ms, _ = grp(("pr.",))
    it_ms, _ = grp(("pr.spmv", "pr.fixup", "pr.step", "pr.finalize"))
    b_pr = (12.0 * e + 32.0 * n) * args.iterations / g
    out = {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": pk["source"],
           "phases": {}}

    def frac(by, ms):
        return (by / (ms / 1e3) / 1e9 / peak) if ms > 0 else None

    out["phases"]["build"] = {
        "ms": b_ms, "b_kern_gb": b_kern / 1e9, "b_min_gb": b_min / 1e9,
        "achieved_gbs": b_kern / (b_ms / 1e3) / 1e9 if b_ms else None,
        "frac": frac(b_kern, b_ms), "compulsory_frac": frac(b_min, b_ms)}
    out["phases"]["pagerank"] = {
        "ms": pr_ms, "iterations_ms": it_ms, "b_pr_gb_per_iteration": b_pr / args.iterations / 1e9,
        "achieved_gbs": b_pr / (it_ms / 1e3) / 1e9 if it_ms else None,
        "frac": frac(b_pr, it_ms), "frac_whole_call": frac(b_pr, pr_ms)}
    t_ms, _ = grp(("tc.",))
    out["phases"]["triangles"] = {
        "ms": t_ms, "bound": "issue (informational)",
        "note": "probes are shared-memory bitmap/hash lookups: no HBM fraction claimed; "
                "ncu sm__throughput and instruction counts in profiles/"}
    hbm = {k: v for k, v in phases.items()
           if k.startswith(("build.", "sort.", "pr.", "dist.")) and not k.startswith("build.h2d")
           and v[2] > 0}
    if hbm:
        name, (ms, cnt, by) = max(hbm.items(), key=lambda kv: kv[1][0])
        ach = by / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        tr = ncu_traffic(args.config, name)
        out.update({"kernel": name, "achieved": ach, "frac": ach / peak,
                    "traffic": (tr or {}).get("bytes_per_launch"), "traffic_source": tr,
                    "bytes_per_launch": by / max(cnt, 1), "ms_per_launch": ms / max(cnt, 1),
                    "share_of_step": (ms / steps) / (elapsed_ms / steps)})
    return out


def ours_arm(args):
    import torch

    rank, world, local = dist_env()
    os.environ["GT_DEVICE"] = str(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        print(f"[bench rank {rank}/{world}] NCCL process group up on cuda:{local} "
              f"(nccl {'.'.join(map(str, torch.cuda.nccl.version()))})", file=sys.stderr,
              flush=True)

    import paper_1503_07881_b200 as gt
    from paper_1503_07881_b200 import _native
    from paper_1503_07881_b200.synth import rmat_device

    spec = spec_for(args.config)
    # strong scaling: rank r holds rows [rR/N, (r+1)R/N) of the config's table
    lo, hi = shard_range(rank, world, spec.rows)
    src, dst = rmat_device(spec, device=f"cuda:{local}", start=lo, rows=hi - lo)
    table = gt.edge_table(src, dst)
    edge_spec = gt.EdgeSpec("src", "dst")
    stream = torch.cuda.ExternalStream(_native.stream_handle(), device=dev)
    iters = args.iterations
    state = {}

    sharded = world > 1 or args.sharded
    with_tc = has_tc(spec)
    if sharded and not dist_ready():
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    if not sharded:
        def step():
            g = gt.table_to_graph(table, edge_spec)
            out = state.get("scores")
            if out is None or out.shape[0] != g.node_count:
                out = state["scores"] = torch.empty(g.node_count, dtype=torch.float64, device=dev)
            if with_tc and args.lanes:  # PageRank (lane 1) next to the count (lane 0)
                _, tc = gt.pagerank_and_triangles(g, 0.85, iters, scores_out_ptr=out.data_ptr())
            else:
                gt.pagerank_device(g, 0.85, iters, out.data_ptr())
                tc = gt.triangle_count(g) if with_tc else None
            state.update(n=g.node_count, e=g.edge_count, tc=tc,
                         m=_native.undirected_edges(g.handle) if with_tc else None)
            del g
    else:
        from paper_1503_07881_b200 import distributed as D

        ops = D.NativeOps(dev)

        stage_ms = state.setdefault("stage_ms", {"build": 0.0, "pagerank": 0.0, "triangles": 0.0})

        def step():
            # stage wall times (every NativeOps call synchronises, so these are
            # device time plus the host's collective orchestration); the
            # library's phase names cannot tell the orientation's sorts
            # (dist.sort) from the build's
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sg = D.build_csr(src, dst, ops=ops)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            D.pagerank(sg, 0.85, iters, ops=ops)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            tc = D.triangle_count(sg, ops=ops) if with_tc else None
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            stage_ms["build"] += (t1 - t0) * 1e3
            stage_ms["pagerank"] += (t2 - t1) * 1e3
            stage_ms["triangles"] += (t3 - t2) * 1e3
            state.update(n=sg.n, e=sg.e, tc=tc)
            del sg

    for _ in range(args.warmup):
        step()
    if sharded:
        state["stage_ms"].update(build=0.0, pagerank=0.0, triangles=0.0)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([x], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    # ---- timed region: K steps, CUDA events on the library stream ----------
    _native.profile_enable(True)
    _native.profile_reset()
    launches0 = _native.launch_count()
    with ClockSampler(local) as clocks:
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    launches = _native.launch_count() - launches0
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    phases = _native.profile_read()
    _native.profile_enable(False)

    rows = spec.rows
    ms_per_step = elapsed_ms / args.steps
    value = rows / (ms_per_step / 1e3)
    n, e, tc = state["n"], state["e"], state["tc"]
    m_und = state.get("m")

    pk = peaks()

    def group(prefixes):
        ms = sum(v[0] for k, v in phases.items() if k.startswith(prefixes)) / args.steps
        return ms

    b_ms = group(("build.", "sort.", "dist."))
    p_ms = group(("pr.",))
    t_ms = group(("tc.",))
    if sharded:  # stage wall times (see step), max over ranks
        b_ms, p_ms, t_ms = (max_over_ranks(state["stage_ms"][k] / args.steps)
                            for k in ("build", "pagerank", "triangles"))
    phase_line = {
        "build": {"ms": b_ms, "value": rows / (b_ms / 1e3) if b_ms else None, "unit": "rows/s"},
        "pagerank": {"ms": p_ms, "value": e * iters / (p_ms / 1e3) if p_ms else None,
                     "unit": "edge-iterations/s"},
        "triangles": {"ms": t_ms, "unit": "undirected edges/s (m / t_TC)",
                      "value": m_und / (t_ms / 1e3) if t_ms and m_und else None,
                      "e_d_value": e / (t_ms / 1e3) if t_ms else None,
                      "e_d_unit": "directed E_d/s (reference bench unit)",
                      "triangles": tc, "undirected_edges": m_und},
    }
    kernels = {}
    for name, (ms, cnt, by) in phases.items():
        kernels[name] = {"ms_per_step": ms / args.steps, "launches_per_step": cnt / args.steps,
                         "gbs": (by / (ms / 1e3) / 1e9) if ms > 0 and by > 0 else None}
    roofline = roofline_block(args, phases, args.steps, rows, n, e, world, pk, elapsed_ms)

    # ---- §8f next #1: graph -> edge table export (device), measured apart ----
    extras = {}
    if not sharded and not args.no_extras:
        # side measurements outside the timed step: at C5 the update rebuild
        # does not fit beside the bench table; record that instead of losing
        # the step line
        try:
            g_x = gt.table_to_graph(table, edge_spec)
            _native.profile_reset()
            _native.profile_enable(True)
            for _ in range(args.steps):
                gt.graph_to_edge_table(g_x, device=True)
            ph_x = _native.profile_read()
            _native.profile_enable(False)
            ms_x, _, by_x = ph_x.get("export.edges", (0.0, 0, 0.0))
            if ms_x > 0:
                ms_x /= args.steps
                extras["graph_to_edge_table"] = {
                    "ms": ms_x, "value": g_x.edge_count / (ms_x / 1e3), "unit": "edges/s",
                    "achieved_gbs": by_x / args.steps / (ms_x / 1e3) / 1e9,
                    "hbm_frac": by_x / args.steps / (ms_x / 1e3) / 1e9 / pk["hbm_gbs"]}
            # §8f next #4: the other CSR consumers on the same graph (wall time of
            # the public call, results to the host; kernel time from the phases)
            from paper_1503_07881_b200.algorithms import _ids_only

            source = int(_ids_only(g_x)[0])
            for name, call in (("sssp", lambda: gt.sssp(g_x, source)),
                               ("connected_components", lambda: gt.connected_components(g_x)),
                               ("scc", lambda: gt.scc(g_x)),
                               ("k_core_k8", lambda: gt.k_core(g_x, 8))):
                call()  # warm-up
                _native.profile_reset()
                _native.profile_enable(True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(args.steps):
                    call()
                wall = (time.perf_counter() - t0) / args.steps
                kern = sum(v[0] for v in _native.profile_read().values()) / args.steps
                _native.profile_enable(False)
                extras[name] = {"ms": wall * 1e3, "kernel_ms": kern,
                                "value": g_x.edge_count / wall, "unit": "edges/s (E / call time)"}
            # batched dynamic update: delete 1% of the rows' edges, add 1% new rows
            k_up = max(1, rows // 100)
            gen = torch.Generator(device=src.device).manual_seed(11)
            pick = torch.randint(0, rows, (k_up,), device=src.device, generator=gen)
            dels = (src[pick], dst[pick])
            adds = (src[torch.randint(0, rows, (k_up,), device=src.device, generator=gen)],
                    dst[torch.randint(0, rows, (k_up,), device=src.device, generator=gen)])
            _native.profile_reset()
            _native.profile_enable(True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                g_x.apply_updates(add=adds, delete=dels)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / args.steps
            kern = sum(v[0] for v in _native.profile_read().values()) / args.steps
            _native.profile_enable(False)
            extras["update_batch"] = {"ms": wall * 1e3, "kernel_ms": kern, "added": k_up,
                                      "deleted": k_up, "edges": g_x.edge_count,
                                      "value": g_x.edge_count / wall,
                                      "unit": "graph edges/s (apply_updates call time, rebuild)"}
            del g_x
            extras.update(relational_extras(table, rows, args, pk))
            if not args.no_tsv:
                extras["load_tsv"] = tsv_extra(src, dst, args, pk)
        except (MemoryError, torch.cuda.OutOfMemoryError) as exc:
            g_x = None
            _native.profile_enable(False)
            torch.cuda.empty_cache()
            extras["skipped"] = f"out of device memory after {sorted(extras)}: {exc}"

    # ---- end to end through the public API with host buffers ---------------
    e2e = None
    if not args.no_e2e:
        my_rows = hi - lo
        h_src = torch.empty(my_rows, dtype=torch.int64, pin_memory=True)
        h_dst = torch.empty(my_rows, dtype=torch.int64, pin_memory=True)
        h_src.copy_(src)
        h_dst.copy_(dst)
        host_table = gt.edge_table(h_src.numpy(), h_dst.numpy())
        del table, src, dst
        state.clear()
        torch.cuda.empty_cache()

        pipe = {"next": None}
        if not sharded:
            def e2e_step():
                # pipelined ingest: this step's table was copied (pinned host ->
                # HBM, side stream) while the previous step computed; the next
                # step's copy is issued first, so that it overlaps this step's
                # build and PageRank: the copy engine's HBM writes flush L2, and
                # the triangle count (whose suffix reads live in L2) measured
                # 824 ms instead of 680 when the copy ran under it (e2e 1178 vs
                # 1036 ms per C4 step, scripts/probe_e2e.py)
                cur = pipe["next"] if pipe["next"] is not None else host_table.prefetch()
                if not os.environ.get("BENCH_E2E_SERIAL"):
                    pipe["next"] = host_table.prefetch()
                g = gt.table_to_graph(cur, edge_spec)
                del cur
                # scores stay in HBM until the count is done, then one D2H read:
                # a read issued while the next table's H2D copy is in flight
                # waited for that copy (C4: +410 ms), one after the count does not
                n_ = g.node_count
                d_sc = pipe.get("d_sc")
                if d_sc is None or d_sc.shape[0] < n_:
                    d_sc = pipe["d_sc"] = torch.empty(n_, dtype=torch.float64, device=dev)
                    pipe["h_sc"] = [torch.empty(n_, dtype=torch.float64, pin_memory=True)
                                    for _ in range(2)]
                if with_tc and args.lanes:
                    _, tc_ = gt.pagerank_and_triangles(g, 0.85, iters,
                                                       scores_out_ptr=d_sc.data_ptr())
                else:
                    gt.pagerank_device(g, 0.85, iters, d_sc.data_ptr())
                    tc_ = gt.triangle_count(g) if with_tc else None
                pipe["flip"] = 1 - pipe.get("flip", 0)
                pr = pipe["h_sc"][pipe["flip"]][:n_]
                pr.copy_(d_sc[:n_])  # device -> pinned host, synchronous
                return pr, tc_
        else:
            def e2e_step():
                s_d = h_src.to(dev, non_blocking=True)
                d_d = h_dst.to(dev, non_blocking=True)
                sg = D.build_csr(s_d, d_d, ops=ops)
                pr = D.pagerank(sg, 0.85, iters, ops=ops).cpu()
                tc_ = D.triangle_count(sg, ops=ops) if with_tc else None
                return pr, tc_

        # warm-up in the timed loop's pattern (the previous step's result
        # alive while the next runs), so that the pinned result buffers the
        # steady state rotates through are allocated before timing
        prev = None
        for _ in range(max(2, min(args.warmup, 3))):
            prev = e2e_step()
        del prev
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pr, tc2 = e2e_step()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()  # the copy issued by the last step completes inside the region
        wall = time.perf_counter() - t0
        barrier()
        e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3) / args.steps)
        assert tc2 == tc, "e2e triangle count differs from the device-resident run"
        e2e = {"value": rows / (e2e_ms / 1e3), "unit": "rows/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": 16 * rows,
               "pipelined": (None if sharded else
                             "ColumnTable.prefetch: each step's table is copied from pinned "
                             "host memory on a side stream while the previous step computes; "
                             "one copy per timed step, all inside the timed region"),
               "d2h_bytes_per_step": (8 * n + 8) if not sharded else (8 * n + 8) * world,
               "api": (("host ColumnTable.prefetch -> table_to_graph -> pagerank_device"
                        if not sharded else "distributed.build_csr(host slice) -> pagerank")
                       + (" -> triangle_count" if with_tc else "")
                       + (" -> scores to pinned host" if not sharded else ""))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = reference_sample(args.config, args.cpu_sample_scale)
        from paper_1503_07881_b200.synth import spec_edges

        s_src, s_dst = spec_edges(sample)
        reps = [run_reference_step(sample, iters, s_src, s_dst) for _ in range(2)]
        tot = sum(r["total_s"] for r in reps)
        info = cpu_info()
        cpu = {"value": sample.rows * len(reps) / tot, "unit": "rows/s", "cores": info["cores"],
               "kind": reps[-1]["kind"],
               "sample": sample_desc(args.config, sample, reps[-1], iters)
                         + f"; {len(reps)} reps, {tot:.2f} s",
               "cpu": info["model"],
               "phases_s": {k: reps[-1][k] for k in ("build_s", "pr_s", "tc_s")}}

    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int64+f64", "data": "synthetic (generated on device, seeded)",
        "config": config_dict(args, spec, world),
        "graph": {"nodes": n, "edges": e, "undirected_edges": m_und, "triangles": tc},
        "phases": phase_line, "extras": extras, "kernels": kernels, "roofline": roofline,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_ready():
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def ncu_traffic(config, phase):
    """DRAM bytes (read + write) per launch of the phase's kernel, from the
    committed `ncu --set full` capture summarised in profiles/ncu_traffic.json
    (scripts/ncu_traffic.py writes it); None when no capture matches."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            entry = json.load(f).get(config, {}).get(phase)
    except (OSError, ValueError):
        return None
    if not entry:
        return None
    return {"bytes_per_launch": entry["dram_bytes"], "kernel": entry["kernel"],
            "source": entry["source"]}


def dry_run_arm(args):
    """The multi-rank harness on CPU (gloo): strong-scaling shards of the
    config's table (a prefix of it), the sharded pipeline of distributed.py
    over the CPU restatement of its primitives, max-over-ranks timing, one
    JSON line from rank 0. Checks the launch plumbing (torchrun re-exec,
    rank/world, shard ranges, collectives), never a performance number."""
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(REPO / "tests"))
    from dist_cpu_ops import CpuOps

    from paper_1503_07881_b200 import distributed as D
    from paper_1503_07881_b200.synth import spec_edges

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29534")
        dist.init_process_group("gloo", rank=0, world_size=1)
    spec = spec_for(args.config)
    rows = min(args.dry_run_rows, spec.rows)
    lo, hi = shard_range(rank, world, rows)
    src_all, dst_all = spec_edges(spec, rows)
    src = torch.from_numpy(src_all[lo:hi].copy())
    dst = torch.from_numpy(dst_all[lo:hi].copy())
    ops = CpuOps()
    state = {}

    def step():
        sg = D.build_csr(src, dst, ops=ops)
        D.pagerank(sg, 0.85, args.iterations, ops=ops)
        tc = D.triangle_count(sg, ops=ops) if has_tc(spec) else None
        state.update(n=sg.n, e=sg.e, tc=tc)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dist.barrier()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) * 1e3 / max(args.steps, 1)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": rows / (ms / 1e3), "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64+f64", "data": "synthetic",
            "dry_run": "gloo ranks on CPU with tests/dist_cpu_ops.py: harness check only",
            "config": config_dict(args, spec, world) | {"dry_run_rows": rows},
            "graph": {"nodes": state["n"], "edges": state["e"], "triangles": state["tc"]},
            "shard": [shard_range(r, world, rows) for r in range(world)]}), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    maybe_reexec(args)
    if args.dry_run:
        return dry_run_arm(args)
    if args.impl == "reference":
        return reference_arm(args)
    return ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())
