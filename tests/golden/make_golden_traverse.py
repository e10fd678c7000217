"""Golden fixtures for the other CSR consumers, by running
the REAL reference (build container only): ``graphtables.sssp``,
``connected_components`` and ``k_core`` (algorithms.py:125-141, 232-248,
206-229) on the tables of ``make_golden.cases()`` plus graphs with isolated
nodes (``Graph.add_node``). Written to ``traverse.npz``:

* ``<case>/ids``            node ids ascending (the reference's node_ids())
* ``<case>/sources``        three source ids (first, middle, last)
* ``<case>/sssp``           [3, N] hop counts aligned with ids, -1 = None
* ``<case>/cc``             [N] component labels aligned with ids
* ``<case>/kcore<k>_ids``   survivor ids of k_core(g, k), k = 1..4
* ``<case>/kcore<k>_out_off``, ``_out_adj``  its CSR (export_csr layout)

Usage: PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_traverse.py
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(HERE))

from make_golden import EDGES, cases, export_csr, ref  # noqa: E402

SMALL = {"dup_collapse", "self_neg", "k4", "path10", "selfloop_tri", "selfloop_only",
         "two_cycle", "in_star", "random_neg_0", "random_neg_1", "random_neg_2",
         "random_500x20000", "sparse_ids", "int64_extremes", "rmat_s10_8192_11",
         "rmat_s11_16384_12_p"}


def graphs():
    for name, src, dst in cases():
        if name not in SMALL:
            continue
        t = ref.ColumnTable(EDGES, [np.asarray(src, np.int64), np.asarray(dst, np.int64)])
        yield name, ref.table_to_graph(t, ref.EdgeSpec("src", "dst")), (src, dst, None)
    # many components: a sparse random graph, and blocks whose id ranges
    # interleave (labels follow each component's smallest id)
    rng = np.random.default_rng(29)
    src = rng.integers(-1000, 2000, size=1400)
    dst = rng.integers(-1000, 2000, size=1400)
    t = ref.ColumnTable(EDGES, [src, dst])
    yield "sparse_forest", ref.table_to_graph(t, ref.EdgeSpec("src", "dst")), (src, dst, None)
    parts_s, parts_d = [], []
    for b in range(6):
        s = rng.integers(0, 50, size=120) * 6 + (5 - b)
        d = rng.integers(0, 50, size=120) * 6 + (5 - b)
        parts_s.append(s)
        parts_d.append(d)
    src, dst = np.concatenate(parts_s), np.concatenate(parts_d)
    t = ref.ColumnTable(EDGES, [src, dst])
    yield "interleaved_blocks", ref.table_to_graph(t, ref.EdgeSpec("src", "dst")), (src, dst, None)
    # isolated nodes (Graph.add_node): unreachable in sssp, singleton components
    rng = np.random.default_rng(31)
    src = rng.integers(0, 40, size=60)
    dst = rng.integers(0, 40, size=60)
    g = ref.from_edges(list(zip(src.tolist(), dst.tolist())))
    extra = [100, 101, -7]
    for x in extra:
        g.add_node(x)
    yield "isolated_extra", g, (src, dst, np.asarray(extra, np.int64))


def main():
    store = {}
    names = []
    for name, g, (src, dst, extra) in graphs():
        t0 = time.perf_counter()
        ids = np.asarray(g.node_ids(), dtype=np.int64)
        store[f"{name}/src"] = np.asarray(src, np.int64)
        store[f"{name}/dst"] = np.asarray(dst, np.int64)
        store[f"{name}/extra"] = extra if extra is not None else np.empty(0, np.int64)
        store[f"{name}/ids"] = ids
        n = ids.shape[0]
        sources = np.asarray([ids[0], ids[n // 2], ids[-1]], dtype=np.int64)
        store[f"{name}/sources"] = sources
        rows = []
        for s in sources.tolist():
            d = ref.sssp(g, int(s))
            rows.append([-1 if d[i] is None else d[i] for i in ids.tolist()])
        store[f"{name}/sssp"] = np.asarray(rows, dtype=np.int64)
        cc = ref.connected_components(g)
        store[f"{name}/cc"] = np.asarray([cc[i] for i in ids.tolist()], dtype=np.int64)
        for k in (1, 2, 3, 4):
            core = ref.k_core(g, k)
            cids, coo, coa, _, _ = export_csr(core)
            store[f"{name}/kcore{k}_ids"] = cids
            store[f"{name}/kcore{k}_out_off"] = coo
            store[f"{name}/kcore{k}_out_adj"] = coa
        names.append(name)
        print(f"{name}: N={n} components={int(store[f'{name}/cc'].max()) + 1 if n else 0} "
              f"({time.perf_counter() - t0:.1f}s)", flush=True)
    store["__names__"] = np.asarray(names)
    np.savez_compressed(HERE / "traverse.npz", **store)


if __name__ == "__main__":
    main()
