"""Golden fixtures for strongly connected components by
running the REAL reference's ``graphtables.scc`` (algorithms.py:144-203,
iterative Tarjan, labels dense by first occurrence over ascending ids) in the
build container. Written to ``scc.npz``: for every case ``<case>/src``,
``<case>/dst``, ``<case>/extra`` (isolated nodes added with Graph.add_node),
``<case>/ids`` (node ids ascending) and ``<case>/scc`` (labels aligned with
ids).

Cases: the graphs of make_golden_traverse (dup/self-loop/negative ids, K4,
paths, stars, R-MAT), plus cycle-rich ones: rings of rings, a long chain with
back edges, nested cycles whose smallest ids interleave, a dense random
digraph and a DAG.

Usage: PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_scc.py
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(HERE))

from make_golden import EDGES, ref  # noqa: E402
from make_golden_traverse import graphs as traverse_graphs  # noqa: E402

sys.setrecursionlimit(10000)


def extra_graphs():
    rng = np.random.default_rng(77)
    # rings of rings: 40 rings of 25 nodes, ring r links to ring r+1 one way
    s, d = [], []
    for r in range(40):
        base = r * 25
        for i in range(25):
            s.append(base + i)
            d.append(base + (i + 1) % 25)
        if r + 1 < 40:
            s.append(base + 3)
            d.append(base + 25 + 7)
    yield "ring_chain", np.asarray(s), np.asarray(d)
    # chain 0..1999 with back edges closing cycles of random length
    s = list(range(1999))
    d = list(range(1, 2000))
    for _ in range(60):
        a = int(rng.integers(10, 2000))
        s.append(a)
        d.append(a - int(rng.integers(1, 10)))
    yield "chain_back_edges", np.asarray(s), np.asarray(d)
    # interleaved cycles: component c holds ids c, c+7, c+14, ... (shuffled order)
    s, d = [], []
    for c in range(7):
        members = [c + 7 * k for k in range(30)]
        rng.shuffle(members)
        for i in range(30):
            s.append(members[i])
            d.append(members[(i + 1) % 30])
    perm = rng.permutation(len(s))
    yield "interleaved_cycles", np.asarray(s)[perm], np.asarray(d)[perm]
    # dense random digraph with negative ids
    s = rng.integers(-300, 300, size=4000)
    d = rng.integers(-300, 300, size=4000)
    yield "dense_random", s, d
    # sparse random digraph: many small SCCs
    s = rng.integers(0, 5000, size=6500)
    d = rng.integers(0, 5000, size=6500)
    yield "sparse_random", s, d
    # a DAG (edges low -> high): every node its own component
    a = rng.integers(0, 3000, size=9000)
    b = rng.integers(0, 3000, size=9000)
    keep = a != b
    yield "dag", np.minimum(a, b)[keep], np.maximum(a, b)[keep]


def main():
    store = {}
    names = []

    def record(name, g, src, dst, extra):
        t0 = time.perf_counter()
        ids = np.asarray(g.node_ids(), dtype=np.int64)
        lab = ref.scc(g)
        store[f"{name}/src"] = np.asarray(src, np.int64)
        store[f"{name}/dst"] = np.asarray(dst, np.int64)
        store[f"{name}/extra"] = extra if extra is not None else np.empty(0, np.int64)
        store[f"{name}/ids"] = ids
        store[f"{name}/scc"] = np.asarray([lab[i] for i in ids.tolist()], dtype=np.int64)
        names.append(name)
        nc = int(store[f"{name}/scc"].max()) + 1 if ids.size else 0
        print(f"{name}: N={ids.size} sccs={nc} ({time.perf_counter() - t0:.1f}s)", flush=True)

    for name, g, (src, dst, extra) in traverse_graphs():
        record(name, g, src, dst, extra)
    for name, src, dst in extra_graphs():
        t = ref.ColumnTable(EDGES, [np.asarray(src, np.int64), np.asarray(dst, np.int64)])
        record(name, ref.table_to_graph(t, ref.EdgeSpec("src", "dst")), src, dst, None)
    store["__names__"] = np.asarray(names)
    np.savez_compressed(HERE / "scc.npz", **store)


if __name__ == "__main__":
    main()
