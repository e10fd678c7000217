"""Golden fixtures for batched dynamic updates by running
the REAL reference's Graph mutation calls (graphs.py:92-144) in the build
container. For every case: a base edge table, a batch (del_nodes,
deletions, add_nodes, additions — mixing present and absent ids / edges,
new ids, duplicates, self-loops), applied to the reference Graph as
del_node* -> del_edge* -> add_node* -> add_edge*, and the resulting CSR in
the export_csr layout. Written to ``updates.npz``.

Usage: PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_updates.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(HERE))

from make_golden import EDGES, export_csr, ref  # noqa: E402
from paper_1503_07881_b200.synth import rmat_edges  # noqa: E402


def batch(rng, src, dst, scale):
    ids = np.unique(np.concatenate([src, dst]))
    k = max(1, ids.size // 50)
    del_nodes = np.concatenate([rng.choice(ids, size=k), [ids.max() + 1000]])
    pick = rng.integers(0, src.size, size=max(1, src.size // 20))
    del_s = np.concatenate([src[pick], rng.integers(-scale, scale, size=5)])
    del_d = np.concatenate([dst[pick], rng.integers(-scale, scale, size=5)])
    add_nodes = np.concatenate([rng.integers(-scale, 2 * scale, size=4), del_nodes[:1]])
    m = max(1, src.size // 10)
    add_s = np.concatenate([rng.integers(-scale, 2 * scale, size=m), src[:3], [7, 7]])
    add_d = np.concatenate([rng.integers(-scale, 2 * scale, size=m), dst[:3], [7, 7]])
    return [np.asarray(a, np.int64) for a in (del_nodes, del_s, del_d, add_nodes, add_s, add_d)]


def main():
    rng = np.random.default_rng(4242)
    store = {}
    names = []
    cases = [("rand_small", rng.integers(0, 30, 60), rng.integers(0, 30, 60), 30),
             ("rand_neg", rng.integers(-500, 500, 3000), rng.integers(-500, 500, 3000), 500)]
    s, d = rmat_edges(11, 16384, seed=12, permute=True)
    cases.append(("rmat_s11", s, d, 2048))
    s, d = rmat_edges(13, 60000, seed=13, permute=False)
    cases.append(("rmat_s13", s, d, 8192))
    for name, src, dst, scale in cases:
        src = np.asarray(src, np.int64)
        dst = np.asarray(dst, np.int64)
        t = ref.ColumnTable(EDGES, [src, dst])
        g = ref.table_to_graph(t, ref.EdgeSpec("src", "dst"))
        dn, ds, dd, an, as_, ad = batch(rng, src, dst, scale)
        for x in dn.tolist():
            g.del_node(x)
        for a, b in zip(ds.tolist(), dd.tolist()):
            g.del_edge(a, b)
        for x in an.tolist():
            g.add_node(x)
        for a, b in zip(as_.tolist(), ad.tolist()):
            g.add_edge(a, b)
        ids, oo, oa, io, ia = export_csr(g)
        for key, val in (("src", src), ("dst", dst), ("del_nodes", dn), ("del_src", ds),
                         ("del_dst", dd), ("add_nodes", an), ("add_src", as_), ("add_dst", ad),
                         ("ids", ids), ("out_off", oo), ("out_adj", oa), ("in_off", io),
                         ("in_adj", ia)):
            store[f"{name}/{key}"] = val
        names.append(name)
        print(name, "N", ids.size, "E", oa.size)
    store["__names__"] = np.asarray(names)
    np.savez_compressed(HERE / "updates.npz", **store)


if __name__ == "__main__":
    main()
