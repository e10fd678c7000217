"""CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the algorithms of the reference package
``graphtables`` (``/root/reference/pkg/src/graphtables``) on the path
ToGraph -> PageRank / triangle count, step for step and with the same
worker-pool discipline, so that it can

* check the CUDA path (tests/, ``__graft_entry__.smoke``), and
* serve as the reference-side CPU baseline (``bench.py --impl reference`` and
  the ``cpu_baseline`` leg), the reference itself being pure Python that is
  not present on the GPU box.

It is pinned against outputs of the real reference, run in the build
container by ``tests/golden/make_golden.py`` (fixtures under
``tests/golden/``; checked by ``tests/test_oracle_golden.py``).

Nothing in the product package imports this module.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

_PARALLEL_SORT_MIN = 1 << 17  # parallel.py:17-19
_LOW32 = np.uint64(0xFFFFFFFF)


# ---------------------------------------------------------------- parallel.py

def resolve_workers(workers):
    """parallel.py:22-28 — None means all logical cores."""
    if workers is None:
        return os.cpu_count() or 1
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    return workers


def split_ranges(n, parts):
    """parallel.py:31-36 — at most `parts` contiguous near-equal ranges."""
    parts = max(1, min(parts, n))
    bounds = np.linspace(0, n, parts + 1).astype(np.int64)
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(parts)
            if bounds[i] < bounds[i + 1]]


def run_partitioned(fn, ranges, workers):
    """parallel.py:39-49 — results in range order."""
    if workers <= 1 or len(ranges) <= 1:
        return [fn(a, b) for a, b in ranges]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        futures = [pool.submit(fn, a, b) for a, b in ranges]
        return [f.result() for f in futures]


def parallel_sort(values, workers):
    """parallel.py:52-93 — splitter buckets sorted by threads; == np.sort."""
    n = values.shape[0]
    if workers <= 2 or n < _PARALLEL_SORT_MIN:
        return np.sort(values, kind="quicksort")
    parts = min(workers, 16)
    sample = np.sort(values[:: max(1, n // (parts * 32))])
    picks = np.linspace(0, sample.size - 1, parts + 1).astype(np.int64)[1:-1]
    splitters = np.unique(sample[picks])
    buckets = []
    lower = None
    for i in range(splitters.size + 1):
        if i == 0:
            mask = values < splitters[0]
        elif i == splitters.size:
            mask = values >= lower
        else:
            mask = (values >= lower) & (values < splitters[i])
        lower = splitters[i] if i < splitters.size else lower
        part = values[mask]
        if part.shape[0]:
            buckets.append(part)
    out = np.empty_like(values)
    offsets = np.concatenate(([0], np.cumsum([b.shape[0] for b in buckets]))).tolist()

    def sort_bucket(i, bucket):
        out[offsets[i]:offsets[i + 1]] = np.sort(bucket, kind="quicksort")

    run_partitioned(sort_bucket, list(enumerate(buckets)), workers)
    return out


# ----------------------------------------------------------------- convert.py

def dense_ids(src, dst):
    """convert.py:45-59 — sorted distinct ids + dense rank arrays."""
    cat = np.concatenate((src, dst))
    nodes = np.unique(cat)
    lo, hi = int(nodes[0]), int(nodes[-1])
    width = hi - lo + 1
    if width <= max(1 << 24, 2 * cat.shape[0]) and nodes.shape[0] < (1 << 31):
        lut = np.empty(width, dtype=np.int64)
        lut[nodes - lo] = np.arange(nodes.shape[0], dtype=np.int64)
        return nodes, lut[src - lo], lut[dst - lo]
    return nodes, np.searchsorted(nodes, src), np.searchsorted(nodes, dst)


def pack(a, b):
    """convert.py:62-63."""
    return (a.astype(np.uint64) << np.uint64(32)) | b.astype(np.uint64)


def unpack(packed):
    """convert.py:66-68."""
    return ((packed >> np.uint64(32)).astype(np.int64),
            (packed & _LOW32).astype(np.int64))


def sorted_unique_pairs(a, b, n_nodes, workers, unique=False):
    """convert.py:71-89 — lexicographically sorted (deduplicated) pairs."""
    if n_nodes < (1 << 32):
        packed = parallel_sort(pack(a, b), workers)
        if not unique and packed.shape[0]:
            keep = np.empty(packed.shape[0], dtype=bool)
            keep[0] = True
            np.not_equal(packed[1:], packed[:-1], out=keep[1:])
            packed = packed[keep]
        return unpack(packed)
    order = np.lexsort((b, a))
    a_s, b_s = a[order], b[order]
    if not unique and a_s.shape[0]:
        keep = np.empty(a_s.shape[0], dtype=bool)
        keep[0] = True
        keep[1:] = (a_s[1:] != a_s[:-1]) | (b_s[1:] != b_s[:-1])
        a_s, b_s = a_s[keep], b_s[keep]
    return a_s, b_s


@dataclass
class CSR:
    """The reference graph in pool form (convert.py:154-174): ids ascending,
    out/in offsets (int64) and out/in pools of original ids."""

    ids: np.ndarray
    out_off: np.ndarray
    out_adj: np.ndarray
    in_off: np.ndarray
    in_adj: np.ndarray

    @property
    def n(self):
        return int(self.ids.shape[0])

    @property
    def e(self):
        return int(self.out_adj.shape[0])


def build_csr(src, dst, workers=None) -> CSR:
    """convert.py:128-175 without the per-node NodeRecord dict.

    The pools are filled from sorted runs (convert.py:92-125); because runs
    arrive sorted and every cursor lands exactly on its degree, pool[i] equals
    nodes[dst_dense] of the i-th sorted pair, which is what is returned.
    """
    workers = resolve_workers(workers)
    src = np.asarray(src, dtype=np.int64).copy()
    dst = np.asarray(dst, dtype=np.int64).copy()
    if src.shape[0] == 0:
        z = np.zeros(1, dtype=np.int64)
        e = np.empty(0, dtype=np.int64)
        return CSR(e, z, e, z.copy(), e.copy())
    nodes, src_d, dst_d = dense_ids(src, dst)
    n = nodes.shape[0]
    out_src, out_dst = sorted_unique_pairs(src_d, dst_d, n, workers)
    in_dst, in_src = sorted_unique_pairs(out_dst, out_src, n, workers, unique=True)
    out_deg = np.bincount(out_src, minlength=n)
    in_deg = np.bincount(in_dst, minlength=n)
    out_off = np.concatenate(([0], np.cumsum(out_deg))).astype(np.int64)
    in_off = np.concatenate(([0], np.cumsum(in_deg))).astype(np.int64)
    return CSR(nodes.astype(np.int64), out_off, nodes[out_dst].astype(np.int64),
               in_off, nodes[in_src].astype(np.int64))


# -------------------------------------------------------------- algorithms.py

def pagerank_csr(g: CSR, damping=0.85, iterations=10, workers=None) -> np.ndarray:
    """algorithms.py:36-87 — scores aligned with g.ids (ascending)."""
    if not 0.0 < damping < 1.0:
        raise ValueError(f"damping must be in (0, 1), got {damping}")
    if iterations < 1:
        raise ValueError(f"iterations must be >= 1, got {iterations}")
    if g.n == 0:
        raise ValueError("pagerank needs a non-empty graph")
    workers = resolve_workers(workers)
    n = g.n
    out_deg = np.diff(g.out_off)
    in_lens = np.diff(g.in_off)
    in_flat = np.searchsorted(g.ids, g.in_adj)  # _DenseIndex.dense, algorithms.py:31-33
    in_off = g.in_off
    edge_dst = np.repeat(np.arange(n, dtype=np.int64), in_lens)
    dangling_mask = out_deg == 0
    inv_out = np.zeros(n, dtype=np.float64)
    np.divide(1.0, out_deg, where=~dangling_mask, out=inv_out)
    node_ranges = split_ranges(n, workers)
    score = np.full(n, 1.0 / n, dtype=np.float64)
    new_score = np.empty(n, dtype=np.float64)
    for _ in range(iterations):
        contrib = score * inv_out
        dangling = float(score[dangling_mask].sum())
        base = (1.0 - damping) / n + damping * (dangling / n)

        def accumulate(a, b, contrib=contrib, base=base, new_score=new_score):
            lo, hi = int(in_off[a]), int(in_off[b])
            sums = np.bincount(edge_dst[lo:hi] - a, weights=contrib[in_flat[lo:hi]],
                               minlength=b - a)
            new_score[a:b] = base + damping * sums

        run_partitioned(accumulate, node_ranges, workers)
        score, new_score = new_score, score
    return score


def undirected_dense(g: CSR):
    """graphs.py:163-167 per node, as dense indices (algorithms.py:102)."""
    n = g.n
    out_d = np.searchsorted(g.ids, g.out_adj)
    in_d = np.searchsorted(g.ids, g.in_adj)
    und = []
    for i in range(n):
        merged = np.union1d(in_d[g.in_off[i]:g.in_off[i + 1]],
                            out_d[g.out_off[i]:g.out_off[i + 1]])
        und.append(merged[merged != i])
    return und


def orientation_dense(g: CSR, und=None):
    """algorithms.py:102-108 — undirected degree and higher(i) (id order)."""
    n = g.n
    if und is None:
        und = undirected_dense(g)
    deg = np.asarray([u.shape[0] for u in und], dtype=np.int64)
    by_rank = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, dtype=np.int64)
    rank[by_rank] = np.arange(n)
    higher = [u[rank[u] > rank[i]] for i, u in enumerate(und)]
    return deg, higher


def triangle_count_csr(g: CSR, workers=None, und=None) -> int:
    """algorithms.py:90-119 — one intersect1d per oriented edge."""
    workers = resolve_workers(workers)
    n = g.n
    if n == 0:
        return 0
    _, higher = orientation_dense(g, und)

    def count_range(a, b):
        total = 0
        for i in range(a, b):
            hi = higher[i]
            for j in hi.tolist():
                total += np.intersect1d(hi, higher[j], assume_unique=True).shape[0]
        return total

    parts = run_partitioned(count_range, split_ranges(n, workers), workers)
    return int(sum(parts))


# ------------------------------------------------------------ fast C checker

def _fast_lib():
    import ctypes
    from pathlib import Path

    path = Path(__file__).resolve().parent / "_build" / "liboracle.so"
    if not path.exists():
        import sys

        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from paper_1503_07881_b200._build import build_oracle

        build_oracle()
    lib = ctypes.CDLL(str(path))
    i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
    i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
    f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
    lib.oracle_triangles.restype = ctypes.c_int64
    lib.oracle_triangles.argtypes = [ctypes.c_int64, i64p, i64p, i64p, i64p, ctypes.c_int]
    lib.oracle_triangles_slice32.restype = ctypes.c_int64
    lib.oracle_triangles_slice32.argtypes = [ctypes.c_int64, i64p, i32p, i64p, i32p,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
    lib.oracle_pagerank32.restype = None
    lib.oracle_pagerank32.argtypes = [ctypes.c_int64, i64p, i32p, i64p, ctypes.c_double,
                                      ctypes.c_int, f64p, ctypes.c_int]
    return lib


def triangle_count_fast(g: CSR, threads: int = 0) -> int:
    """Same algorithm as triangle_count_csr, in C (oracle/fast_oracle.c)."""
    if g.n == 0:
        return 0
    lib = _fast_lib()
    out_d = np.ascontiguousarray(np.searchsorted(g.ids, g.out_adj), dtype=np.int64)
    in_d = np.ascontiguousarray(np.searchsorted(g.ids, g.in_adj), dtype=np.int64)
    return int(lib.oracle_triangles(g.n, np.ascontiguousarray(g.out_off), out_d,
                                    np.ascontiguousarray(g.in_off), in_d, int(threads)))


def triangles_slice_dense32(n, out_off, out_adj, in_off, in_adj, part, nparts, threads=0):
    """Triangles whose middle vertex in (undirected degree, id) rank order has
    rank % nparts == part (algorithms.py:103-116 restated in C over the
    dense int32 CSR pair; the slice gt_triangles_part counts)."""
    lib = _fast_lib()
    return int(lib.oracle_triangles_slice32(
        int(n), np.ascontiguousarray(out_off, np.int64), np.ascontiguousarray(out_adj, np.int32),
        np.ascontiguousarray(in_off, np.int64), np.ascontiguousarray(in_adj, np.int32),
        int(part), int(nparts), int(threads)))


def pagerank_dense32(n, in_off, in_adj, out_off, damping, iterations, threads=0):
    """algorithms.py:45-85 in C over the dense int32 in-CSR (scores in dense
    index order)."""
    lib = _fast_lib()
    out = np.empty(int(n), dtype=np.float64)
    lib.oracle_pagerank32(int(n), np.ascontiguousarray(in_off, np.int64),
                          np.ascontiguousarray(in_adj, np.int32),
                          np.ascontiguousarray(out_off, np.int64), float(damping),
                          int(iterations), out, int(threads))
    return out


# ------------------------------------- algorithms.py:122-248 (§8f next #4)

def sssp_csr(g: CSR, source_index: int) -> np.ndarray:
    """algorithms.py:125-141 — BFS over out-edges from the node of dense index
    source_index; hop counts aligned with g.ids, -1 for unreachable (None)."""
    from collections import deque

    n = g.n
    out_d = np.searchsorted(g.ids, g.out_adj)
    dist = np.full(n, -1, dtype=np.int64)
    dist[source_index] = 0
    queue = deque([source_index])
    while queue:
        u = queue.popleft()
        d = dist[u] + 1
        for v in out_d[g.out_off[u]:g.out_off[u + 1]].tolist():
            if dist[v] < 0:
                dist[v] = d
                queue.append(v)
    return dist


def components_csr(g: CSR, und=None) -> np.ndarray:
    """algorithms.py:232-248 — BFS over undirected neighbours from every
    unlabelled node in ascending id order; labels dense in that order."""
    from collections import deque

    n = g.n
    if und is None:
        und = undirected_dense(g)
    labels = np.full(n, -1, dtype=np.int64)
    nxt = 0
    for start in range(n):
        if labels[start] >= 0:
            continue
        labels[start] = nxt
        queue = deque([start])
        while queue:
            u = queue.popleft()
            for v in und[u].tolist():
                if labels[v] < 0:
                    labels[v] = nxt
                    queue.append(v)
        nxt += 1
    return labels


def k_core_csr(g: CSR, k: int, und=None) -> CSR:
    """algorithms.py:206-229 — peel nodes with fewer than k distinct undirected
    neighbours (queue order), then graphs.py:169-183's induced subgraph on the
    survivors (every original edge between two survivors)."""
    from collections import deque

    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    n = g.n
    if und is None:
        und = undirected_dense(g)
    deg = np.asarray([u.shape[0] for u in und], dtype=np.int64)
    alive = np.ones(n, dtype=bool)
    queue = deque(i for i in range(n) if deg[i] < k)
    while queue:
        i = queue.popleft()
        if not alive[i]:
            continue
        alive[i] = False
        for m in und[i].tolist():
            if alive[m]:
                deg[m] -= 1
                if deg[m] == k - 1:
                    queue.append(m)
    out_d = np.searchsorted(g.ids, g.out_adj)
    src_d = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.out_off))
    keep = alive[src_d] & alive[out_d] if out_d.size else np.zeros(0, dtype=bool)
    return build_csr(g.ids[src_d[keep]], g.ids[out_d[keep]], workers=1)


def add_isolated(g: CSR, extra) -> CSR:
    """graphs.py:92-96 (Graph.add_node) on a CSR: the ids in `extra` not yet
    present become nodes without edges (empty rows at their sorted place)."""
    extra = np.setdiff1d(np.asarray(extra, dtype=np.int64), g.ids)
    if extra.size == 0:
        return g
    ids = np.union1d(g.ids, extra)
    pos = np.searchsorted(ids, g.ids)
    out_deg = np.zeros(ids.size, dtype=np.int64)
    in_deg = np.zeros(ids.size, dtype=np.int64)
    out_deg[pos] = np.diff(g.out_off)
    in_deg[pos] = np.diff(g.in_off)
    out_off = np.concatenate(([0], np.cumsum(out_deg))).astype(np.int64)
    in_off = np.concatenate(([0], np.cumsum(in_deg))).astype(np.int64)
    return CSR(ids, out_off, g.out_adj, in_off, g.in_adj)


# ------------------------------------------------------ tables.py: select / join

_CMP = {"=": np.equal, "!=": np.not_equal, "<": np.less, "<=": np.less_equal,
        ">": np.greater, ">=": np.greater_equal}


def select_indices(col, typ, pool, op, value):
    """tables.py:325-344 — ascending indices of the rows that satisfy the
    predicate. col: int64 (int / str codes) or float64 numpy column."""
    col = np.asarray(col)
    if typ == "str":
        if op in ("=", "!="):
            # encode_value (tables.py:201-205): pool code or None
            code = {s: i for i, s in enumerate(pool)}.get(value)
            if code is None:
                mask = np.full(col.shape[0], op == "!=", dtype=bool)
            else:
                mask = _CMP[op](col, code)
        else:  # ordering comparisons on the decoded strings (tables.py:339-341)
            import operator
            cmp = {"<": operator.lt, "<=": operator.le, ">": operator.gt,
                   ">=": operator.ge}[op]
            mask = np.array([cmp(pool[c], value) for c in col.tolist()], dtype=bool)
    else:
        mask = _CMP[op](col, value)
    return np.flatnonzero(mask).astype(np.int64)


def join_indices(lkeys, rkeys):
    """tables.py:397-426 — (left rows, right rows) of the equi-join: hash join
    building on the smaller side (left when len(left) <= len(right)), pairs in
    probe-row order and, per probe row, build rows in ascending order. Keys are
    python-comparable values (decoded strings, ints or floats), so dict
    semantics apply (-0.0 == 0.0, NaN never equal to another NaN object)."""
    lkeys = list(lkeys)
    rkeys = list(rkeys)
    build_left = len(lkeys) <= len(rkeys)
    bkeys, pkeys = (lkeys, rkeys) if build_left else (rkeys, lkeys)
    buckets = {}
    for i, k in enumerate(bkeys):
        buckets.setdefault(k, []).append(i)
    bi, pi = [], []
    for i, k in enumerate(pkeys):
        hit = buckets.get(k)
        if hit:
            bi.extend(hit)
            pi.extend([i] * len(hit))
    bi = np.asarray(bi, dtype=np.int64)
    pi = np.asarray(pi, dtype=np.int64)
    return (bi, pi) if build_left else (pi, bi)


# ------------------------------------------------------------ algorithms.scc

def scc_csr(g: CSR) -> np.ndarray:
    """algorithms.py:144-203 — iterative Tarjan over ascending ids, then dense
    relabelling by first occurrence over ascending ids. Returns labels aligned
    with g.ids."""
    n = g.ids.shape[0]
    out_off = g.out_off
    out_adj = np.searchsorted(g.ids, g.out_adj).astype(np.int64)  # dense dst per edge
    index = np.full(n, -1, dtype=np.int64)
    low = np.zeros(n, dtype=np.int64)
    on_stack = np.zeros(n, dtype=bool)
    comp = np.full(n, -1, dtype=np.int64)
    stack = []
    next_index = 0
    n_comps = 0
    for root in range(n):
        if index[root] >= 0:
            continue
        work = [(root, 0)]
        while work:
            v, child = work[-1]
            if child == 0:
                index[v] = low[v] = next_index
                next_index += 1
                stack.append(v)
                on_stack[v] = True
            a, b = int(out_off[v]), int(out_off[v + 1])
            advanced = False
            while child < b - a:
                w = int(out_adj[a + child])
                child += 1
                if index[w] < 0:
                    work[-1] = (v, child)
                    work.append((w, 0))
                    advanced = True
                    break
                if on_stack[w]:
                    low[v] = min(low[v], index[w])
            if advanced:
                continue
            work.pop()
            if work:
                parent = work[-1][0]
                low[parent] = min(low[parent], low[v])
            if low[v] == index[v]:
                while True:
                    w = stack.pop()
                    on_stack[w] = False
                    comp[w] = n_comps
                    if w == v:
                        break
                n_comps += 1
    remap = {}
    labels = np.empty(n, dtype=np.int64)
    for i in range(n):
        c = int(comp[i])
        if c not in remap:
            remap[c] = len(remap)
        labels[i] = remap[c]
    return labels


# ------------------------------------------- graphs.py:92-144 batched mutation

def update_csr(g: CSR, add=None, delete=None, add_nodes=(), del_nodes=()) -> CSR:
    """The reference's del_node* -> del_edge* -> add_node* -> add_edge* calls
    (graphs.py:92-144) on the graph `g`, restated on edge sets: nodes minus
    del_nodes, edges minus those incident to them and minus `delete`, then
    add_nodes and the endpoints + edges of `add` (duplicates collapse)."""
    src = np.repeat(g.ids, np.diff(g.out_off))
    dst = g.out_adj
    dead = set(int(x) for x in np.asarray(del_nodes, np.int64).tolist())
    gone = set(zip(*(np.asarray(a, np.int64).tolist() for a in delete))) if delete else set()
    edges = [(a, b) for a, b in zip(src.tolist(), dst.tolist())
             if a not in dead and b not in dead and (a, b) not in gone]
    nodes = [x for x in g.ids.tolist() if x not in dead]
    nodes += [int(x) for x in np.asarray(add_nodes, np.int64).tolist()]
    if add:
        edges += list(zip(*(np.asarray(a, np.int64).tolist() for a in add)))
    s = np.asarray([a for a, _ in edges], np.int64)
    d = np.asarray([b for _, b in edges], np.int64)
    out = build_csr(s, d, workers=1)
    return add_isolated(out, np.asarray(nodes, np.int64)) if nodes else out
