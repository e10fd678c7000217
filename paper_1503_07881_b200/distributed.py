"""Multi-GPU hot path: one process per GPU over ``torch.distributed``.

The reference runs on one big-memory host with a thread pool
(``parallel.py:39-93``); this module shards the same three steps across the
GPUs of one box, NCCL over NVLink for the exchanges:

* **ToGraph** — every rank holds a slice of the edge table. Node set: global
  id range (all-reduce MIN/MAX) and presence flags (all-reduce MAX), so every
  rank derives the same dense ranks (convert.py:45-59). Out-CSR: local sort +
  dedupe, then a *sample sort by src range* — splitters from an all-reduced
  histogram of src-rank buckets (the GPU form of ``parallel_sort``'s
  splitters, parallel.py:52-93) — and one all-to-all shuffle; each rank sorts
  and dedupes what it received and owns the out-rows of its src range. In-CSR:
  the owned edges, swapped to (dst, src), take a second shuffle by dst range.
* **PageRank** — 1D dst-range partition of the in-CSR; the contribution
  vector is replicated: every iteration all-gathers the owned slices and
  all-reduces the dangling mass (algorithms.py:72-85).
* **Triangles** — the degree-ordered orientation is built sharded (each rank
  symmetrises, ranks and orients its own rows; the oriented arcs are
  all-gathered once), every rank counts the triangles of an interleaved share
  of the middle vertices, and the counts are all-reduced (algorithms.py:98-118).

All O(rows) / O(edges) work runs in libgtb200 kernels (``NativeOps``); this
module only moves buffers and makes the O(ranks) decisions. ``ops`` is a
parameter so that the CPU tests can drive the same collective logic with
``gloo`` and a CPU restatement of the primitives (tests/dist_cpu_ops.py);
the product path always uses ``NativeOps`` and has no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from .errors import CapacityError

SPLIT_BITS = 12  # splitter histogram: 4096 buckets of src (dst) ranks
MAX_SPAN = 1 << 33  # presence flags of the id range (1 byte per id)


def _bits_for(n: int) -> int:
    b = 1
    while b < 63 and (1 << b) < n:
        b += 1
    return b


# --------------------------------------------------------------------- ops --

class NativeOps:
    """Per-rank primitives in libgtb200.so on this process's GPU."""

    def __init__(self, device=None):
        from . import _native

        self._n = _native
        self.lib = _native.ensure_init()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)

    # every call below synchronises the library stream before returning; the
    # torch stream is synchronised first so collectives have landed
    def _pre(self):
        torch.cuda.current_stream(self.device).synchronize()

    def _ck(self, rc, what):
        self._n.check(rc, what)

    def empty(self, n, dtype):
        return torch.empty(int(n), dtype=dtype, device=self.device)

    def id_minmax(self, src, dst):
        self._pre()
        out = self.empty(2, torch.int64)
        self._ck(self.lib.gt_id_minmax(src.data_ptr(), dst.data_ptr(), src.numel(),
                                       out.data_ptr()), "gt_id_minmax")
        return out

    def id_presence(self, src, dst, lo, span):
        self._pre()
        flags = self.empty(span, torch.uint8)
        self._ck(self.lib.gt_id_presence(src.data_ptr(), dst.data_ptr(), src.numel(), lo, span,
                                         flags.data_ptr()), "gt_id_presence")
        return flags

    def id_rankmap(self, flags):
        import ctypes

        self._pre()
        span = flags.numel()
        words = self.empty(2 * ((span + 31) // 32), torch.int32)
        n = ctypes.c_int64()
        self._ck(self.lib.gt_id_rankmap(flags.data_ptr(), span, words.data_ptr(),
                                        ctypes.byref(n)), "gt_id_rankmap")
        return words, int(n.value)

    def id_list(self, words, span, lo, n):
        self._pre()
        ids = self.empty(n, torch.int64)
        self._ck(self.lib.gt_id_list(words.data_ptr(), span, lo, ids.data_ptr()), "gt_id_list")
        return ids

    def pack_keys(self, src, dst, lo, words, kbits):
        self._pre()
        keys = self.empty(src.numel(), torch.int64)
        self._ck(self.lib.gt_pack_keys(src.data_ptr(), dst.data_ptr(), src.numel(), lo,
                                       words.data_ptr(), kbits, keys.data_ptr()), "gt_pack_keys")
        return keys

    def sort_keys(self, keys, lo_bit, hi_bit):
        import ctypes

        keys = keys.contiguous().clone()  # torch-stream copy: ordered before the sort by _pre
        tmp = torch.empty_like(keys)
        self._pre()
        which = ctypes.c_int()
        self._ck(self.lib.gt_sort_keys(keys.data_ptr(), tmp.data_ptr(), keys.numel(), lo_bit,
                                       hi_bit, ctypes.byref(which)), "gt_sort_keys")
        return tmp if which.value else keys

    def merge_runs(self, keys, run_sizes):
        """Merge consecutive sorted runs of the given sizes (gt_merge_runs)."""
        import ctypes

        keys = keys.contiguous().clone()  # torch-stream copy: ordered before the merge by _pre
        tmp = torch.empty_like(keys)
        off = np.concatenate([[0], np.cumsum(np.asarray(run_sizes, dtype=np.int64))])
        off = np.ascontiguousarray(off, dtype=np.int64)
        self._pre()
        which = ctypes.c_int()
        self._ck(self.lib.gt_merge_runs(keys.data_ptr(), tmp.data_ptr(), keys.numel(),
                                        off.ctypes.data, len(run_sizes), ctypes.byref(which)),
                 "gt_merge_runs")
        return tmp if which.value else keys

    def unique_keys(self, keys):
        import ctypes

        self._pre()
        out = torch.empty_like(keys)
        m = ctypes.c_int64()
        self._ck(self.lib.gt_unique_keys(keys.data_ptr(), keys.numel(), out.data_ptr(),
                                         ctypes.byref(m)), "gt_unique_keys")
        return out[: m.value]

    def bucket_counts(self, keys, shift, nbuckets):
        self._pre()
        counts = self.empty(nbuckets, torch.int64)
        self._ck(self.lib.gt_key_bucket_counts(keys.data_ptr(), keys.numel(), shift, nbuckets,
                                               counts.data_ptr()), "gt_key_bucket_counts")
        return counts

    def lower_bounds(self, sorted_keys, bounds):
        self._pre()
        b = np.ascontiguousarray(np.asarray(bounds, dtype=np.uint64))
        out = np.empty(b.shape[0], dtype=np.int64)
        self._ck(self.lib.gt_key_lower_bounds(sorted_keys.data_ptr(), sorted_keys.numel(),
                                              b.ctypes.data, b.shape[0], out.ctypes.data),
                 "gt_key_lower_bounds")
        return out

    def swap_halves(self, keys, kbits):
        self._pre()
        out = torch.empty_like(keys)
        self._ck(self.lib.gt_swap_key_halves(keys.data_ptr(), keys.numel(), kbits,
                                             out.data_ptr()), "gt_swap_key_halves")
        return out

    def csr_from_keys(self, keys, kbits, row_lo, rows):
        self._pre()
        off = self.empty(rows + 1, torch.int64)
        adj = self.empty(max(keys.numel(), 1), torch.int32)
        tmp = torch.empty_like(keys) if row_lo and keys.numel() else keys
        self._ck(self.lib.gt_csr_from_keys(keys.data_ptr(), keys.numel(), kbits, row_lo, rows,
                                           tmp.data_ptr(), off.data_ptr(), adj.data_ptr()),
                 "gt_csr_from_keys")
        return off, adj[: keys.numel()]

    def graph_from_csr(self, n, e, ids, out_off, out_adj, in_off, in_adj):
        import ctypes

        from .graph import DeviceGraph

        self._pre()
        h = ctypes.c_void_p()
        self._ck(self.lib.gt_graph_from_csr(n, e, ids.data_ptr(), out_off.data_ptr(),
                                            out_adj.data_ptr(), in_off.data_ptr(),
                                            in_adj.data_ptr(), ctypes.byref(h)),
                 "gt_graph_from_csr")
        return DeviceGraph(h.value)

    def inv_degree(self, off):
        self._pre()
        rows = off.numel() - 1
        inv = self.empty(max(rows, 1), torch.float64)
        self._ck(self.lib.gt_inv_degree(off.data_ptr(), rows, inv.data_ptr()), "gt_inv_degree")
        return inv[:rows]

    def remap_padded(self, in_adj, bounds, m):
        self._pre()
        b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
        out = torch.empty_like(in_adj)
        self._ck(self.lib.gt_remap_padded(in_adj.data_ptr(), in_adj.numel(), b.ctypes.data,
                                          len(bounds) - 1, int(m), out.data_ptr()),
                 "gt_remap_padded")
        return out

    def pagerank_init(self, inv_full):
        self._pre()
        n = inv_full.numel()
        contrib = self.empty(n, torch.float64)
        dangling = self.empty(1, torch.float64)
        self._ck(self.lib.gt_pagerank_init(inv_full.data_ptr(), n, contrib.data_ptr(),
                                           dangling.data_ptr()), "gt_pagerank_init")
        return contrib, dangling

    def pagerank_step(self, in_off, in_adj, n_total, contrib, inv_rows, dangling, damping, last):
        self._pre()
        rows = in_off.numel() - 1
        score = self.empty(max(rows, 1), torch.float64)
        nxt = self.empty(max(rows, 1), torch.float64)
        part = self.empty(1, torch.float64)
        self._ck(self.lib.gt_pagerank_step(in_off.data_ptr(), in_adj.data_ptr(), rows,
                                           in_adj.numel(), n_total, contrib.data_ptr(),
                                           inv_rows.data_ptr(), dangling.data_ptr(), damping,
                                           int(last), score.data_ptr(), nxt.data_ptr(),
                                           part.data_ptr()), "gt_pagerank_step")
        return (score[:rows] if last else nxt[:rows]), part

    def undirected_keys(self, off, adj, kbits, row_lo):
        import ctypes

        self._pre()
        rows = off.numel() - 1
        keys = self.empty(2 * adj.numel(), torch.int64)
        n = ctypes.c_int64()
        self._ck(self.lib.gt_tc_undirected_keys(off.data_ptr(), adj.data_ptr(), rows, row_lo, kbits,
                                                keys.data_ptr(), ctypes.byref(n)),
                 "gt_tc_undirected_keys")
        return keys[:n.value]

    def degree_rank(self, deg):
        self._pre()
        rank = self.empty(deg.numel(), torch.int32)
        self._ck(self.lib.gt_tc_degree_rank(deg.data_ptr(), deg.numel(), rank.data_ptr()),
                 "gt_tc_degree_rank")
        return rank

    def orient_keys(self, off, adj, row_lo, rank, kbits):
        import ctypes

        self._pre()
        rows = off.numel() - 1
        keys = self.empty(adj.numel(), torch.int64)
        m = ctypes.c_int64()
        self._ck(self.lib.gt_tc_orient_keys(off.data_ptr(), adj.data_ptr(), rows, row_lo,
                                            rank.data_ptr(), kbits, keys.data_ptr(),
                                            ctypes.byref(m)), "gt_tc_orient_keys")
        return keys[:m.value]

    def triangles_oriented_part(self, off_p, adj_p, part, nparts):
        import ctypes

        self._pre()
        c = ctypes.c_int64()
        self._ck(self.lib.gt_triangles_oriented_part(off_p.data_ptr(), adj_p.data_ptr(),
                                                     off_p.numel() - 1, adj_p.numel(), part,
                                                     nparts, ctypes.byref(c)),
                 "gt_triangles_oriented_part")
        return int(c.value)

    def triangles_part(self, graph, part, nparts):
        import ctypes

        self._pre()
        c = ctypes.c_int64()
        self._ck(self.lib.gt_triangles_part(graph.handle, part, nparts, ctypes.byref(c)),
                 "gt_triangles_part")
        return int(c.value)


# ----------------------------------------------------------------- helpers --

def _world(group):
    return dist.get_world_size(group), dist.get_rank(group)


def _exchange(send: torch.Tensor, splits: np.ndarray, group):
    """all-to-all with uneven splits: part r of `send` goes to rank r.
    Returns the received keys (source-rank order) and the per-source sizes."""
    world, _ = _world(group)
    send_counts = torch.tensor(np.diff(splits), dtype=torch.int64, device=send.device)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc = [int(x) for x in recv_counts.tolist()]
    sc = [int(x) for x in send_counts.tolist()]
    out = torch.empty(sum(rc), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(out, send.contiguous(), output_split_sizes=rc, input_split_sizes=sc,
                           group=group)
    return out, rc


def _range_bounds(counts: np.ndarray, world: int, rows: int, bucket_rows: int) -> list[int]:
    """Row boundaries of `world` ranges balancing the bucketed counts."""
    cum = np.cumsum(counts)
    total = int(cum[-1]) if cum.size else 0
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left")) + 1  # buckets [0, b) go left
        bounds.append(min(max(b * bucket_rows, bounds[-1]), rows))
    bounds.append(rows)
    return bounds


def _shuffle_by_rows(keys_sorted, kbits, bounds, ops, group):
    """Send each key to the rank owning its row (key >> kbits)."""
    key_bounds = [int(b) << kbits for b in bounds]
    idx = ops.lower_bounds(keys_sorted, key_bounds)
    idx[0], idx[-1] = 0, keys_sorted.numel()
    return _exchange(keys_sorted, idx, group)


def _split_plan(n: int, kbits: int):
    sb = min(SPLIT_BITS, kbits)
    return sb, 1 << (kbits - sb)  # bucket bits, rows per bucket


# ------------------------------------------------------------------- build --

@dataclass
class ShardedGraph:
    """This rank's part of the graph; the ranges are identical on every rank."""

    n: int
    e: int
    kbits: int
    ids: torch.Tensor                      # int64 [n], replicated
    out_bounds: list[int]                  # src-row ranges of the ranks
    in_bounds: list[int]                   # dst-row ranges of the ranks
    out_off: torch.Tensor                  # int64 [rows+1], local offsets
    out_adj: torch.Tensor                  # int32 dense dst
    in_off: torch.Tensor
    in_adj: torch.Tensor                   # int32 dense src
    out_counts: list[int] = field(default_factory=list)
    in_counts: list[int] = field(default_factory=list)


def build_csr(src: torch.Tensor, dst: torch.Tensor, group=None, ops=None) -> ShardedGraph:
    """Distributed ToGraph over the row slices (src, dst) of all ranks."""
    ops = ops or NativeOps()
    world, rank = _world(group)
    dev = src.device
    mm = ops.id_minmax(src, dst)
    lo_t, hi_t = mm[0:1].clone(), mm[1:2].clone()
    dist.all_reduce(lo_t, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi_t, op=dist.ReduceOp.MAX, group=group)
    lo, hi = int(lo_t.item()), int(hi_t.item())
    empty64 = torch.zeros(1, dtype=torch.int64, device=dev)
    if lo > hi:  # no rows anywhere: empty graph (convert.py:142-143)
        z32 = torch.zeros(0, dtype=torch.int32, device=dev)
        return ShardedGraph(0, 0, 1, torch.zeros(0, dtype=torch.int64, device=dev),
                            [0] * (world + 1), [0] * (world + 1), empty64, z32, empty64.clone(),
                            z32, [0] * world, [0] * world)
    span = hi - lo + 1
    if span > MAX_SPAN:
        raise CapacityError(f"distributed build needs an id range <= 2^33, got {span}")
    flags = ops.id_presence(src, dst, lo, span)
    dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    words, n = ops.id_rankmap(flags)
    del flags
    if n >= (1 << 31):
        raise CapacityError("graph has >= 2^31 distinct node ids")
    ids = ops.id_list(words, span, lo, n)
    kbits = _bits_for(n)
    sb, bucket_rows = _split_plan(n, kbits)

    # out-CSR: local sort + dedupe, sample sort by src range, merge + dedupe
    keys = ops.pack_keys(src, dst, lo, words, kbits)
    del words
    keys = ops.unique_keys(ops.sort_keys(keys, 0, 2 * kbits))
    counts = ops.bucket_counts(keys, 2 * kbits - sb, 1 << sb)
    dist.all_reduce(counts, group=group)
    out_bounds = _range_bounds(counts.cpu().numpy(), world, n, bucket_rows)
    # the received runs (one per source rank) are each sorted: merge them
    mine, sizes = _shuffle_by_rows(keys, kbits, out_bounds, ops, group)
    mine = ops.unique_keys(ops.merge_runs(mine, sizes))
    o_lo, o_hi = out_bounds[rank], out_bounds[rank + 1]
    out_off, out_adj = ops.csr_from_keys(mine, kbits, o_lo, o_hi - o_lo)

    # in-CSR: the owned edges as (dst, src), shuffled by dst range. `mine` is
    # sorted by (src, dst), so after the swap a stable sort over the dst bits
    # alone leaves src ascending inside every dst (the single-GPU in-sort)
    ikeys = ops.sort_keys(ops.swap_halves(mine, kbits), kbits, 2 * kbits)
    del mine
    counts = ops.bucket_counts(ikeys, 2 * kbits - sb, 1 << sb)
    dist.all_reduce(counts, group=group)
    in_bounds = _range_bounds(counts.cpu().numpy(), world, n, bucket_rows)
    theirs, sizes = _shuffle_by_rows(ikeys, kbits, in_bounds, ops, group)
    del ikeys
    # the received runs arrive in source-rank order, each sorted by the whole
    # (dst, src) key: merging them gives (dst, src) order
    theirs = ops.merge_runs(theirs, sizes)
    i_lo, i_hi = in_bounds[rank], in_bounds[rank + 1]
    in_off, in_adj = ops.csr_from_keys(theirs, kbits, i_lo, i_hi - i_lo)

    ec = torch.tensor([out_adj.numel(), in_adj.numel()], dtype=torch.int64, device=dev)
    all_ec = [torch.empty_like(ec) for _ in range(world)]
    dist.all_gather(all_ec, ec, group=group)
    out_counts = [int(x[0].item()) for x in all_ec]
    in_counts = [int(x[1].item()) for x in all_ec]
    return ShardedGraph(n, sum(out_counts), kbits, ids, out_bounds, in_bounds, out_off, out_adj,
                        in_off, in_adj, out_counts, in_counts)


def gather_csr(sg: ShardedGraph, group=None):
    """Replicate the full CSR pair on every rank (offsets rebased)."""
    world, _ = _world(group)

    def full(off, adj, counts, bounds):
        rows = [bounds[r + 1] - bounds[r] for r in range(world)]
        offs = _gather_known(off[:-1], rows, group)  # sizes known everywhere
        adjs = _gather_known(adj, list(counts), group)
        base = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        row_base = torch.from_numpy(np.repeat(base[:-1], rows)).to(off.device)
        tail = torch.tensor([int(base[-1])], dtype=torch.int64, device=off.device)
        return torch.cat([offs + row_base, tail]), adjs

    out_off, out_adj = full(sg.out_off, sg.out_adj, sg.out_counts, sg.out_bounds)
    in_off, in_adj = full(sg.in_off, sg.in_adj, sg.in_counts, sg.in_bounds)
    return out_off, out_adj, in_off, in_adj


# ---------------------------------------------------------------- PageRank --

def _gather_known(t: torch.Tensor, sizes: list[int], group) -> torch.Tensor:
    """All-gather of 1-D slices whose sizes every rank already knows (no size
    exchange, no host syncs): one all_gather_into_tensor of m-sized chunks."""
    world, rank = _world(group)
    m = max(max(sizes), 1)
    buf = torch.empty(world * m, dtype=t.dtype, device=t.device)
    buf[rank * m: rank * m + t.numel()] = t
    dist.all_gather_into_tensor(buf, buf[rank * m:(rank + 1) * m], group=group)
    return torch.cat([buf[r * m: r * m + sizes[r]] for r in range(world)])


def pagerank(sg: ShardedGraph, damping: float = 0.85, iterations: int = 10, group=None,
             ops=None) -> torch.Tensor:
    """Scores of all nodes (id order) on every rank (algorithms.py:36-87).

    1D dst-range partition: rank r computes the rows
    [in_bounds[r], in_bounds[r+1]); the contribution vector lives in a padded
    buffer of one m-sized chunk per rank, filled every iteration by ONE
    in-place all_gather_into_tensor (the slice sizes follow from the
    replicated bounds: no size exchange, no host round trip); the local
    in-adjacency is remapped once to padded positions. The dangling mass is
    one all-reduced double per iteration."""
    if not 0.0 < damping < 1.0:
        raise ValueError(f"damping must be in (0, 1), got {damping}")
    if iterations < 1:
        raise ValueError(f"iterations must be >= 1, got {iterations}")
    if sg.n == 0:
        raise ValueError("pagerank needs a non-empty graph")
    ops = ops or NativeOps()
    world, rank = _world(group)
    out_sizes = [sg.out_bounds[r + 1] - sg.out_bounds[r] for r in range(world)]
    sizes = [sg.in_bounds[r + 1] - sg.in_bounds[r] for r in range(world)]
    m = max(max(sizes), 1)
    inv_full = _gather_known(ops.inv_degree(sg.out_off), out_sizes, group)
    contrib0, dangling = ops.pagerank_init(inv_full)
    i_lo, i_hi = sg.in_bounds[rank], sg.in_bounds[rank + 1]
    inv_rows = inv_full[i_lo:i_hi].contiguous()
    adj_p = ops.remap_padded(sg.in_adj, sg.in_bounds, m)
    bufs = [torch.zeros(world * m, dtype=torch.float64, device=contrib0.device) for _ in range(2)]
    for r in range(world):  # initial contributions in the padded layout
        a, b = sg.in_bounds[r], sg.in_bounds[r + 1]
        bufs[0][r * m: r * m + (b - a)] = contrib0[a:b]
    del contrib0
    for it in range(iterations):
        last = it == iterations - 1
        cur, nxt = bufs[it & 1], bufs[(it + 1) & 1]
        vals, part = ops.pagerank_step(sg.in_off, adj_p, sg.n, cur, inv_rows, dangling,
                                       damping, last)
        nxt[rank * m: rank * m + vals.numel()] = vals
        dist.all_gather_into_tensor(nxt, nxt[rank * m:(rank + 1) * m], group=group)
        if last:
            return torch.cat([nxt[r * m: r * m + sizes[r]] for r in range(world)])
        dist.all_reduce(part, group=group)
        dangling = part
    raise AssertionError("unreachable")


# --------------------------------------------------------------- triangles --

def orient(sg: ShardedGraph, group=None, ops=None):
    """Degree-ordered orientation, sharded (algorithms.py:98-108): returns the
    rank-space oriented CSR (off_p int64[n+1], adj_p int32[m]) replicated on
    every rank. Each rank works on its own rows only:

    1. both directions of its out-edges as undirected keys, sorted, deduped,
       shuffled by first endpoint (the splitters as in build_csr) and merged:
       rank r owns the undirected rows N(i) of an id range (graphs.py:163-167);
    2. degrees all-gathered (n values), the (degree, id) rank computed on every
       rank (one sort of n keys);
    3. each rank orients its rows (arcs to higher-ranked neighbours), sorts
       them, and ONE all-gather of the arcs plus a merge of the sorted runs
       gives every rank the whole orientation — no replicated CSR pair and no
       replicated orientation work."""
    ops = ops or NativeOps()
    world, rank = _world(group)
    k = sg.kbits
    sb, bucket_rows = _split_plan(sg.n, k)
    und = ops.unique_keys(ops.sort_keys(ops.undirected_keys(sg.out_off, sg.out_adj, k,
                                                             sg.out_bounds[rank]), 0, 2 * k))
    counts = ops.bucket_counts(und, 2 * k - sb, 1 << sb)
    dist.all_reduce(counts, group=group)
    bounds = _range_bounds(counts.cpu().numpy(), world, sg.n, bucket_rows)
    mine, sizes = _shuffle_by_rows(und, k, bounds, ops, group)
    del und
    mine = ops.unique_keys(ops.merge_runs(mine, sizes))
    lo, hi = bounds[rank], bounds[rank + 1]
    und_off, und_adj = ops.csr_from_keys(mine, k, lo, hi - lo)
    del mine
    rows = [bounds[r + 1] - bounds[r] for r in range(world)]
    deg = _gather_known(und_off[1:] - und_off[:-1], rows, group)
    rank_of = ops.degree_rank(deg)
    arcs = ops.sort_keys(ops.orient_keys(und_off, und_adj, lo, rank_of, k), 0, 2 * k)
    del und_off, und_adj
    sizes_t = torch.tensor([arcs.numel()], dtype=torch.int64, device=arcs.device)
    all_sizes = [torch.empty_like(sizes_t) for _ in range(world)]
    dist.all_gather(all_sizes, sizes_t, group=group)
    msizes = [int(x.item()) for x in all_sizes]
    arcs = ops.merge_runs(_gather_known(arcs, msizes, group), msizes)
    return ops.csr_from_keys(arcs, k, 0, sg.n)


def triangle_count(sg: ShardedGraph, group=None, ops=None) -> int:
    """Exact triangle count (algorithms.py:90-119): the sharded orientation
    (`orient`), every rank counts the triangles whose middle vertex v is
    rank (mod world) over the replicated N+ rows, one all-reduce."""
    if sg.n == 0 or sg.e == 0:
        return 0
    ops = ops or NativeOps()
    world, rank = _world(group)
    off_p, adj_p = orient(sg, group, ops)
    c = torch.tensor([ops.triangles_oriented_part(off_p, adj_p, rank, world)],
                     dtype=torch.int64, device=sg.ids.device)
    dist.all_reduce(c, group=group)
    return int(c.item())
