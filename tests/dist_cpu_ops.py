"""CPU restatement of the per-rank primitives of distributed.NativeOps.

TEST INFRASTRUCTURE ONLY: lets the multi-GPU orchestration in
paper_1503_07881_b200/distributed.py (collectives, splitters, shuffles,
offset rebasing) run on CPU tensors with the gloo backend, world size 2.
Each method has the semantics of the C-ABI call it stands for
(include/gtb200.h, "multi-GPU primitives"); keys are int64 tensors holding
uint64 bit patterns, as on the device.
"""

from __future__ import annotations

import numpy as np
import torch

_I64_MAX = np.iinfo(np.int64).max
_I64_MIN = np.iinfo(np.int64).min


def _u64(t: torch.Tensor) -> np.ndarray:
    return t.numpy().view(np.uint64)


def _t64(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy())


class CpuOps:
    device = torch.device("cpu")

    def id_minmax(self, src, dst):
        a = np.concatenate([src.numpy(), dst.numpy()])
        if a.size == 0:
            return torch.tensor([_I64_MAX, _I64_MIN], dtype=torch.int64)
        return torch.tensor([int(a.min()), int(a.max())], dtype=torch.int64)

    def id_presence(self, src, dst, lo, span):
        flags = np.zeros(span, dtype=np.uint8)
        flags[src.numpy() - lo] = 1
        flags[dst.numpy() - lo] = 1
        return torch.from_numpy(flags)

    def id_rankmap(self, flags):
        f = flags.numpy().astype(np.int64)
        prefix = np.concatenate([[0], np.cumsum(f)])
        return (torch.from_numpy(f), torch.from_numpy(prefix)), int(prefix[-1])

    def id_list(self, words, span, lo, n):
        f, _ = words
        return torch.from_numpy(np.nonzero(f.numpy())[0].astype(np.int64) + lo)

    def pack_keys(self, src, dst, lo, words, kbits):
        _, prefix = words
        p = prefix.numpy()
        rs = p[src.numpy() - lo].astype(np.uint64)
        rd = p[dst.numpy() - lo].astype(np.uint64)
        return _t64((rs << np.uint64(kbits)) | rd)

    def sort_keys(self, keys, lo_bit, hi_bit):
        k = _u64(keys)
        digit = (k >> np.uint64(lo_bit)) & np.uint64((1 << (hi_bit - lo_bit)) - 1)
        return _t64(k[np.argsort(digit, kind="stable")])

    def merge_runs(self, keys, run_sizes):
        k = _u64(keys)
        off = np.concatenate([[0], np.cumsum(np.asarray(run_sizes, dtype=np.int64))])
        assert off[-1] == k.size
        for r in range(len(run_sizes)):  # precondition of gt_merge_runs
            seg = k[off[r]:off[r + 1]]
            assert np.all(seg[1:] >= seg[:-1]), "merge_runs: run not sorted"
        return _t64(np.sort(k, kind="stable"))

    def unique_keys(self, keys):
        k = _u64(keys)
        if k.size == 0:
            return keys.clone()
        keep = np.ones(k.size, dtype=bool)
        keep[1:] = k[1:] != k[:-1]
        return _t64(k[keep])

    def bucket_counts(self, keys, shift, nbuckets):
        b = np.minimum(_u64(keys) >> np.uint64(shift), np.uint64(nbuckets - 1)).astype(np.int64)
        return torch.from_numpy(np.bincount(b, minlength=nbuckets).astype(np.int64))

    def lower_bounds(self, sorted_keys, bounds):
        return np.searchsorted(_u64(sorted_keys), np.asarray(bounds, dtype=np.uint64),
                               side="left").astype(np.int64)

    def swap_halves(self, keys, kbits):
        k = _u64(keys)
        low = np.uint64((1 << kbits) - 1)
        return _t64(((k & low) << np.uint64(kbits)) | (k >> np.uint64(kbits)))

    def csr_from_keys(self, keys, kbits, row_lo, rows):
        k = _u64(keys)
        r = (k >> np.uint64(kbits)).astype(np.int64) - row_lo
        off = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=rows))]).astype(np.int64)
        adj = (k & np.uint64((1 << kbits) - 1)).astype(np.int32)
        return torch.from_numpy(off), torch.from_numpy(adj)

    def graph_from_csr(self, n, e, ids, out_off, out_adj, in_off, in_adj):
        return {"n": n, "e": e, "out_off": out_off.numpy(), "out_adj": out_adj.numpy(),
                "in_off": in_off.numpy(), "in_adj": in_adj.numpy()}

    def inv_degree(self, off):
        d = np.diff(off.numpy())
        inv = np.zeros(d.size, dtype=np.float64)
        inv[d > 0] = 1.0 / d[d > 0]
        return torch.from_numpy(inv)

    def remap_padded(self, in_adj, bounds, m):
        v = in_adj.numpy().astype(np.int64)
        b = np.asarray(bounds, dtype=np.int64)
        r = np.searchsorted(b[1:-1], v, side="right")
        return torch.from_numpy((r * m + (v - b[r])).astype(np.int32))

    def pagerank_init(self, inv_full):
        inv = inv_full.numpy()
        n = inv.size
        contrib = inv * (1.0 / n)
        dangling = np.array([np.count_nonzero(inv == 0.0) * (1.0 / n)])
        return torch.from_numpy(contrib), torch.from_numpy(dangling)

    def pagerank_step(self, in_off, in_adj, n_total, contrib, inv_rows, dangling, damping, last):
        off = in_off.numpy()
        rows = off.size - 1
        row_of = np.repeat(np.arange(rows), np.diff(off))
        sums = np.bincount(row_of, weights=contrib.numpy()[in_adj.numpy()], minlength=rows)
        base = (1.0 - damping) / n_total + damping * (float(dangling.numpy()[0]) / n_total)
        sc = base + damping * sums
        inv = inv_rows.numpy()
        part = torch.tensor([float(sc[inv == 0.0].sum())], dtype=torch.float64)
        return torch.from_numpy(sc if last else sc * inv), part

    def undirected_keys(self, off, adj, kbits, row_lo):
        o, a = off.numpy(), adj.numpy().astype(np.uint64)
        u = (np.repeat(np.arange(o.size - 1), np.diff(o)) + row_lo).astype(np.uint64)
        keep = a != u
        u, a = u[keep], a[keep]
        k = np.uint64(kbits)
        return _t64(np.concatenate([(u << k) | a, (a << k) | u]))

    def degree_rank(self, deg):
        d = deg.numpy()
        order = np.lexsort((np.arange(d.size), d))
        rank = np.empty(d.size, dtype=np.int32)
        rank[order] = np.arange(d.size, dtype=np.int32)
        return torch.from_numpy(rank)

    def orient_keys(self, off, adj, row_lo, rank, kbits):
        o, a, r = off.numpy(), adj.numpy(), rank.numpy()
        u = np.repeat(np.arange(o.size - 1), np.diff(o)) + row_lo
        ru, rv = r[u].astype(np.uint64), r[a].astype(np.uint64)
        keep = rv > ru
        return _t64((ru[keep] << np.uint64(kbits)) | rv[keep])

    def triangles_oriented_part(self, off_p, adj_p, part, nparts):
        """sum over middle vertices v = part mod nparts of |N+(u) & N+(v)|, u in N-(v)."""
        o, a = off_p.numpy(), adj_p.numpy()
        n = o.size - 1
        plus = [set(a[o[i]:o[i + 1]].tolist()) for i in range(n)]
        total = 0
        for u in range(n):
            for v in a[o[u]:o[u + 1]].tolist():
                if v % nparts == part:
                    total += len(plus[u] & plus[v])
        return total

    def triangles_part(self, graph, part, nparts):
        """v-centred count (u < v < w in (degree, id) rank) over v = part mod nparts."""
        n = graph["n"]
        oo, oa, io, ia = graph["out_off"], graph["out_adj"], graph["in_off"], graph["in_adj"]
        und = []
        for i in range(n):
            s = set(oa[oo[i]:oo[i + 1]].tolist()) | set(ia[io[i]:io[i + 1]].tolist())
            s.discard(i)
            und.append(s)
        deg = [len(s) for s in und]
        higher = [{j for j in und[i] if (deg[j], j) > (deg[i], i)} for i in range(n)]
        lower = [[j for j in und[i] if (deg[j], j) < (deg[i], i)] for i in range(n)]
        return sum(len(higher[u] & higher[v]) for v in range(part, n, nparts) for u in lower[v])
