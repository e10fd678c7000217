"""Multi-GPU primitives on the B200 (NativeOps) — parity with their CPU
restatement, the pipeline over NCCL at world size 1, and the multi-rank
PageRank / triangle splits emulated rank by rank on the one GPU (no kernel
ever waits on another rank's kernel)."""

import os
import socket

import numpy as np
import pytest
import torch

from dist_cpu_ops import CpuOps
from oracle import reference_port as ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_1503_07881_b200.distributed import NativeOps

    return NativeOps("cuda:0")


def _keys(rng, n, bits):
    return torch.from_numpy(rng.integers(0, 1 << bits, size=n, dtype=np.int64))


@pytest.mark.parametrize("n,bits,lo,hi", [(1, 20, 0, 20), (5000, 44, 0, 44), (70000, 40, 0, 40),
                                          (30000, 54, 32, 54), (4099, 16, 3, 11)])
def test_sort_unique_bounds_match_cpu(native, n, bits, lo, hi):
    rng = np.random.default_rng(n + bits)
    k = _keys(rng, n, bits)
    cpu = CpuOps()
    got = native.sort_keys(k.cuda(), lo, hi).cpu()
    want = cpu.sort_keys(k, lo, hi)
    assert torch.equal(got, want)  # stable: identical permutation
    if lo == 0 and hi == bits:
        assert torch.equal(native.unique_keys(got.cuda()).cpu(), cpu.unique_keys(want))
        b = np.sort(rng.integers(0, 1 << bits, size=9).astype(np.uint64))
        assert np.array_equal(native.lower_bounds(got.cuda(), b), cpu.lower_bounds(want, b))
        sh = max(0, bits - 12)
        assert torch.equal(native.bucket_counts(got.cuda(), sh, 1 << min(12, bits)).cpu(),
                           cpu.bucket_counts(want, sh, 1 << min(12, bits)))


def _runs_by_dst_then_src(rng, nruns, kbits, per_run):
    """Runs as the in-CSR shuffle delivers them: run r holds edges whose src
    lie in [r*w, (r+1)*w) (rank r's out-CSR rows), each run sorted by
    (dst, src), keys (dst << kbits) | src."""
    w = (1 << kbits) // nruns
    runs, sizes = [], []
    for r in range(nruns):
        m = int(per_run[r])
        src = rng.integers(r * w, (r + 1) * w, size=m).astype(np.uint64)
        dst = rng.integers(0, 1 << kbits, size=m).astype(np.uint64)
        k = np.unique((dst << np.uint64(kbits)) | src)
        runs.append(k)
        sizes.append(k.size)
    return torch.from_numpy(np.concatenate(runs).view(np.int64).copy()), sizes


@pytest.mark.parametrize("nruns,kbits,seed", [(2, 12, 1), (3, 17, 2), (4, 20, 3), (8, 22, 4)])
def test_sort_dst_bits_over_concatenated_runs(native, nruns, kbits, seed):
    """The in-CSR receive side before gt_merge_runs: a stable sort over the
    dst bits [kbits, 2*kbits) of >= 2 concatenated (dst, src)-sorted runs with
    disjoint ascending src ranges equals the full sort over (0, 2*kbits)."""
    rng = np.random.default_rng(seed)
    keys, _ = _runs_by_dst_then_src(rng, nruns, kbits, rng.integers(1000, 60000, nruns))
    got = native.sort_keys(keys.cuda(), kbits, 2 * kbits).cpu()
    want = native.sort_keys(keys.cuda(), 0, 2 * kbits).cpu()
    assert torch.equal(got, want)
    assert np.array_equal(got.numpy().view(np.uint64), np.sort(keys.numpy().view(np.uint64)))


@pytest.mark.parametrize("sizes", [[0], [1], [5, 0], [0, 7], [2048, 2048], [1, 2047, 4096, 3],
                                   [100_000, 3, 250_000], [0, 0, 0, 0],
                                   [30_000] * 8, [70_001, 0, 12, 9_999, 400_000, 1, 2, 65_536]])
def test_merge_runs_matches_sort(native, sizes):
    """gt_merge_runs: pairwise merge-path rounds over any number of sorted runs,
    empty and ragged ones included, with heavy duplicates across runs."""
    rng = np.random.default_rng(sum(sizes) + len(sizes))
    runs = [np.sort(rng.integers(0, 1 << 16, size=m).astype(np.uint64) << np.uint64(40)
                    | rng.integers(0, 4, size=m).astype(np.uint64)) for m in sizes]
    keys = torch.from_numpy(np.concatenate(runs).view(np.int64).copy())
    got = native.merge_runs(keys.cuda(), sizes).cpu()
    assert np.array_equal(got.numpy().view(np.uint64), np.sort(keys.numpy().view(np.uint64)))
    assert torch.equal(got, CpuOps().merge_runs(keys, sizes))


def test_merge_runs_in_csr_runs_and_unsigned_order(native):
    """Merging in-CSR runs gives the (dst, src) sort; keys with the top bit set
    order as unsigned (the keys are uint64 bit patterns in int64 tensors)."""
    rng = np.random.default_rng(11)
    keys, sizes = _runs_by_dst_then_src(rng, 4, 20, [50_000, 1, 80_000, 20_000])
    got = native.merge_runs(keys.cuda(), sizes).cpu()
    assert torch.equal(got, native.sort_keys(keys.cuda(), 0, 40).cpu())
    hi = np.uint64(1) << np.uint64(63)
    a = np.sort(rng.integers(0, 1 << 62, 5000).astype(np.uint64) | hi)
    b = np.sort(rng.integers(0, 1 << 62, 7000).astype(np.uint64))
    k = torch.from_numpy(np.concatenate([a, b]).view(np.int64).copy())
    got = native.merge_runs(k.cuda(), [a.size, b.size]).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, np.sort(np.concatenate([a, b])))


def test_merge_runs_rejects_bad_offsets(native):
    k = torch.arange(10, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        native.merge_runs(k, [4, 5])  # sizes do not add up to n
    with pytest.raises(ValueError):
        native.merge_runs(k, [12, -2])


def test_id_map_pack_swap_csr_match_cpu(native):
    rng = np.random.default_rng(3)
    src = torch.from_numpy(rng.integers(-500, 9000, size=20000))
    dst = torch.from_numpy(rng.integers(-500, 9000, size=20000))
    cpu = CpuOps()
    mm = native.id_minmax(src.cuda(), dst.cuda()).cpu()
    assert torch.equal(mm, cpu.id_minmax(src, dst))
    lo, hi = int(mm[0]), int(mm[1])
    span = hi - lo + 1
    flags = native.id_presence(src.cuda(), dst.cuda(), lo, span)
    assert torch.equal(flags.cpu(), cpu.id_presence(src, dst, lo, span))
    words, n = native.id_rankmap(flags)
    cw, cn = cpu.id_rankmap(flags.cpu())
    assert n == cn
    assert torch.equal(native.id_list(words, span, lo, n).cpu(), cpu.id_list(cw, span, lo, n))
    kb = 14
    keys = native.pack_keys(src.cuda(), dst.cuda(), lo, words, kb)
    assert torch.equal(keys.cpu(), cpu.pack_keys(src, dst, lo, cw, kb))
    assert torch.equal(native.swap_halves(keys, kb).cpu(), cpu.swap_halves(keys.cpu(), kb))
    srt = native.unique_keys(native.sort_keys(keys, 0, 2 * kb))
    for row_lo, rows in ((0, n), (100, n - 100), (n // 3, n - n // 3)):
        sel = srt[(srt >> kb) >= row_lo]
        off, adj = native.csr_from_keys(sel, kb, row_lo, rows)
        coff, cadj = cpu.csr_from_keys(sel.cpu(), kb, row_lo, rows)
        assert torch.equal(off.cpu(), coff) and torch.equal(adj.cpu(), cadj)


def _split_rows(in_off, parts):
    n = in_off.shape[0] - 1
    cuts = [n * p // parts for p in range(parts + 1)]
    return cuts


def test_pagerank_row_ranges_emulated(native):
    """3 'ranks' of a dst-row partition, run one after the other; the
    all-gather / all-reduce are done by hand between the steps."""
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(11, 30000, seed=8)
    g = ref.build_csr(src, dst, workers=1)
    n = g.n
    ids = g.ids
    out_off = torch.from_numpy(g.out_off)
    in_off = g.in_off
    in_adj = np.searchsorted(ids, g.in_adj).astype(np.int32)
    inv_full = native.inv_degree(out_off.cuda())
    contrib, dangling = native.pagerank_init(inv_full)
    cuts = _split_rows(in_off, 3)
    iters = 10
    for it in range(iters):
        last = it == iters - 1
        outs, parts = [], []
        for r in range(3):
            a, b = cuts[r], cuts[r + 1]
            loc_off = torch.from_numpy(in_off[a:b + 1] - in_off[a]).cuda()
            loc_adj = torch.from_numpy(in_adj[in_off[a]:in_off[b]].copy()).cuda()
            v, p = native.pagerank_step(loc_off, loc_adj, n, contrib, inv_full[a:b].contiguous(),
                                        dangling, 0.85, last)
            outs.append(v)
            parts.append(p)
        dangling = torch.stack(parts).sum(0)
        if last:
            scores = torch.cat(outs).cpu().numpy()
        else:
            contrib = torch.cat(outs)
    want = ref.pagerank_csr(g, 0.85, iters, workers=1)
    assert float(np.abs(scores - want).sum()) <= 1e-9


def test_triangle_parts_sum_to_total(native):
    import paper_1503_07881_b200 as gt
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(12, 40000, seed=9, permute=True)
    g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
    total = gt.triangle_count(g)
    assert total == ref.triangle_count_fast(ref.build_csr(src, dst))
    for parts in (2, 3, 8):
        assert sum(native.triangles_part(g, p, parts) for p in range(parts)) == total


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_orientation_primitives_match_cpu(native, world):
    """The sharded orientation's per-rank primitives (undirected keys of a row
    range, the (degree, id) rank, the oriented arcs of a row range, the count
    over an orientation) against their CPU restatement, rank slices emulated
    one after another; the parts sum to the single-GPU count."""
    import paper_1503_07881_b200 as gt
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(11, 30000, seed=12 + world, permute=True)
    src = np.concatenate([src, src[:50]])  # self-loops and reciprocal pairs
    dst = np.concatenate([dst, src[:50]])
    want = ref.build_csr(src, dst, workers=1)
    n, k, cpu = want.n, max(1, int(want.n - 1).bit_length()), CpuOps()
    pos = {int(x): i for i, x in enumerate(want.ids)}
    dense = np.array([pos[int(x)] for x in want.out_adj], dtype=np.int32)
    cuts = [n * r // world for r in range(world + 1)]
    und = []
    for r in range(world):
        a, b = cuts[r], cuts[r + 1]
        off = torch.from_numpy(want.out_off[a:b + 1] - want.out_off[a])
        adj = torch.from_numpy(dense[want.out_off[a]:want.out_off[b]])
        got = native.undirected_keys(off.cuda(), adj.cuda(), k, a).cpu()
        exp = cpu.undirected_keys(off, adj, k, a)
        assert torch.equal(torch.sort(got).values, torch.sort(exp).values)
        und.append(exp)
    allk = torch.unique(torch.cat(und))
    uoff, uadj = cpu.csr_from_keys(allk, k, 0, n)
    deg = uoff[1:] - uoff[:-1]
    rank = native.degree_rank(deg.cuda()).cpu()
    assert torch.equal(rank, cpu.degree_rank(deg))
    arcs = []
    for r in range(world):
        a, b = cuts[r], cuts[r + 1]
        off = uoff[a:b + 1] - uoff[a]
        adj = uadj[uoff[a]:uoff[b]]
        got = native.orient_keys(off.cuda(), adj.cuda(), a, rank.cuda(), k).cpu()
        assert torch.equal(got, cpu.orient_keys(off, adj, a, rank, k))
        arcs.append(got)
    off_p, adj_p = cpu.csr_from_keys(torch.sort(torch.cat(arcs)).values, k, 0, n)
    g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
    total = gt.triangle_count(g)
    parts = [native.triangles_oriented_part(off_p.cuda(), adj_p.cuda(), p, world)
             for p in range(world)]
    assert parts == [cpu.triangles_oriented_part(off_p, adj_p, p, world) for p in range(world)]
    assert sum(parts) == total == ref.triangle_count_fast(want)


def test_nccl_world1_pipeline_matches_oracle(native):
    import torch.distributed as dist

    from paper_1503_07881_b200 import distributed as D
    from paper_1503_07881_b200.synth import rmat_edges

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        src, dst = rmat_edges(12, 50000, seed=10, permute=True)
        sg = D.build_csr(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), ops=native)
        out_off, out_adj, in_off, in_adj = D.gather_csr(sg)
        want = ref.build_csr(src, dst, workers=1)
        ids = sg.ids.cpu().numpy()
        assert np.array_equal(ids, want.ids)
        assert np.array_equal(out_off.cpu().numpy(), want.out_off)
        assert np.array_equal(in_off.cpu().numpy(), want.in_off)
        assert np.array_equal(ids[out_adj.cpu().numpy()], want.out_adj)
        assert np.array_equal(ids[in_adj.cpu().numpy()], want.in_adj)
        pr = D.pagerank(sg, 0.85, 10, ops=native).cpu().numpy()
        assert float(np.abs(pr - ref.pagerank_csr(want, 0.85, 10, workers=1)).sum()) <= 1e-9
        assert D.triangle_count(sg, ops=native) == ref.triangle_count_fast(want)
    finally:
        dist.destroy_process_group()
