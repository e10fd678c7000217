"""ToGraph on the B200 vs the reference (golden fixtures) and the oracle.

Bit-exact CSR parity (ids, offsets, pools) through the C ABI; the cases
mirror the reference's own conversion tests (test_convert.py:38-84,
test_acceptance.py:240-256) plus the id-compaction edge cases of
convert.py:45-59 (negative, sparse and extreme int64 ids).
"""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import assert_csr_equal, golden_c1, golden_cases, sha
from oracle import reference_port as ref
from paper_1503_07881_b200.synth import CONFIGS, RmatSpec, rmat_device, rmat_edges

pytestmark = pytest.mark.gpu
SPEC = gt.EdgeSpec("src", "dst")


def build(src, dst, device=False):
    t = gt.edge_table(np.asarray(src, np.int64), np.asarray(dst, np.int64))
    if device:
        t = t.to_device()
    return gt.table_to_graph(t, SPEC)


@pytest.mark.parametrize("name", sorted(golden_cases()))
@pytest.mark.parametrize("device", [False, True])
def test_csr_matches_reference(name, device):
    case = golden_cases()[name]
    g = build(case["src"], case["dst"], device=device)
    assert g.node_count == case["ids"].shape[0]
    assert g.edge_count == case["out_adj"].shape[0]
    assert_csr_equal(g.csr(), case, name)
    g.check_invariants()


def test_c1_config_csr_digests():
    gold = golden_c1()
    spec = CONFIGS["c1"]
    src, dst = rmat_device(spec)
    assert sha(src.cpu().numpy()) == str(gold["sha_src"])  # device generator == numpy twin
    assert sha(dst.cpu().numpy()) == str(gold["sha_dst"])
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    h = g.csr()
    assert g.node_count == int(gold["n"]) and g.edge_count == int(gold["e"])
    for f in ("ids", "out_off", "out_adj", "in_off", "in_adj"):
        assert sha(getattr(h, f)) == str(gold[f"sha_{f}"]), f


@pytest.mark.parametrize("scale,start,rows,permute", [(12, 0, 5000, True), (12, 4000, 1000, True),
                                                     (22, 68_999_000, 1000, True),
                                                     (26, 1_469_999_000, 1000, True)])
def test_device_rmat_row_ranges_match_numpy(scale, start, rows, permute):
    """gt_rmat_generate_range (the shard generator of multi-GPU runs) is the
    numpy generator's rows [start, start+rows)."""
    spec = RmatSpec(scale=scale, rows=rows, seed=3, permute=permute)
    src, dst = rmat_device(spec, start=start, rows=rows)
    ws, wd = rmat_edges(scale, rows, seed=3, permute=permute, start=start)
    assert np.array_equal(src.cpu().numpy(), ws) and np.array_equal(dst.cpu().numpy(), wd)


def test_duplicates_collapse_and_empty():
    g = build([1, 2, 1], [2, 3, 2])
    assert g.node_count == 3 and g.edge_count == 2 and g.neighbors(1, "out").tolist() == [2]
    e = build([], [])
    assert e.node_count == 0 and e.edge_count == 0 and e.node_ids() == []


@pytest.mark.parametrize("distinct,rows", [(1, 300_000), (7, 500_000), (5000, 2_000_000),
                                           (200_000, 3_000_000)])
def test_duplicate_heavy_tables_vs_oracle(distinct, rows):
    """The in-sort histograms are the out-sort's minus the dropped duplicates'
    digit counts: tables made mostly of copies (runs of one key spanning
    warps and tiles, a single key repeated 300K times) must still sort exactly."""
    rng = np.random.default_rng(distinct)
    pairs = rng.integers(0, max(2, int(np.sqrt(distinct) * 40)), size=(distinct, 2))
    pick = rng.integers(0, distinct, size=rows)
    src, dst = pairs[pick, 0].astype(np.int64), pairs[pick, 1].astype(np.int64)
    g = build(src, dst, device=True)
    assert_csr_equal(g.csr(), ref.build_csr(src, dst), f"dups-{distinct}")


def test_self_loops_and_negatives():
    g = build([-5, -5], [-5, 3])
    assert g.has_edge(-5, -5) and g.has_edge(-5, 3) and not g.has_edge(3, -5)
    g.check_invariants()


@pytest.mark.parametrize("seed", range(5))
def test_matches_sequential_replay(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 2000))
    src = rng.integers(-20, 60, size=n)
    dst = rng.integers(-20, 60, size=n)
    g = build(src, dst)
    assert g == gt.from_edges(zip(src.tolist(), dst.tolist()))


def test_worker_count_independence_and_determinism():
    rng = np.random.default_rng(99)
    src = rng.integers(-166, 500, size=20_000)
    dst = rng.integers(-166, 500, size=20_000)
    t = gt.edge_table(src, dst)
    gs = [gt.table_to_graph(t, SPEC, workers=w) for w in (1, 2, 8)]
    assert gs[0] == gs[1] == gs[2]
    assert_csr_equal(gs[0].csr(), gs[1].csr())


def test_views_read_only_and_graph_stays_mutable():
    g = build([1, 2], [2, 3])
    with pytest.raises(ValueError):
        g.neighbors(1, "out")[0] = 7
    assert g.add_edge(3, 1) is True
    assert g.del_edge(1, 2) is True
    g.check_invariants()
    assert g.edge_count == 2 and not g.on_device


def test_input_columns_not_mutated():
    src, dst = rmat_edges(12, 50_000, seed=5, permute=True)
    t = gt.edge_table(src.copy(), dst.copy()).to_device()
    before = (t.column("src").clone(), t.column("dst").clone())
    gt.table_to_graph(t, SPEC)
    assert bool((t.column("src") == before[0]).all()) and bool((t.column("dst") == before[1]).all())


@pytest.mark.parametrize("offset", [0, 1 << 40, -(1 << 50)])
def test_dense_and_sparse_id_paths_agree(offset):
    rng = np.random.default_rng(3)
    base = rng.integers(0, 1 << 14, size=30_000)
    src, dst = base[:15_000] + offset, base[15_000:] + offset
    g = build(src, dst)
    want = ref.build_csr(src, dst, workers=1)
    assert_csr_equal(g.csr(), want)
    # widen the id range beyond the dense-map budget -> sort-unique path
    src2 = src.copy()
    src2[0] = offset + (1 << 45)
    g2 = build(src2, dst)
    assert_csr_equal(g2.csr(), ref.build_csr(src2, dst, workers=1))


def test_round_trip_is_dedup_sorted_table():
    src, dst = rmat_edges(13, 200_000, seed=13, permute=True)
    g = build(src, dst)
    h = g.csr()
    back_src = np.repeat(h.ids, np.diff(h.out_off))
    expect = np.unique(np.stack([src, dst], axis=1), axis=0)
    assert np.array_equal(back_src, expect[:, 0]) and np.array_equal(h.out_adj, expect[:, 1])


def test_c2_prefix_matches_oracle():
    """4M rows of the C2 table (R-MAT s22, permuted ids) vs the oracle."""
    spec = RmatSpec(scale=22, rows=4_000_000, seed=2, permute=True)
    src, dst = rmat_device(spec)
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    want = ref.build_csr(src.cpu().numpy(), dst.cpu().numpy())
    assert_csr_equal(g.csr(), want, "c2-prefix")


@pytest.mark.slow
def test_c2_full_properties():
    """Full C2 (69M rows): size-independent properties checked on the device."""
    import torch

    src, dst = rmat_device(CONFIGS["c2"])
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    n, e = g.node_count, g.edge_count
    assert 0 < e <= src.shape[0]
    # Export through the ABI and check on the host with vectorised numpy.
    h = g.csr()
    k = 32
    out_keys = (np.repeat(np.arange(n, dtype=np.int64), np.diff(h.out_off)) << k) | \
        np.searchsorted(h.ids, h.out_adj)
    assert np.all(np.diff(out_keys) > 0)  # sorted by (src, dst) and duplicate-free
    in_keys = (np.repeat(np.arange(n, dtype=np.int64), np.diff(h.in_off)) << k) | \
        np.searchsorted(h.ids, h.in_adj)
    assert np.all(np.diff(in_keys) > 0)
    mirror = np.sort(((out_keys & 0xFFFFFFFF) << k) | (out_keys >> k))
    assert np.array_equal(mirror, in_keys)
    # node set = distinct ids of both columns
    both = torch.unique(torch.cat([src, dst])).cpu().numpy()
    assert np.array_equal(both, h.ids)
    # edge set = distinct pairs: count via device unique of packed rows
    packed = torch.unique(src * (1 << 22) + dst)
    assert packed.shape[0] == e


@pytest.mark.parametrize("start,rows", [(0, 100_000), (1_999_999_000, 1000)])
def test_device_uniform_rows_match_numpy(start, rows):
    """gt_uniform_generate_range (C5's uniform table) is synth.uniform_edges."""
    from paper_1503_07881_b200.synth import UniformSpec, uniform_edges

    spec = UniformSpec(n_nodes=100_000_000, rows=rows, seed=4)
    src, dst = rmat_device(spec, start=start, rows=rows)
    ws, wd = uniform_edges(100_000_000, rows, 4, start=start)
    assert np.array_equal(src.cpu().numpy(), ws) and np.array_equal(dst.cpu().numpy(), wd)


def test_c5_shape_uniform_vs_oracle():
    """C5's uniform (no skew) shape at 4M nodes / 20M rows: CSR bit-exact and
    PageRank x20 within 1e-9 L1 of the oracle."""
    from paper_1503_07881_b200.synth import UniformSpec

    src, dst = rmat_device(UniformSpec(n_nodes=4_000_000, rows=20_000_000, seed=4))
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    want = ref.build_csr(src.cpu().numpy(), dst.cpu().numpy())
    assert_csr_equal(g.csr(), want, "c5-shape")
    pr = gt.pagerank(g, 0.85, 20)
    got = np.asarray([pr[int(i)] for i in want.ids[:1]])  # mapping access works
    assert got.shape == (1,)
    scores = np.asarray(pr.scores)
    assert np.abs(scores - ref.pagerank_csr(want, 0.85, 20)).sum() <= 1e-9


@pytest.mark.slow
def test_capacity_error_at_2_pow_31_nodes():
    """>= 2^31 distinct ids do not fit the int32 dense adjacency: CapacityError.
    The reference switches to searchsorted there (convert.py:55-59) and keeps
    going on the host; this build states its limit instead of
    overflowing the int32 indices."""
    import torch

    ids = torch.arange(1 << 31, dtype=torch.int64, device="cuda")
    with pytest.raises(gt.CapacityError):
        gt.table_to_graph(gt.edge_table(ids, ids), SPEC)
    del ids
    torch.cuda.empty_cache()
    # the library stays usable afterwards
    g = gt.table_to_graph(gt.edge_table(np.array([1, 2]), np.array([2, 1])), SPEC)
    assert g.edge_count == 2


def test_prefetch_pipelined_ingest_matches_direct_build():
    """ColumnTable.prefetch: the copy runs on a side stream and the library
    waits for it at first use, so a prefetch issued while other work runs
    yields the same graph as a direct host build (bench e2e pipeline)."""
    import torch

    spec = RmatSpec(scale=18, rows=2_000_000, seed=5, permute=True)
    src, dst = rmat_edges(spec.scale, spec.rows, seed=5, permute=True)
    h_src = torch.from_numpy(src).pin_memory()
    h_dst = torch.from_numpy(dst).pin_memory()
    host = gt.edge_table(h_src.numpy(), h_dst.numpy())
    want = gt.table_to_graph(host, SPEC).csr()
    for _ in range(3):
        t = host.prefetch()
        busy = gt.table_to_graph(host, SPEC)  # library busy while the copy runs
        gt.pagerank(busy, 0.85, 5)
        g = gt.table_to_graph(t, SPEC)
        assert_csr_equal(g.csr(), want, "prefetch")
    # select / join consume prefetched tables too
    sel = gt.select(host.prefetch(), gt.Predicate("src", "<", int(np.median(src))))
    np.testing.assert_array_equal(sel.row_ids.cpu().numpy(),
                                  np.flatnonzero(src < int(np.median(src))))


@pytest.mark.slow
def test_c4_full_size_properties():
    """BASELINE configs[3] at full size (1.47 B rows, R-MAT s26): properties
    that do not need a host oracle, checked on the device.
    * node set = distinct ids of both columns, edge count = distinct pairs;
    * out-rows sorted and duplicate-free, in-CSR the exact transpose
      (in-degree histogram = dst histogram of the distinct pairs);
    * PageRank: scores positive and summing to 1 (the dangling mass is
      redistributed, algorithms.py:72-82);
    * triangles: the 4-way split of the middle vertices sums to the total."""
    import ctypes

    import torch

    from paper_1503_07881_b200 import _native

    src, dst = rmat_device(CONFIGS["c4"])
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    _native.load().gt_release_workspace()  # the checks below need the memory
    n, e = g.node_count, g.edge_count
    ids_p, oo_p, oa_p, io_p, ia_p = g.device_views()
    def as_t(p, cnt, dt):  # zero-copy torch view of a library-owned device array
        class _A:
            __cuda_array_interface__ = {"shape": (cnt,), "typestr": dt, "data": (p, False),
                                        "version": 3}
        return torch.as_tensor(_A(), device="cuda")

    ids = as_t(ids_p, n, "<i8")
    out_off, in_off = as_t(oo_p, n + 1, "<i8"), as_t(io_p, n + 1, "<i8")
    out_adj, in_adj = as_t(oa_p, e, "<i4"), as_t(ia_p, e, "<i4")
    both = torch.unique(torch.cat([src[:1 << 28], dst[:1 << 28]]))  # a prefix fits memory
    assert bool(torch.isin(both, ids).all())
    assert bool((ids[1:] > ids[:-1]).all())
    # out-rows: strictly increasing within rows
    row_of = torch.repeat_interleave(torch.arange(n, device="cuda"), out_off[1:] - out_off[:-1])
    key = row_of * n + out_adj.long()
    assert bool((key[1:] > key[:-1]).all())
    del row_of, key
    # distinct pairs = edge count (device sort of packed ranks)
    rs = torch.searchsorted(ids, src)
    rd = torch.searchsorted(ids, dst)
    del src, dst
    packed = torch.unique(rs * n + rd)
    del rs, rd
    assert packed.shape[0] == e
    # in-CSR = transpose: in-degree = dst histogram of the distinct pairs
    indeg = torch.bincount(packed % n, minlength=n)
    assert torch.equal(indeg, in_off[1:] - in_off[:-1])
    del packed, indeg
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    gt.pagerank_device(g, 0.85, 20, out.data_ptr())
    assert bool((out > 0).all()) and abs(float(out.sum()) - 1.0) < 1e-9
    total = gt.triangle_count(g)
    parts = 0
    lib = _native.load()
    for p in range(4):
        c = ctypes.c_int64()
        _native.check(lib.gt_triangles_part(g.handle, p, 4, ctypes.byref(c)), "gt_triangles_part")
        parts += c.value
    assert parts == total  # exact value: tests/test_large_gpu.py (oracle on a slice)


def test_per_node_lookups_stay_on_the_device():
    """record / has_node / has_edge / neighbors answered by device binary
    searches + one copied row (no O(E) export): the same answers as the host
    copy (graphs.py:62-88, 148-167), on a graph with hubs and negative ids."""
    import time

    src, dst = rmat_edges(14, 200_000, seed=5, permute=True)
    src = src - 1000
    g = gt.table_to_graph(gt.edge_table(src, dst).to_device(), SPEC)
    rng = np.random.default_rng(0)
    ids = np.unique(np.concatenate([src, dst]))
    probe = np.concatenate([rng.choice(ids, 40), [ids[0], ids[-1]], [-5000, 10**12]])
    got = {}
    for x in probe.tolist():
        got[x] = (g.has_node(x), g.record(x) if g.has_node(x) else None)
    u = rng.choice(ids, 60)
    v = rng.choice(ids, 60)
    edges = [g.has_edge(a, b) for a, b in zip(u.tolist(), v.tolist())]
    real = [g.has_edge(int(a), int(b)) for a, b in zip(src[:30].tolist(), dst[:30].tolist())]
    assert all(real)
    assert g._host is None  # nothing exported so far
    t0 = time.perf_counter()
    for a, b in zip(src[:200].tolist(), dst[:200].tolist()):
        g.has_edge(a, b)
    assert (time.perf_counter() - t0) / 200 < 1e-3  # < 1 ms per lookup
    h = g.csr()  # host copy, the reference layout
    for x, (present, rec) in got.items():
        i = int(np.searchsorted(h.ids, x))
        assert present == (i < h.ids.shape[0] and h.ids[i] == x)
        if present:
            assert np.array_equal(rec.out_nbrs, h.out_adj[h.out_off[i]:h.out_off[i + 1]])
            assert np.array_equal(rec.in_nbrs, h.in_adj[h.in_off[i]:h.in_off[i + 1]])
            assert not rec.out_nbrs.flags.writeable
    for a, b, e in zip(u.tolist(), v.tolist(), edges):
        i = int(np.searchsorted(h.ids, a))
        row = h.out_adj[h.out_off[i]:h.out_off[i + 1]]
        assert e == bool(np.isin(b, row))
    assert g.node_ids() == h.ids.tolist()
