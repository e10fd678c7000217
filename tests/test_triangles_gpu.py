"""Triangle counting on the B200: exact vs the reference (golden), the cubic
brute-force oracle (oracles.py:163-167) and the C restatement."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import cubic_triangles, golden_c1, golden_cases, random_digraph_edges
from oracle import reference_port as ref
from paper_1503_07881_b200.synth import CONFIGS, RmatSpec, rmat_device

pytestmark = pytest.mark.gpu
SPEC = gt.EdgeSpec("src", "dst")


def build(src, dst):
    return gt.table_to_graph(gt.edge_table(np.asarray(src, np.int64),
                                           np.asarray(dst, np.int64)), SPEC)


@pytest.mark.parametrize("name", sorted(golden_cases()))
def test_matches_reference(name):
    case = golden_cases()[name]
    assert gt.triangle_count(build(case["src"], case["dst"])) == int(case["tc"][0])


def test_c1_config_matches_reference():
    src, dst = rmat_device(CONFIGS["c1"])
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    assert gt.triangle_count(g) == int(golden_c1()["tc"][0])


def test_known_answers():
    k4 = [(a, b) for a in range(4) for b in range(4) if a < b]
    assert gt.triangle_count(gt.from_edges(k4)) == 4
    assert gt.triangle_count(gt.from_edges([(i, i + 1) for i in range(9)])) == 0
    assert gt.triangle_count(gt.from_edges([(0, 0), (0, 1), (1, 2), (2, 0)])) == 1
    assert gt.triangle_count(build([], [])) == 0
    assert gt.triangle_count(build([5], [5])) == 0


def test_direction_flips_do_not_change_count():
    rng = np.random.default_rng(4)
    src, dst = random_digraph_edges(rng, 40, 0.1)
    base = gt.triangle_count(build(src, dst))
    flip = rng.random(src.shape[0]) < 0.5
    s2 = np.where(flip, dst, src)
    d2 = np.where(flip, src, dst)
    assert gt.triangle_count(build(s2, d2)) == base


def test_random_vs_cubic_enumeration():
    rng = np.random.default_rng(77)
    for i in range(50):
        n = int(rng.integers(2, 41)) if i % 2 else int(rng.integers(40, 129))
        p = float(rng.uniform(0.05, 0.4)) if i % 2 else float(rng.uniform(0.01, 8 / n))
        src, dst = random_digraph_edges(rng, n, p)
        adj = np.zeros((n, n), dtype=bool)
        adj[src, dst] = True
        want = cubic_triangles(adj | adj.T)
        got = gt.triangle_count(build(src, dst)) if src.size else 0
        assert got == want


def test_hub_heavy_graph_vs_oracle():
    """Dense core (d+(u) beyond the shared-memory cap) + long tails."""
    rng = np.random.default_rng(5)
    core = rng.integers(0, 3000, size=(400_000, 2))
    tail = rng.integers(0, 200_000, size=(300_000, 2))
    e = np.concatenate([core, tail])
    g = build(e[:, 0], e[:, 1])
    want = ref.triangle_count_fast(ref.build_csr(e[:, 0], e[:, 1]))
    assert gt.triangle_count(g) == want


def test_c3_prefix_vs_oracle():
    src, dst = rmat_device(RmatSpec(scale=22, rows=4_000_000, seed=2, permute=True))
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    want = ref.triangle_count_fast(ref.build_csr(src.cpu().numpy(), dst.cpu().numpy()))
    assert gt.triangle_count(g) == want


def test_repeatable():
    src, dst = rmat_device(RmatSpec(scale=18, rows=2_000_000, seed=9, permute=True))
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    assert gt.triangle_count(g) == gt.triangle_count(g)


@pytest.mark.slow
def test_c3_full_vs_oracle():
    src, dst = rmat_device(CONFIGS["c2"])
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    h = g.csr()
    want = ref.triangle_count_fast(ref.CSR(h.ids, h.out_off, h.out_adj, h.in_off, h.in_adj))
    assert gt.triangle_count(g) == want


@pytest.mark.parametrize("window,smem_cap,cta_window", [
    (None, None, None), ("64", None, None), ("64", "1024", None), ("256", None, None),
    ("64", None, "1024"), ("64", None, "700")])
def test_hub_orientation_all_table_paths(monkeypatch, window, smem_cap, cta_window):
    """K_n with n = 1200: oriented out-degrees 0..1199. GT_TC_WINDOW shrinks
    the bitmap window so that the split (bitmap + hash), warp-hash and CTA
    paths all run; GT_TC_TABLE_SMEM_MAX forces the CTA path's global table;
    GT_TC_CTA_WINDOW turns on the CTA bitmap for the CTA tasks within that
    distance of the top (700: some CTA tasks bitmap, the rest hash)."""
    if window is not None:
        monkeypatch.setenv("GT_TC_WINDOW", window)
    if smem_cap is not None:
        monkeypatch.setenv("GT_TC_TABLE_SMEM_MAX", smem_cap)
    if cta_window is not None:
        monkeypatch.setenv("GT_TC_CTA_WINDOW", cta_window)
    n = 1200
    a, b = np.triu_indices(n, 1)
    rng = np.random.default_rng(5)
    flip = rng.random(a.shape[0]) < 0.5
    src = np.where(flip, b, a) * 7 + 3
    dst = np.where(flip, a, b) * 7 + 3
    want = n * (n - 1) * (n - 2) // 6
    assert gt.triangle_count(build(src, dst)) == want


@pytest.mark.parametrize("n", [2600, 5000])
def test_clique_rows_past_the_warp_sorts(n):
    """K_n: oriented rows of every length up to n-1, so the packed (<= 32),
    warp-radix, mid (warp per row, larger buffers) and CTA-bitonic row sorts
    all run; at n = 5000 every row has more than TC_FILL_BIG candidates (the
    chunked hub fill). Every rank-space row must come out strictly ascending."""
    from paper_1503_07881_b200 import _native

    a, b = np.triu_indices(n, 1)
    rng = np.random.default_rng(17)
    flip = rng.random(a.shape[0]) < 0.5
    src = np.where(flip, b, a) * 3 - 1000
    dst = np.where(flip, a, b) * 3 - 1000
    dg = build(src, dst)
    deg, rank, off, adj = _native.triangle_orientation(dg.handle, dg.node_count)
    assert np.all(deg == n - 1)
    d = np.diff(off)
    assert sorted(d.tolist()) == list(range(n))
    inner = np.ones(adj.shape[0], dtype=bool)
    starts = off[1:-1]
    inner[starts[starts < adj.shape[0]]] = False  # a row's first element vs the previous row
    assert np.all(np.diff(adj)[inner[1:]] > 0)
    assert gt.triangle_count(dg) == n * (n - 1) * (n - 2) // 6


@pytest.mark.parametrize("window", ["64", "1024"])
def test_small_windows_match_reference_on_rmat(monkeypatch, window):
    from paper_1503_07881_b200.synth import rmat_edges

    monkeypatch.setenv("GT_TC_WINDOW", window)
    src, dst = rmat_edges(13, 60000, seed=12, permute=True)
    want = ref.triangle_count_fast(ref.build_csr(src, dst))
    assert gt.triangle_count(build(src, dst)) == want


def test_clique_plus_sparse_tail():
    """A 1100-clique glued to a sparse random graph: mixes warp and CTA tasks."""
    rng = np.random.default_rng(9)
    n = 1100
    a, b = np.triu_indices(n, 1)
    s2, d2 = random_digraph_edges(rng, 300, 0.03)
    src = np.concatenate([a, s2 + n - 50])
    dst = np.concatenate([b, d2 + n - 50])
    want = ref.triangle_count_fast(ref.build_csr(src.astype(np.int64), dst.astype(np.int64)))
    assert gt.triangle_count(build(src, dst)) == want


def _reference_orientation(src, dst):
    """algorithms.py:97-108 restated: undirected degree and higher(i) sets."""
    g = ref.build_csr(np.asarray(src, np.int64), np.asarray(dst, np.int64))
    deg, higher = ref.orientation_dense(g)
    return g, deg, higher


@pytest.mark.parametrize("name", ["random_500x20000", "rmat_s10"])
def test_orientation_matches_reference(name):
    from paper_1503_07881_b200 import _native

    if name == "rmat_s10":
        from paper_1503_07881_b200.synth import rmat_edges

        src, dst = rmat_edges(10, 8192, seed=11)
    else:
        case = golden_cases()[name]
        src, dst = case["src"], case["dst"]
    g, want_deg, want_higher = _reference_orientation(src, dst)
    dg = build(src, dst)
    deg, rank, off, adj = _native.triangle_orientation(dg.handle, dg.node_count)
    assert np.array_equal(deg, want_deg)
    n = dg.node_count
    want_rank = np.empty(n, dtype=np.int64)
    want_rank[np.lexsort((np.arange(n), want_deg))] = np.arange(n)  # algorithms.py:104-106
    assert np.array_equal(rank, want_rank)
    order = np.argsort(rank)
    for r in range(n):  # rank-space rows, ascending, = higher(order[r]) relabelled
        row = adj[off[r]:off[r + 1]]
        assert np.all(np.diff(row) > 0)
        assert sorted(order[row].tolist()) == sorted(want_higher[order[r]].tolist())
    assert gt.triangle_count(dg) == ref.triangle_count_fast(g)


def test_pagerank_and_triangles_on_two_lanes_match_serial():
    """pagerank_and_triangles runs PageRank on lane 1 next to the count on
    lane 0 (own streams and workspaces): same scores (bitwise) and count as
    the serial calls, repeatedly."""
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(18, 3_000_000, seed=21, permute=True)
    g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
    pr0 = gt.pagerank(g, 0.85, 20)
    tc0 = gt.triangle_count(g)
    for _ in range(3):
        pr, tc = gt.pagerank_and_triangles(g, 0.85, 20)
        assert tc == tc0
        assert np.array_equal(np.asarray(pr.scores), np.asarray(pr0.scores))


@pytest.mark.slow
def test_c2_c3_full_size_vs_oracles():
    """BASELINE configs[1] / [2] at full size (69 M rows, R-MAT s22, permuted
    ids): CSR arrays bit-exact and PageRank x20 within 1e-9 L1 against the
    numpy port, the C3 triangle total against the C/OpenMP oracle."""
    import time

    from paper_1503_07881_b200.synth import CONFIGS, rmat_device

    src, dst = rmat_device(CONFIGS["c2"])
    g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
    h_src, h_dst = src.cpu().numpy(), dst.cpu().numpy()
    del src, dst
    t0 = time.perf_counter()
    want = ref.build_csr(h_src, h_dst)
    h = g.csr()
    for f in ("ids", "out_off", "out_adj", "in_off", "in_adj"):
        assert np.array_equal(getattr(h, f), getattr(want, f)), f
    pr = gt.pagerank(g, 0.85, 20)
    assert np.abs(np.asarray(pr.scores) - ref.pagerank_csr(want, 0.85, 20)).sum() <= 1e-9
    tc = gt.triangle_count(g)
    assert tc == ref.triangle_count_fast(want)
    print(f"c2/c3 full size: N={h.ids.shape[0]} E={h.out_adj.shape[0]} triangles={tc} "
          f"(oracles {time.perf_counter() - t0:.0f}s)")
