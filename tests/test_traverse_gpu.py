"""BFS hop distances, weakly connected components and k-core on the B200
(csrc/traverse.cu) against the real reference's outputs
(tests/golden/traverse.npz) and the oracle restatement at larger sizes."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import golden_traverse
from oracle import reference_port as ref
from paper_1503_07881_b200.errors import UnknownNodeError
from paper_1503_07881_b200.synth import rmat_edges

pytestmark = pytest.mark.gpu

SPEC = gt.EdgeSpec("src", "dst")
TRAVERSE = sorted(golden_traverse())


def device_graph(case):
    if case["extra"].size:
        g = gt.from_edges(list(zip(case["src"].tolist(), case["dst"].tolist())))
        for x in case["extra"].tolist():
            g.add_node(x)
        return gt.upload(g)
    return gt.table_to_graph(gt.edge_table(case["src"], case["dst"]), SPEC)


@pytest.mark.parametrize("name", TRAVERSE)
def test_traversals_match_reference(name):
    case = golden_traverse()[name]
    g = device_graph(case)
    ids = case["ids"]
    assert np.array_equal(np.asarray(g.node_ids()), ids)
    for row, s in zip(case["sssp"], case["sources"].tolist()):
        d = gt.sssp(g, s)
        assert [(-1 if d[i] is None else d[i]) for i in ids.tolist()] == row.tolist()
    cc = gt.connected_components(g)
    assert [cc[i] for i in ids.tolist()] == case["cc"].tolist()
    for k in (1, 2, 3, 4):
        core = gt.k_core(g, k)
        h = core.csr()
        assert np.array_equal(h.ids, case[f"kcore{k}_ids"])
        assert np.array_equal(h.out_off, case[f"kcore{k}_out_off"])
        assert np.array_equal(h.out_adj, case[f"kcore{k}_out_adj"])


@pytest.mark.parametrize("scale,rows,seed", [(14, 200_000, 3), (16, 1_000_000, 4)])
def test_rmat_vs_oracle(scale, rows, seed):
    src, dst = rmat_edges(scale, rows, seed=seed, permute=True)
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    want = ref.build_csr(src, dst)
    und = ref.undirected_dense(want)
    rng = np.random.default_rng(seed)
    for s in rng.integers(0, want.n, size=3).tolist():
        d = gt.sssp(g, int(want.ids[s]))
        assert np.array_equal(d.values_, ref.sssp_csr(want, s))
    cc = gt.connected_components(g)
    assert np.array_equal(cc.values_, ref.components_csr(want, und))
    for k in (2, 5, 9):
        core = gt.k_core(g, k).csr()
        w = ref.k_core_csr(want, k, und)
        for f in ("ids", "out_off", "out_adj", "in_off", "in_adj"):
            assert np.array_equal(getattr(core, f), getattr(w, f)), f


def test_bfs_levels_on_long_path_and_star():
    """A 5000-hop path (5000 top-down levels) and a 20000-leaf star (one
    bottom-up level)."""
    n = 5000
    g = gt.table_to_graph(gt.edge_table(np.arange(n), np.arange(1, n + 1)), SPEC)
    d = gt.sssp(g, 0)
    assert d.values_.tolist() == list(range(n + 1))
    assert gt.sssp(g, n)[0] is None
    leaves = np.arange(1, 20001)
    g = gt.table_to_graph(gt.edge_table(np.zeros_like(leaves), leaves), SPEC)
    d = gt.sssp(g, 0)
    assert d[0] == 0 and set(d.values_[1:].tolist()) == {1}


def test_errors_and_empty_graphs():
    g = gt.table_to_graph(gt.edge_table(np.array([0, 1]), np.array([1, 2])), SPEC)
    with pytest.raises(UnknownNodeError):
        gt.sssp(g, 7)
    with pytest.raises(UnknownNodeError):
        gt.sssp(gt.Graph(), 3)
    with pytest.raises(ValueError):
        gt.k_core(g, 0)
    empty = gt.table_to_graph(gt.edge_table(np.zeros(0, np.int64), np.zeros(0, np.int64)), SPEC)
    assert len(gt.connected_components(empty)) == 0
    assert gt.k_core(empty, 1).node_count == 0
    assert gt.k_core(g, 2).node_count == 0  # a path has no 2-core


def test_components_hooking_is_order_independent():
    """Many components whose smallest ids appear late in the table."""
    rng = np.random.default_rng(5)
    blocks = [(rng.integers(0, 300, size=900) * 50 + (49 - b),
               rng.integers(0, 300, size=900) * 50 + (49 - b)) for b in range(50)]
    src = np.concatenate([b[0] for b in blocks])
    dst = np.concatenate([b[1] for b in blocks])
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    want = ref.build_csr(src, dst)
    assert np.array_equal(gt.connected_components(g).values_, ref.components_csr(want))
