"""Strongly connected components on the B200 (csrc/scc.cu; SURVEY §8f next
#4; algorithms.scc, algorithms.py:144-203) against the real reference's
labels (tests/golden/scc.npz: 25 graphs incl. rings of rings, chains with
back edges, interleaved cycles, DAGs, isolated nodes) and, at larger sizes,
against the oracle's Tarjan restatement and scipy's strong components
(same partition, labels by ascending smallest id)."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import golden_scc
from oracle import reference_port as ref
from paper_1503_07881_b200.synth import rmat_edges

pytestmark = pytest.mark.gpu

SPEC = gt.EdgeSpec("src", "dst")


def device_graph(case):
    if case["extra"].size:
        g = gt.from_edges(list(zip(case["src"].tolist(), case["dst"].tolist())))
        for x in case["extra"].tolist():
            g.add_node(x)
        return gt.upload(g)
    return gt.table_to_graph(gt.edge_table(case["src"], case["dst"]), SPEC)


@pytest.mark.parametrize("name", sorted(golden_scc()))
def test_scc_matches_reference(name):
    case = golden_scc()[name]
    g = device_graph(case)
    lab = gt.scc(g)
    assert [lab[i] for i in case["ids"].tolist()] == case["scc"].tolist()


def labels_by_min_id(comp):
    """Relabel a component array densely by first occurrence (ascending index)."""
    _, first, inv = np.unique(comp, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.shape[0])
    return rank[inv]


@pytest.mark.parametrize("scale,rows,seed", [(12, 40_000, 5), (16, 1_000_000, 6),
                                             (20, 8_000_000, 7)])
def test_scc_rmat_vs_scipy(scale, rows, seed):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    src, dst = rmat_edges(scale, rows, seed=seed, permute=True)
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    want = ref.build_csr(src, dst)
    n = want.ids.shape[0]
    col = np.searchsorted(want.ids, want.out_adj)
    a = csr_matrix((np.ones(col.shape[0], np.int8), col, want.out_off), shape=(n, n))
    _, comp = connected_components(a, directed=True, connection="strong")
    lab = gt.scc(g)
    assert np.array_equal(lab.values_, labels_by_min_id(comp))
    if rows <= 40_000:
        assert np.array_equal(lab.values_, ref.scc_csr(want))


def test_scc_empty_and_trivial():
    assert len(gt.scc(gt.Graph())) == 0
    g = gt.table_to_graph(gt.edge_table(np.array([5, 6, 7]), np.array([6, 7, 5])), SPEC)
    lab = gt.scc(g)
    assert [lab[i] for i in (5, 6, 7)] == [0, 0, 0]
    g = gt.table_to_graph(gt.edge_table(np.array([9, 3]), np.array([3, 9])), SPEC)
    assert dict(gt.scc(g).items()) == {3: 0, 9: 0}
