"""Graph -> table on the B200: graph_to_edge_table
(convert.py:178-197), graph_to_node_table (convert.py:200-217),
table_from_map (tables.py:662-670) and the front-end TableFromHashMap /
GraphToTable, against the oracle CSR and the reference's round-trip property
(test_acceptance.py:240-256: the exported table is the deduplicated, sorted
input)."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import golden_cases
from oracle import reference_port as ref
from paper_1503_07881_b200.errors import CoverageError

pytestmark = pytest.mark.gpu
SPEC = gt.EdgeSpec("src", "dst")


def build(src, dst):
    return gt.table_to_graph(gt.edge_table(np.asarray(src, np.int64),
                                           np.asarray(dst, np.int64)), SPEC)


@pytest.mark.parametrize("name", sorted(golden_cases()))
def test_edge_table_round_trip(name):
    case = golden_cases()[name]
    g = build(case["src"], case["dst"])
    t = gt.graph_to_edge_table(g)
    pairs = np.unique(np.stack([case["src"], case["dst"]], axis=1), axis=0)
    assert np.array_equal(t.column("src"), pairs[:, 0].astype(np.int64))
    assert np.array_equal(t.column("dst"), pairs[:, 1].astype(np.int64))
    assert t.schema.names == ["src", "dst"]


def test_edge_table_on_device_and_rebuild():
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(14, 200000, seed=3, permute=True)
    g = build(src, dst)
    t = gt.graph_to_edge_table(g, device=True)
    assert t.column("src").is_cuda
    g2 = gt.table_to_graph(t, SPEC)  # export -> ToGraph is the identity on the CSR
    a, b = g.csr(), g2.csr()
    for f in ("ids", "out_off", "out_adj", "in_off", "in_adj"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_node_table_and_scores():
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(11, 20000, seed=4)
    g = build(src, dst)
    want = ref.build_csr(src, dst)
    pr = gt.pagerank(g, 0.85, 10)
    t = gt.graph_to_node_table(g, pr, value_name="rank")
    assert np.array_equal(t.column("node"), want.ids)
    assert np.array_equal(t.column("out_deg"), np.diff(want.out_off))
    assert np.array_equal(t.column("in_deg"), np.diff(want.in_off))
    assert np.array_equal(t.column("rank"), np.asarray(pr.scores))
    assert gt.graph_to_node_table(g, pr.to_dict()).column("value").shape[0] == want.n
    with pytest.raises(CoverageError):
        gt.graph_to_node_table(g, {int(want.ids[0]): 1.0})


def test_table_from_map_and_frontend(tmp_path):
    from paper_1503_07881_b200 import graphdesk as gd

    src = np.array([1, 2, 3, 3, 9], dtype=np.int64)
    dst = np.array([2, 3, 1, 9, 1], dtype=np.int64)
    t = gd.TableHandle(gt.edge_table(src, dst))
    G = gd.ToGraph(t, "src", "dst")
    pr = gd.GetPageRank(G, 0.85, 10)
    tab = gd.TableFromHashMap(pr, "node", "score")
    assert tab.column_names == ["node", "score"]
    rows = tab.rows()
    assert [r[0] for r in rows] == [1, 2, 3, 9]
    assert abs(sum(r[1] for r in rows) - 1.0) < 1e-12
    same = gt.table_from_map(dict(pr.items()), "node", "score")
    assert same.to_rows() == rows
    e = gd.GraphToTable(G)
    assert e.rows() == sorted(set(zip(src.tolist(), dst.tolist())))
    gd.SaveTableTSV(tab, tmp_path / "scores.tsv")
    assert (tmp_path / "scores.tsv").read_text().count("\n") == 4
