"""Host-side contract of the drop-in (CPU): validation, errors, handles,
host Graph semantics, and that the compute path has no CPU fallback."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from paper_1503_07881_b200 import graphdesk
from paper_1503_07881_b200.algorithms import RankMap


def edges(pairs):
    a = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    return gt.edge_table(a[:, 0], a[:, 1])


def test_edge_spec_rejects_non_int_and_unknown_columns():
    t = gt.ColumnTable(gt.Schema([("src", "float"), ("dst", "int")]),
                       [np.array([1.0]), np.array([2])])
    with pytest.raises(gt.TypeMismatchError):
        gt.table_to_graph(t, gt.EdgeSpec("src", "dst"))
    with pytest.raises(gt.UnknownColumnError):
        gt.table_to_graph(edges([(1, 2)]), gt.EdgeSpec("src", "nope"))
    s = gt.ColumnTable(gt.Schema([("src", "str"), ("dst", "int")]), [np.array([0]), np.array([1])])
    with pytest.raises(gt.TypeMismatchError):  # string codes are not ids (convert.py:37-42)
        gt.table_to_graph(s, gt.EdgeSpec("src", "dst"))


def test_worker_validation():
    with pytest.raises(ValueError):
        gt.table_to_graph(edges([(1, 2)]), gt.EdgeSpec("src", "dst"), workers=0)


def test_pagerank_parameter_validation_before_device():
    g = gt.from_edges([(0, 1)])
    with pytest.raises(ValueError):
        gt.pagerank(g, damping=1.0)
    with pytest.raises(ValueError):
        gt.pagerank(g, damping=0.0)
    with pytest.raises(ValueError):
        gt.pagerank(g, iterations=0)
    with pytest.raises(ValueError):
        gt.pagerank(gt.Graph())


def test_triangles_on_empty_graph_is_zero():
    assert gt.triangle_count(gt.Graph()) == 0


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gt.NativeError):
        gt.table_to_graph(edges([(1, 2)]), gt.EdgeSpec("src", "dst"))
    with pytest.raises(gt.NativeError):
        gt.triangle_count(gt.from_edges([(0, 1), (1, 2), (2, 0)]))


def test_frontend_wraps_engine_errors(tmp_path):
    with pytest.raises(graphdesk.FrontendError) as err:
        graphdesk.LoadTableTSV("src:int,dst:int", "/no/such/file.tsv")
    assert "file.tsv" in str(err.value)
    bad = tmp_path / "bad.tsv"
    bad.write_text("1\t2\nx\t3\n")
    with pytest.raises(graphdesk.FrontendError) as err:
        graphdesk.LoadTableTSV("src:int,dst:int", str(bad))
    assert isinstance(err.value.engine_error, gt.ParseError)
    assert err.value.engine_error.line == 2 and err.value.engine_error.column == "src"
    ok = tmp_path / "ok.tsv"
    ok.write_text("1\t2\n2\t3\n")
    t = graphdesk.LoadTableTSV("src:int,dst:int", str(ok))
    assert t.row_count == 2 and t.column_names == ["src", "dst"]
    with pytest.raises(graphdesk.FrontendError) as err:
        graphdesk.ToGraph(t, "src", "missing")
    assert isinstance(err.value.engine_error, gt.UnknownColumnError)


def test_frontend_aliases():
    assert graphdesk.get_triangles is graphdesk.GetTriangles
    assert graphdesk.Workspace.to_graph is graphdesk.Workspace.ToGraph
    assert graphdesk.load_table_tsv is graphdesk.LoadTableTSV


def test_rank_handle_top_breaks_ties_by_id():
    r = graphdesk.RankHandle(RankMap(np.array([1, 2, 3]), np.array([0.5, 0.25, 0.5])))
    assert r.top(2) == [(1, 0.5), (3, 0.5)]
    assert len(r) == 3 and r[2] == 0.25 and list(r) == [1, 2, 3]


def test_rank_map_is_a_mapping():
    r = RankMap(np.array([-4, 7, 9]), np.array([0.2, 0.3, 0.5]))
    assert r[7] == 0.3 and 9 in r and 8 not in r
    with pytest.raises(KeyError):
        r[8]
    assert dict(r.items()) == {-4: 0.2, 7: 0.3, 9: 0.5}
    assert r == {-4: 0.2, 7: 0.3, 9: 0.5}
    assert abs(sum(r.values()) - 1.0) < 1e-12


def test_host_graph_replay_and_mutation():
    g = gt.from_edges([(1, 2), (2, 3), (1, 2), (3, 3)])
    assert g.node_count == 3 and g.edge_count == 3
    assert g.neighbors(1, "out").tolist() == [2]
    with pytest.raises(ValueError):
        g.neighbors(1, "out")[0] = 9
    assert g.add_edge(3, 1) and not g.add_edge(3, 1)
    assert g.del_edge(1, 2) and not g.del_edge(1, 2)
    g.check_invariants()
    assert g.undirected_neighbors(3).tolist() == [1, 2]
    assert g.del_node(3) and g.edge_count == 0
    g.check_invariants()
    with pytest.raises(gt.UnknownNodeError):
        g.record(99)


def test_host_graph_equality():
    a = gt.from_edges([(1, 2), (2, 3)])
    b = gt.from_edges([(2, 3), (1, 2)])
    c = gt.from_edges([(1, 2), (3, 2)])
    assert a == b and not (a == c)


def test_schema_and_tables():
    s = gt.Schema.parse("a:int, b:float,c:str")
    assert s.names == ["a", "b", "c"] and s.type_of("b") == "float"
    with pytest.raises(gt.SchemaError):
        gt.Schema([("a", "int"), ("a", "int")])
    with pytest.raises(gt.SchemaError):
        gt.ColumnTable(gt.Schema([("a", "int"), ("b", "int")]), [np.arange(3), np.arange(4)])
