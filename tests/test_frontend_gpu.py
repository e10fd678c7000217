"""graphdesk mirror through the device engine (frontend test_frontend.py:63-89,
117-125 shapes) plus the new GetTriangles."""

import gc
import weakref

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from paper_1503_07881_b200 import graphdesk
from paper_1503_07881_b200.synth import rmat_edges

pytestmark = pytest.mark.gpu


def test_to_graph_on_edge_fixture(tmp_path):
    path = tmp_path / "edges.tsv"
    path.write_text("1\t2\n2\t3\n")
    t = graphdesk.LoadTableTSV("src:int,dst:int", str(path))
    g = graphdesk.ToGraph(t, "src", "dst")
    assert g.edge_count == 2 and g.node_count == 3


def test_chain_matches_engine(tmp_path):
    src, dst = rmat_edges(11, 20_000, seed=4, permute=True)
    path = tmp_path / "e.tsv"
    path.write_text("".join(f"{a}\t{b}\n" for a, b in zip(src.tolist(), dst.tolist())))
    ws = graphdesk.Workspace()
    t = ws.LoadTableTSV("src:int,dst:int", str(path))
    g = ws.ToGraph(t.to_device(), "src", "dst")
    pr = ws.GetPageRank(g)
    tri = ws.GetTriangles(g)
    eg = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
    assert dict(pr.items()) == gt.pagerank(eg, damping=0.85, iterations=10).to_dict()
    assert tri == gt.triangle_count(eg)
    top = pr.top(3)
    assert top == sorted(pr.items(), key=lambda kv: (-kv[1], kv[0]))[:3]


def test_errors_are_wrapped():
    t = graphdesk.TableHandle(gt.edge_table(np.array([0]), np.array([1])))
    g = graphdesk.ToGraph(t, "src", "dst")
    with pytest.raises(graphdesk.FrontendError) as err:
        graphdesk.GetPageRank(g, damping=2.0)
    assert isinstance(err.value.engine_error, ValueError)


def test_dropping_last_handle_releases_device_graph():
    t = graphdesk.TableHandle(gt.edge_table(np.array([0, 1]), np.array([1, 2])))
    h = graphdesk.ToGraph(t, "src", "dst")
    ref = weakref.ref(h._graph)
    fin = h._graph._finalizer
    del h
    gc.collect()
    assert ref() is None and not fin.alive
