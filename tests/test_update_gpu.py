"""Batched dynamic updates on the device (csrc/update.cu):
DeviceGraph.apply_updates against the real reference's Graph mutation calls
(graphs.py:92-144, tests/golden/updates.npz) and the oracle's restatement at
larger sizes. CSR arrays bit-exact."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import golden_updates
from oracle import reference_port as ref
from paper_1503_07881_b200.synth import rmat_edges

pytestmark = pytest.mark.gpu
SPEC = gt.EdgeSpec("src", "dst")
FIELDS = ("ids", "out_off", "out_adj", "in_off", "in_adj")


def assert_same(dg, want):
    h = dg.csr()
    for f in FIELDS:
        assert np.array_equal(getattr(h, f), want[f] if isinstance(want, dict) else
                              getattr(want, f)), f


@pytest.mark.parametrize("name", sorted(golden_updates()))
def test_updates_match_reference(name):
    c = golden_updates()[name]
    g = gt.table_to_graph(gt.edge_table(c["src"], c["dst"]), SPEC)
    g.apply_updates(add=(c["add_src"], c["add_dst"]), delete=(c["del_src"], c["del_dst"]),
                    add_nodes=c["add_nodes"], del_nodes=c["del_nodes"])
    assert g.on_device
    assert_same(g, c)
    g.check_invariants()
    assert g.edge_count == c["out_adj"].shape[0]


def test_updates_rmat_vs_oracle_device_inputs():
    import torch

    src, dst = rmat_edges(17, 1_000_000, seed=9, permute=True)
    g = gt.table_to_graph(gt.edge_table(src, dst), SPEC)
    rng = np.random.default_rng(9)
    pick = rng.integers(0, src.size, 50_000)
    dels = (src[pick], dst[pick])
    adds = (rng.integers(0, 1 << 18, 100_000), rng.integers(0, 1 << 18, 100_000))
    dn = rng.choice(np.unique(src), 500)
    an = rng.integers(1 << 18, 1 << 19, 50)
    dev = torch.device("cuda")
    g.apply_updates(add=tuple(torch.from_numpy(a).to(dev) for a in adds),
                    delete=dels, add_nodes=an, del_nodes=torch.from_numpy(dn).to(dev))
    want = ref.update_csr(ref.build_csr(src, dst), add=adds, delete=dels, add_nodes=an,
                          del_nodes=dn)
    assert_same(g, want)
    # results feed the other consumers directly
    assert gt.triangle_count(g) == ref.triangle_count_fast(want)


def test_updates_edge_cases():
    g = gt.table_to_graph(gt.edge_table(np.array([1, 2]), np.array([2, 3])), SPEC)
    g.apply_updates()  # empty batch: unchanged
    assert g.node_ids() == [1, 2, 3] and g.edge_count == 2
    g.apply_updates(delete=(np.array([1]), np.array([2])))  # nodes stay (del_edge)
    assert g.node_ids() == [1, 2, 3] and g.edge_count == 1
    g.apply_updates(del_nodes=np.array([1, 2, 3]))
    assert g.node_count == 0 and g.edge_count == 0
    g.apply_updates(add=(np.array([5, 5]), np.array([5, 6])), add_nodes=np.array([9]))
    assert g.node_ids() == [5, 6, 9] and g.edge_count == 2
    with pytest.raises(ValueError):
        g.apply_updates(add=(np.array([1, 2]), np.array([1])))
    # a graph already mutated on the host keeps the reference's per-call semantics
    g.add_edge(6, 5)
    g.apply_updates(add=(np.array([9]), np.array([5])), del_nodes=np.array([6]))
    assert sorted(g.node_ids()) == [5, 9] and g.edge_count == 2
