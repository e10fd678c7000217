"""Pin the CPU oracle against outputs of the real reference (CPU only).

The fixtures were recorded by tests/golden/make_golden.py running the
unmodified reference ``graphtables`` in the build container; here the
restatement (oracle/reference_port.py, oracle/fast_oracle.c) must reproduce
them exactly (CSR, triangles) and to 1e-12 (PageRank: same algorithm, same
summation order).
"""

import numpy as np
import pytest

from helpers import assert_csr_equal, golden_c1, golden_cases, sha
from oracle import reference_port as ref
from paper_1503_07881_b200.synth import rmat_edges

CASES = sorted(golden_cases())


@pytest.mark.parametrize("name", CASES)
def test_oracle_build_matches_reference(name):
    case = golden_cases()[name]
    got = ref.build_csr(case["src"], case["dst"], workers=4)
    assert_csr_equal(got, case, name)


@pytest.mark.parametrize("name", CASES)
def test_oracle_pagerank_matches_reference(name):
    case = golden_cases()[name]
    if case["ids"].shape[0] == 0:
        pytest.skip("empty graph")
    g = ref.build_csr(case["src"], case["dst"], workers=2)
    pr = ref.pagerank_csr(g, 0.85, 10, workers=3)
    assert np.max(np.abs(pr - case["pr"])) <= 1e-12


@pytest.mark.parametrize("name", CASES)
def test_fast_triangle_oracle_matches_reference(name):
    case = golden_cases()[name]
    g = ref.build_csr(case["src"], case["dst"], workers=1)
    assert ref.triangle_count_fast(g, threads=2) == int(case["tc"][0])


@pytest.mark.parametrize("name", [n for n in CASES if golden_cases()[n]["ids"].shape[0] <= 2000])
def test_numpy_triangle_oracle_matches_reference(name):
    case = golden_cases()[name]
    g = ref.build_csr(case["src"], case["dst"], workers=1)
    assert ref.triangle_count_csr(g, workers=2) == int(case["tc"][0])


def test_c1_config_matches_reference():
    """BASELINE config 0 (R-MAT s17, 1,048,576 rows, seed 1) end to end."""
    gold = golden_c1()
    src, dst = rmat_edges(17, 1_048_576, seed=1, permute=False)
    assert sha(src) == str(gold["sha_src"]) and sha(dst) == str(gold["sha_dst"])
    g = ref.build_csr(src, dst)
    for f in ("ids", "out_off", "out_adj", "in_off", "in_adj"):
        assert sha(getattr(g, f)) == str(gold[f"sha_{f}"]), f
    pr = ref.pagerank_csr(g, 0.85, 10)
    assert np.max(np.abs(pr - gold["pr"])) <= 1e-12
    assert ref.triangle_count_fast(g) == int(gold["tc"][0])


def test_parallel_sort_equals_np_sort():
    rng = np.random.default_rng(0)
    v = rng.integers(0, 1 << 40, size=300_000).astype(np.uint64)
    for w in (1, 3, 8):
        assert np.array_equal(ref.parallel_sort(v, w), np.sort(v))


# ---- sssp / connected_components / k_core --------------

TRAVERSE = sorted(__import__("helpers").golden_traverse())


def _traverse_csr(case):
    g = ref.build_csr(case["src"], case["dst"], workers=1)
    return ref.add_isolated(g, case["extra"]) if case["extra"].size else g


@pytest.mark.parametrize("name", TRAVERSE)
def test_oracle_traversals_match_reference(name):
    from helpers import golden_traverse

    case = golden_traverse()[name]
    g = _traverse_csr(case)
    assert np.array_equal(g.ids, case["ids"])
    und = ref.undirected_dense(g)
    for row, s in zip(case["sssp"], case["sources"].tolist()):
        assert np.array_equal(ref.sssp_csr(g, int(np.searchsorted(g.ids, s))), row)
    assert np.array_equal(ref.components_csr(g, und), case["cc"])
    for k in (1, 2, 3, 4):
        core = ref.k_core_csr(g, k, und)
        assert np.array_equal(core.ids, case[f"kcore{k}_ids"])
        assert np.array_equal(core.out_off, case[f"kcore{k}_out_off"])
        assert np.array_equal(core.out_adj, case[f"kcore{k}_out_adj"])


def test_oracle_k_core_rejects_k0():
    g = ref.build_csr([0], [1])
    with pytest.raises(ValueError):
        ref.k_core_csr(g, 0)


# ---- scc ---------------------------------------------

SCC_CASES = sorted(__import__("helpers").golden_scc())


@pytest.mark.parametrize("name", SCC_CASES)
def test_oracle_scc_matches_reference(name):
    from helpers import golden_scc

    case = golden_scc()[name]
    g = _traverse_csr(case)
    assert np.array_equal(g.ids, case["ids"])
    assert np.array_equal(ref.scc_csr(g), case["scc"])


# ---- batched dynamic updates ---------------------------

UPDATE_CASES = sorted(__import__("helpers").golden_updates())


@pytest.mark.parametrize("name", UPDATE_CASES)
def test_oracle_updates_match_reference(name):
    from helpers import golden_updates

    c = golden_updates()[name]
    g = ref.build_csr(c["src"], c["dst"], workers=1)
    got = ref.update_csr(g, add=(c["add_src"], c["add_dst"]), delete=(c["del_src"], c["del_dst"]),
                         add_nodes=c["add_nodes"], del_nodes=c["del_nodes"])
    for f in ("ids", "out_off", "out_adj", "in_off", "in_adj"):
        assert np.array_equal(getattr(got, f), c[f]), f


def _dense32(case):
    ids = case["ids"]
    return (np.searchsorted(ids, case["out_adj"]).astype(np.int32),
            np.searchsorted(ids, case["in_adj"]).astype(np.int32))


@pytest.mark.parametrize("name", CASES)
def test_large_size_checkers_match_reference(name):
    """The int32 checkers used at BASELINE configs[3]/[4] (triangle slices by
    middle-vertex rank, pull PageRank) reproduce the reference's outputs."""
    case = golden_cases()[name]
    n = case["ids"].shape[0]
    if n == 0:
        pytest.skip("empty graph")
    oa, ia = _dense32(case)
    for nparts in (1, 5):
        parts = sum(ref.triangles_slice_dense32(n, case["out_off"], oa, case["in_off"], ia, p,
                                                nparts, threads=2) for p in range(nparts))
        assert parts == int(case["tc"][0])
    pr = ref.pagerank_dense32(n, case["in_off"], ia, case["out_off"], 0.85, 10, threads=2)
    assert np.max(np.abs(pr - case["pr"])) <= 1e-12
