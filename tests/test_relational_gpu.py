"""Device Select / Join feeding ToGraph on the B200.

Parity against the real reference's outputs (tests/golden/relational.npz:
select row ids for 29 predicates x 7 tables, join pairs in output order for
13 table pairs on int / str / float keys, the demo chain of demo.py:37-47),
the reference's own TestSelect / TestJoin cases (test_tables.py:116-231),
and the oracle restatement on larger seeded tables. All exact (integer row
indices); the demo's PageRank within 1e-9 L1."""

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import REL_SCHEMA, golden_relational, join_keys_py, pair_digest
from oracle import reference_port as ref
from paper_1503_07881_b200 import graphdesk

pytestmark = pytest.mark.gpu
G = golden_relational()
SCHEMA = gt.Schema(list(REL_SCHEMA))


def golden_table(t, index_col=None):
    cols, pool = G["tables"][t]
    names = [n for n, _ in REL_SCHEMA]
    arrays = [cols[n] for n in names]
    schema = SCHEMA
    if index_col:
        schema = gt.Schema(list(REL_SCHEMA) + [(index_col, "int")])
        arrays.append(np.arange(arrays[0].shape[0], dtype=np.int64))
    return gt.ColumnTable(schema, arrays, pool=list(pool))


def host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def make(schema_cols, rows):
    return gt.ColumnTable.from_rows(gt.Schema(schema_cols), rows)


# ------------------------------------------------------------------ select --

@pytest.mark.parametrize("t", range(len(G["tables"])))
def test_select_matches_reference(t):
    table = golden_table(t)
    rows = table.to_rows()
    for i, (c, op, v) in enumerate(G["preds"]):
        got = gt.select(table, gt.Predicate(c, op, v))
        want = G["sel"][(t, i)]
        np.testing.assert_array_equal(host(got.row_ids), want, err_msg=f"{c}{op}{v!r}")
        assert got.n_rows == want.shape[0]
        got_rows = got.to_rows()
        want_rows = [rows[r] for r in want.tolist()]
        # NaN cells compare unequal to themselves: compare their repr
        assert [tuple(map(repr, r)) for r in got_rows] == [tuple(map(repr, r)) for r in want_rows]


def test_select_result_is_device_resident_and_feeds_to_graph():
    rng = np.random.default_rng(5)
    n = 2_000_000
    src = rng.integers(0, 50_000, n, dtype=np.int64)
    dst = rng.integers(0, 50_000, n, dtype=np.int64)
    w = rng.integers(0, 10, n, dtype=np.int64)
    t = gt.ColumnTable(gt.Schema([("src", "int"), ("dst", "int"), ("w", "int")]),
                       [src, dst, w]).to_device()
    sel = gt.select(t, gt.Predicate("w", "<", 3))
    assert sel.is_device_resident("src") and sel.is_device_resident("dst")
    keep = ref.select_indices(w, "int", [], "<", 3)
    np.testing.assert_array_equal(host(sel.row_ids), keep)
    g = gt.table_to_graph(sel, gt.EdgeSpec("src", "dst"))
    want = ref.build_csr(src[keep], dst[keep])
    got_ids = host(g.node_ids())
    np.testing.assert_array_equal(got_ids, want.ids)
    assert g.edge_count == int(want.out_off[-1])


def test_select_reference_cases():
    # test_tables.py:116-169
    t = make([("age", "int")], [(1,), (5,), (9,)])
    got = gt.select(t, gt.Predicate("age", ">", 4))
    assert got.to_rows() == [(5,), (9,)]
    assert host(got.row_ids).tolist() == [1, 2]
    assert gt.select(t, gt.Predicate("age", ">", 100)).n_rows == 0
    t = make([("age", "int")], [(1,), (5,), (9,)])
    got = gt.select(t, gt.Predicate("age", ">=", 1), in_place=True)
    assert got is t and t.n_rows == 3 and host(t.row_ids).tolist() == [0, 1, 2]
    gt.select(t, gt.Predicate("age", ">", 1), in_place=True)
    gt.select(t, gt.Predicate("age", "<", 9), in_place=True)
    assert host(t.row_ids).tolist() == [1] and t.to_rows() == [(5,)]
    w = make([("w", "str")], [("zebra",), ("apple",)])
    assert gt.select(w, gt.Predicate("w", "<", "mango")).to_rows() == [("apple",)]


def test_select_idempotent():
    t = golden_table(5)
    p = gt.Predicate("k", "<=", 3)
    once = gt.select(t, p)
    twice = gt.select(once, p)
    assert once.cell_equal(twice) or [tuple(map(repr, r)) for r in once.to_rows()] == \
        [tuple(map(repr, r)) for r in twice.to_rows()]
    np.testing.assert_array_equal(host(once.row_ids), host(twice.row_ids))


def test_select_empty_table():
    t = gt.ColumnTable(SCHEMA, [np.empty(0, np.int64), np.empty(0), np.empty(0, np.int64),
                                np.empty(0, np.int64)])
    assert gt.select(t, gt.Predicate("k", "=", 1)).n_rows == 0
    assert gt.select(t, gt.Predicate("s", "<", "m")).n_rows == 0


# -------------------------------------------------------------------- join --

@pytest.mark.parametrize("j", range(len(G["joins"])))
def test_join_matches_reference(j):
    rec = G["joins"][j]
    left = golden_table(rec["left"], "li")
    right = golden_table(rec["right"], "ri")
    got = gt.join(left, right, rec["key"], rec["key"])
    assert got.schema.names == rec["names"]
    assert got.n_rows == rec["n"]
    li, ri = host(got.column("li")), host(got.column("ri"))
    if "li" in rec:
        np.testing.assert_array_equal(li, rec["li"])
        np.testing.assert_array_equal(ri, rec["ri"])
    else:
        assert pair_digest(li, ri) == rec["sha"]
    assert host(got.row_ids).tolist() == list(range(rec["n"]))
    if 0 < rec["n"] <= 5000:  # every cell: left row li then right row ri, decoded
        lrows, rrows = left.to_rows(), right.to_rows()
        want = [lrows[a] + rrows[b] for a, b in zip(li.tolist(), ri.tolist())]
        assert [tuple(map(repr, r)) for r in got.to_rows()] == \
            [tuple(map(repr, r)) for r in want]


def test_join_reference_cases():
    from collections import Counter

    # test_tables.py:181-222
    left = make([("k", "int")], [(1,), (2,), (2,)])
    right = make([("k", "int")], [(2,), (2,), (3,)])
    got = gt.join(left, right, "k", "k")
    assert got.n_rows == 4
    assert Counter(got.to_rows()) == Counter([(2, 2)] * 4)
    assert gt.join(make([("k", "int")], [(1,)]), make([("k", "int")], [(2,)]),
                   "k", "k").n_rows == 0
    t = make([("k", "int"), ("v", "str")], [(1, "a"), (2, "b"), (3, "c")])
    assert gt.join(t, t, "k", "k").n_rows == 3
    got = gt.join(make([("k", "int"), ("u", "int")], [(1, 10)]),
                  make([("k", "int"), ("w", "int")], [(1, 20)]), "k", "k")
    assert got.schema.names == ["k-1", "u", "k-2", "w"]
    left = make([("k", "int")], [(7,), (7,)])
    assert host(gt.join(left, left, "k", "k").row_ids).tolist() == [0, 1, 2, 3]
    left = make([("t", "str")], [("b",), ("a",)])
    right = make([("t", "str"), ("v", "int")], [("a", 1), ("c", 2)])
    assert gt.join(left, right, "t", "t").to_rows() == [("a", "a", 1)]


@pytest.mark.parametrize("nl,nr,hi", [(1_000_000, 3_000_000, 2_000_000), (3_000_000, 900_000, 50),
                                       (500_000, 500_000, 1 << 40)])
def test_join_large_vs_oracle(nl, nr, hi):
    rng = np.random.default_rng(nl ^ nr)
    lk = rng.integers(-hi, hi, nl, dtype=np.int64)
    rk = rng.integers(-hi, hi, nr, dtype=np.int64)
    if hi == 50:  # heavy multiplicities: cap the probe side to bound the output
        rk = rk[:2000]
    schema_l, schema_r = gt.Schema([("k", "int")]), gt.Schema([("k", "int")])
    got = gt.join(gt.ColumnTable(schema_l, [lk]).to_device(),
                  gt.ColumnTable(schema_r, [rk]).to_device(), "k", "k")
    li, ri = ref.join_indices(lk.tolist(), rk.tolist())
    assert got.n_rows == li.shape[0]
    np.testing.assert_array_equal(host(got.column("k-1")), lk[li])
    np.testing.assert_array_equal(host(got.column("k-2")), rk[ri])


# --------------------------------------------------------------- demo chain --

def test_demo_chain_matches_reference():
    """demo.py:37-47 through the front-end: Select x3 -> Join -> ToGraph ->
    GetPageRank on the reference's own qa-forum posts table."""
    qa = G["qa"]
    schema = gt.Schema([("PostId", "int"), ("Type", "str"), ("Tag", "str"), ("UserId", "int"),
                        ("AnswerId", "int")])
    posts = graphdesk.TableHandle(gt.ColumnTable(
        schema, [qa[n] for n in schema.names], pool=qa["pool"].tolist()))
    tagged = graphdesk.Select(posts, "Tag=Java")
    questions = graphdesk.Select(tagged, "Type=question")
    answers = graphdesk.Select(tagged, "Type=answer")
    joined = graphdesk.Join(questions, answers, "AnswerId", "PostId")
    np.testing.assert_array_equal(host(joined._table.column("UserId-1")), qa["u1"])
    np.testing.assert_array_equal(host(joined._table.column("UserId-2")), qa["u2"])
    graph = graphdesk.ToGraph(joined, "UserId-1", "UserId-2")
    ranks = graphdesk.GetPageRank(graph)
    got = np.array([ranks[int(i)] for i in qa["pr_ids"].tolist()])
    assert len(ranks) == qa["pr_ids"].shape[0]
    assert np.abs(got - qa["pr"]).sum() <= 1e-9
    with pytest.raises(graphdesk.FrontendError):
        graphdesk.Select(posts, "NoSuchColumn=1")


# ------------------------------------------------------------ property-based --

from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

_ROWS = st.lists(st.tuples(st.integers(-5, 5), st.sampled_from([0.0, -0.0, 1.5, float("nan")]),
                           st.sampled_from(["a", "b", "", "zz"]), st.integers(-(2 ** 63), 2 ** 63 - 1)),
                 max_size=60)


@settings(max_examples=40, deadline=None)
@given(_ROWS, _ROWS, st.sampled_from(["k", "x", "s", "v"]))
def test_join_property_vs_oracle(lrows, rrows, key):
    """Random tables (duplicates, +-0.0, NaN, int64 extremes, shared and
    disjoint string pools): the device join equals the oracle's hash join
    row for row, in order (tables.py:397-426)."""
    left = make(list(SCHEMA.columns), lrows)
    right = make(list(SCHEMA.columns), rrows)
    got = gt.join(left, right, key, key)
    i = "kxsv".index(key)

    def keys(rows):  # as the reference hashes them: decoded, then .tolist() (fresh NaNs)
        vals = [r[i] for r in rows]
        return np.asarray(vals, dtype=np.float64).tolist() if key == "x" else vals

    li, ri = ref.join_indices(keys(lrows), keys(rrows))
    want = [lrows[a] + rrows[b] for a, b in zip(li.tolist(), ri.tolist())]
    assert [tuple(map(repr, r)) for r in got.to_rows()] == [tuple(map(repr, r)) for r in want]


@settings(max_examples=40, deadline=None)
@given(_ROWS, st.sampled_from(["=", "!=", "<", "<=", ">", ">="]),
       st.one_of(st.integers(-7, 7), st.floats(allow_nan=True, allow_infinity=True),
                 st.integers(-(2 ** 70), 2 ** 70)))
def test_select_int_property_vs_oracle(rows, op, value):
    """INT column against ints, floats (non-integral, inf, NaN) and
    beyond-int64 constants: numpy's comparison result (tables.py:343)."""
    t = make(list(SCHEMA.columns), rows)
    got = gt.select(t, gt.Predicate("v", op, value))
    col = np.asarray([r[3] for r in rows], dtype=np.int64)
    want = ref.select_indices(col, "int", [], op, value)
    np.testing.assert_array_equal(host(got.row_ids), want)
