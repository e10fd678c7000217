"""The select / join restatement in oracle/reference_port.py against the
outputs of the real reference (tests/golden/relational.npz, recorded by
tests/golden/make_golden_relational.py): select row ids for every predicate
on every table, join pairs in output order (tables.py:325-344, 397-426)."""

import numpy as np
import pytest

from helpers import golden_relational, join_keys_py, pair_digest
from oracle import reference_port as ref

G = golden_relational()
TYPES = dict((("k", "int"), ("x", "float"), ("s", "str"), ("v", "int")))


@pytest.mark.parametrize("t", range(len(G["tables"])))
def test_select_oracle_matches_reference(t):
    cols, pool = G["tables"][t]
    for i, (c, op, v) in enumerate(G["preds"]):
        got = ref.select_indices(cols[c], TYPES[c], pool, op, v)
        np.testing.assert_array_equal(got, G["sel"][(t, i)], err_msg=f"table {t} pred {c}{op}{v!r}")


@pytest.mark.parametrize("j", range(len(G["joins"])))
def test_join_oracle_matches_reference(j):
    rec = G["joins"][j]
    lcols, lpool = G["tables"][rec["left"]]
    rcols, rpool = G["tables"][rec["right"]]
    li, ri = ref.join_indices(join_keys_py(lcols, lpool, rec["key"]),
                              join_keys_py(rcols, rpool, rec["key"]))
    assert li.shape[0] == rec["n"]
    if "li" in rec:
        np.testing.assert_array_equal(li, rec["li"])
        np.testing.assert_array_equal(ri, rec["ri"])
    else:
        assert pair_digest(li, ri) == rec["sha"]


def test_predicate_parse_and_errors_host_only():
    import paper_1503_07881_b200 as gt

    schema = gt.Schema([("age", "int"), ("w", "float"), ("tag", "str")])
    assert gt.Predicate.parse("age>=30", schema) == gt.Predicate("age", ">=", 30)
    assert gt.Predicate.parse(" w < 2.5", schema) == gt.Predicate("w", "<", 2.5)
    assert gt.Predicate.parse("tag=Java", schema) == gt.Predicate("tag", "=", "Java")
    assert gt.Predicate.parse("tag!=a=b", schema) == gt.Predicate("tag", "!=", "a=b")
    with pytest.raises(ValueError):
        gt.Predicate("age", "~", 1)
    with pytest.raises(ValueError):
        gt.Predicate.parse("age 30", schema)
    with pytest.raises(gt.UnknownColumnError):
        gt.Predicate.parse("nope=1", schema)
    t = gt.ColumnTable(schema, [np.array([1]), np.array([1.0]), np.array([0])], pool=["x"])
    with pytest.raises(gt.TypeMismatchError):
        gt.select(t, gt.Predicate("age", "=", "old"))
    with pytest.raises(gt.TypeMismatchError):
        gt.select(t, gt.Predicate("tag", "=", 3))
    with pytest.raises(gt.UnknownColumnError):
        gt.select(t, gt.Predicate("weight", ">", 4))
    right = gt.ColumnTable(gt.Schema([("age", "str")]), [np.array([0])], pool=["1"])
    with pytest.raises(gt.TypeMismatchError):
        gt.join(t, right, "age", "age")
    with pytest.raises(gt.SchemaError):
        gt.project(t, [])
    p = gt.project(t, ["tag", "age"])
    assert p.schema.names == ["tag", "age"] and p.to_rows() == [("x", 1)]


def test_fresh_row_ids_and_pool_helpers():
    import paper_1503_07881_b200 as gt

    t = gt.ColumnTable.from_rows(gt.Schema([("w", "str"), ("n", "int")]),
                                 [("zebra", 1), ("apple", 2), ("zebra", 3)])
    assert t.pool == ["zebra", "apple"]
    assert t.row_ids.tolist() == [0, 1, 2]
    assert t.encode_value("apple") == 1 and t.encode_value("kiwi") is None
    assert t.decoded("w").tolist() == ["zebra", "apple", "zebra"]
    assert t.cell_equal(gt.ColumnTable.from_rows(t.schema, t.to_rows()))
