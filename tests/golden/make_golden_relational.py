"""Golden fixtures for Select / Join from the REAL reference.

Runs the unmodified reference ``graphtables`` (``/root/reference/pkg/src``,
build container only) and records into ``relational.npz``:

* ``tab{t}_*``   — seeded mixed-type tables (int / float / str columns,
  duplicate keys, -1, INT64_MIN, +-0.0, NaN, repeated strings): columns,
  string pool.
* ``sel{t}_{i}`` — for every predicate in ``SELECT_PREDICATES``: the
  reference ``select``'s surviving row ids (its output keeps the ids,
  tables.py:232-240, so ids + the input table pin the result).
* ``join{j}_*``  — reference ``join`` (tables.py:397-426) of table pairs on
  int / str / float keys: the (left row, right row) of every output row in
  output order (recovered from an index column appended to each input;
  outputs above 100,000 pairs as a sha256 of the two lists), and the output
  schema names.
* ``qa_*``       — the demo chain of the reference front-end
  (demo.py:37-47): the qa-forum posts table from the reference's own
  generator (synth.qa_forum, 4000 questions / 6000 answers, seed 2718), the
  joined (UserId-1, UserId-2) columns and the PageRank (10 iterations) of
  the resulting graph, ids ascending.

Usage: PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_relational.py
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import graphtables as ref  # noqa: E402  (the reference)
from graphtables.synth import qa_forum  # noqa: E402

I64_MIN = -(1 << 63)
WORDS = ["apple", "zebra", "mango", "Java", "python", "", "a b", "Zed", "apple2", "kiwi"]

# (column, op, value); values chosen to hit every comparison path
SELECT_PREDICATES = [
    ("k", "=", 3), ("k", "!=", 3), ("k", "<", 0), ("k", "<=", -1), ("k", ">", 5),
    ("k", ">=", I64_MIN), ("k", ">", 2.5), ("k", "<", 2.5), ("k", "=", 2.5),
    ("k", "!=", 2.5), ("k", "<=", 4.0), ("k", "<", float("inf")), ("k", ">", float("nan")),
    ("k", "!=", float("nan")), ("k", "<", 2 ** 70), ("k", ">", -(2 ** 70)),
    ("x", "<", 0.0), ("x", "=", 0.0), ("x", "!=", 0.0), ("x", ">=", -1.5), ("x", ">", 2),
    ("s", "=", "apple"), ("s", "!=", "apple"), ("s", "=", "missing"), ("s", "!=", "missing"),
    ("s", "<", "mango"), ("s", ">=", "Zed"), ("s", ">", ""), ("s", "<=", "apple"),
]


def random_table(rng, n):
    k = rng.integers(-3, 9, size=n).astype(np.int64)
    if n:
        k[rng.random(n) < 0.05] = I64_MIN
        k[rng.random(n) < 0.05] = -1
    x = rng.choice(np.array([0.0, -0.0, 1.5, -1.5, 2.0, np.nan, 3.25]), size=n)
    s = [WORDS[i] for i in rng.integers(0, len(WORDS), size=n)]
    v = rng.integers(0, 1000, size=n).astype(np.int64)
    rows = list(zip(k.tolist(), x.tolist(), s, v.tolist()))
    schema = ref.Schema([("k", "int"), ("x", "float"), ("s", "str"), ("v", "int")])
    return ref.ColumnTable.from_rows(schema, rows)


BIG = 100_000


def pair_digest(li, ri):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(li, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(ri, dtype="<i8").tobytes())
    return h.hexdigest()


def encode_value(v):
    """Predicate constant as text: i:<int>, f:<float.hex>, s:<str>."""
    if isinstance(v, str):
        return "s:" + v
    if isinstance(v, float):
        return "f:" + v.hex()
    return "i:" + str(int(v))


def with_index(t, name):
    schema = ref.Schema(list(t.schema.columns) + [(name, "int")])
    return ref.ColumnTable(schema, list(t.columns) + [np.arange(t.n_rows, dtype=np.int64)],
                           pool=t.pool)


def main():
    rng = np.random.default_rng(20260)
    out = {}
    sizes = [0, 1, 7, 40, 200, 3000, 25000]
    tabs = [random_table(rng, n) for n in sizes]
    for t, tab in enumerate(tabs):
        for ci, (name, _) in enumerate(tab.schema.columns):
            out[f"tab{t}_{name}"] = tab.columns[ci]
        out[f"tab{t}_pool"] = np.asarray(tab.pool, dtype=str)
        for i, (col, op, val) in enumerate(SELECT_PREDICATES):
            got = ref.select(tab, ref.Predicate(col, op, val))
            out[f"sel{t}_{i}"] = np.asarray(got.row_ids, dtype=np.int64)
    pairs = [(2, 3, "k"), (3, 2, "k"), (3, 3, "k"), (4, 5, "k"), (5, 4, "s"), (4, 4, "s"),
             (3, 4, "x"), (5, 5, "x"), (0, 4, "k"), (4, 0, "s"), (5, 6, "k"), (6, 5, "s"),
             (1, 1, "k")]
    for j, (a, b, key) in enumerate(pairs):
        left = with_index(tabs[a], "li")
        right = with_index(tabs[b], "ri")
        got = ref.join(left, right, key, key)
        out[f"join{j}_spec"] = np.array([a, b, "kxs".index(key)], dtype=np.int64)
        li = np.asarray(got.column("li"), dtype=np.int64)
        ri = np.asarray(got.column("ri"), dtype=np.int64)
        out[f"join{j}_n"] = np.array([li.shape[0]], dtype=np.int64)
        if li.shape[0] <= BIG:
            out[f"join{j}_li"], out[f"join{j}_ri"] = li, ri
        else:  # large outputs: digest of the pair lists in output order
            out[f"join{j}_sha"] = np.asarray([pair_digest(li, ri)], dtype=str)
        out[f"join{j}_names"] = np.asarray(got.schema.names, dtype=str)
    # the demo chain (demo.py:37-47) on the reference's own posts generator
    posts = qa_forum(4000, 6000, seed=2718)
    for ci, (name, _) in enumerate(posts.schema.columns):
        out[f"qa_{name}"] = posts.columns[ci]
    out["qa_pool"] = np.asarray(posts.pool, dtype=str)
    tagged = ref.select(posts, ref.Predicate("Tag", "=", "Java"))
    questions = ref.select(tagged, ref.Predicate("Type", "=", "question"))
    answers = ref.select(tagged, ref.Predicate("Type", "=", "answer"))
    qa = ref.join(questions, answers, "AnswerId", "PostId")
    out["qa_u1"] = np.asarray(qa.column("UserId-1"), dtype=np.int64)
    out["qa_u2"] = np.asarray(qa.column("UserId-2"), dtype=np.int64)
    g = ref.table_to_graph(qa, ref.EdgeSpec("UserId-1", "UserId-2"))
    pr = ref.pagerank(g)
    ids = np.asarray(sorted(pr), dtype=np.int64)
    out["qa_pr_ids"] = ids
    out["qa_pr"] = np.asarray([pr[int(i)] for i in ids], dtype=np.float64)
    out["sel_preds"] = np.asarray([f"{c}\t{op}\t{encode_value(v)}"
                                   for c, op, v in SELECT_PREDICATES], dtype=str)
    out["n_tabs"] = np.array([len(tabs)])
    out["n_joins"] = np.array([len(pairs)])
    np.savez_compressed(HERE / "relational.npz", **out)
    print("wrote", HERE / "relational.npz", len(out), "arrays;",
          "qa pairs", out["qa_u1"].shape[0], "join sizes",
          [int(out[f"join{j}_n"][0]) for j in range(len(pairs))])


if __name__ == "__main__":
    main()
