"""Shared test helpers: golden fixtures and CSR comparison."""

from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CSR_FIELDS = ("ids", "out_off", "out_adj", "in_off", "in_adj")


@lru_cache(maxsize=1)
def golden_cases() -> dict:
    """{case name: {field: array}} recorded from the real reference."""
    data = np.load(GOLDEN / "cases.npz")
    out = {}
    for name in data["__names__"].tolist():
        out[name] = {k.split("/", 1)[1]: data[k] for k in data.files if k.startswith(name + "/")}
    return out


@lru_cache(maxsize=1)
def golden_traverse() -> dict:
    """{case: {field: array}} of sssp / connected_components / k_core recorded
    from the real reference (tests/golden/make_golden_traverse.py)."""
    data = np.load(GOLDEN / "traverse.npz")
    out = {}
    for name in data["__names__"].tolist():
        out[name] = {k.split("/", 1)[1]: data[k] for k in data.files if k.startswith(name + "/")}
    return out


@lru_cache(maxsize=1)
def golden_scc() -> dict:
    """{case: {src, dst, extra, ids, scc}} recorded from the real reference's
    graphtables.scc (tests/golden/make_golden_scc.py)."""
    data = np.load(GOLDEN / "scc.npz")
    out = {}
    for name in data["__names__"].tolist():
        out[name] = {k.split("/", 1)[1]: data[k] for k in data.files if k.startswith(name + "/")}
    return out


@lru_cache(maxsize=1)
def golden_updates() -> dict:
    """{case: {src, dst, del_nodes, del_src, del_dst, add_nodes, add_src,
    add_dst, ids, out_off, out_adj, in_off, in_adj}} from the real reference's
    Graph mutation calls (tests/golden/make_golden_updates.py)."""
    data = np.load(GOLDEN / "updates.npz")
    out = {}
    for name in data["__names__"].tolist():
        out[name] = {k.split("/", 1)[1]: data[k] for k in data.files if k.startswith(name + "/")}
    return out


def golden_c1() -> dict:
    data = np.load(GOLDEN / "c1.npz")
    return {k: data[k] for k in data.files}


def assert_csr_equal(got, want, where=""):
    for f in CSR_FIELDS:
        a = np.asarray(getattr(got, f) if not isinstance(got, dict) else got[f])
        b = np.asarray(getattr(want, f) if not isinstance(want, dict) else want[f])
        assert a.shape == b.shape and np.array_equal(a, b), f"{where}: CSR field {f} differs"


def sha(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_digraph_edges(rng, n_nodes, p):
    """Edges of the reference test helper's random digraph (util.py:28-34)."""
    mask = rng.random((n_nodes, n_nodes)) < p
    src, dst = np.nonzero(mask)
    return src.astype(np.int64), dst.astype(np.int64)


def dense_pagerank(adj, damping, iterations):
    """Independent dense power iteration (oracles.py:149-160 formula)."""
    n = adj.shape[0]
    out_deg = adj.sum(axis=1)
    m = np.zeros((n, n))
    nz = out_deg > 0
    m[nz] = adj[nz] / out_deg[nz, None]
    score = np.full(n, 1.0 / n)
    for _ in range(iterations):
        dangling = score[~nz].sum()
        score = (1 - damping) / n + damping * (m.T @ score + dangling / n)
    return score


def cubic_triangles(sym_adj):
    """Brute-force closed-walk count / 6 (oracles.py:163-167 formula)."""
    a = sym_adj.astype(np.float64)
    np.fill_diagonal(a, 0.0)
    return int(round(np.einsum("ij,jk,ki->", a, a, a) / 6.0))


# ---------------------------------------------------------- select / join goldens

REL_SCHEMA = (("k", "int"), ("x", "float"), ("s", "str"), ("v", "int"))


def decode_const(text: str):
    """Predicate constant written by make_golden_relational.encode_value."""
    tag, val = text[:2], text[2:]
    if tag == "s:":
        return val
    if tag == "f:":
        return float.fromhex(val)
    return int(val)


@lru_cache(maxsize=1)
def golden_relational() -> dict:
    """Select / join outputs of the real reference (make_golden_relational.py):
    {"tables": [(columns dict, pool list)], "preds": [(col, op, value)],
     "sel": {(t, i): row ids}, "joins": [dict], "qa": dict}."""
    d = np.load(GOLDEN / "relational.npz")
    tabs = []
    for t in range(int(d["n_tabs"][0])):
        cols = {name: d[f"tab{t}_{name}"] for name, _ in REL_SCHEMA}
        tabs.append((cols, d[f"tab{t}_pool"].tolist()))
    preds = []
    for line in d["sel_preds"].tolist():
        c, op, v = line.split("\t")
        preds.append((c, op, decode_const(v)))
    sel = {(t, i): d[f"sel{t}_{i}"] for t in range(len(tabs)) for i in range(len(preds))}
    joins = []
    for j in range(int(d["n_joins"][0])):
        a, b, key = d[f"join{j}_spec"].tolist()
        rec = {"left": a, "right": b, "key": "kxs"[key], "n": int(d[f"join{j}_n"][0]),
               "names": d[f"join{j}_names"].tolist()}
        if f"join{j}_li" in d.files:
            rec["li"], rec["ri"] = d[f"join{j}_li"], d[f"join{j}_ri"]
        else:
            rec["sha"] = str(d[f"join{j}_sha"][0])
        joins.append(rec)
    qa = {k[3:]: d[k] for k in d.files if k.startswith("qa_")}
    return {"tables": tabs, "preds": preds, "sel": sel, "joins": joins, "qa": qa}


def pair_digest(li, ri) -> str:
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(li, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(ri, dtype="<i8").tobytes())
    return h.hexdigest()


def join_keys_py(cols, pool, key):
    """Key column as python values the way the reference hashes them
    (tables.py:408-409: decoded strings, .tolist())."""
    col = cols[key]
    if key == "s":
        return [pool[c] for c in col.tolist()]
    return col.tolist()
