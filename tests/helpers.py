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
