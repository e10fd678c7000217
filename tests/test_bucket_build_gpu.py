"""The MSD bucket build (csrc/bucket_build.cu) against the LSD sort build and
the oracle, on tables shaped to reach every one of its paths.

Both device builds must give the reference's CSR bit for bit (convert.py:
128-175): node set and dense order (convert.py:51-52), duplicates dropped
(convert.py:76-80), rows sorted (convert.py:71-89), int64 offsets
(convert.py:154-157). GT_BUILD selects the path per call ("bucket" forces
the bucket build for any size, "sort" the LSD pipeline).

Paths exercised: one and two partition levels; leaves grouping many small
buckets; huge buckets split by row; hub rows split by column with grouped
children; column children larger than a leaf (shared-memory bitmap); runs of
one duplicated key larger than a leaf; negative and extreme ids; extra
isolated nodes.
"""

import os

import numpy as np
import pytest

import paper_1503_07881_b200 as gt
from helpers import assert_csr_equal
from oracle import reference_port as ref
from paper_1503_07881_b200.synth import rmat_edges

pytestmark = pytest.mark.gpu
SPEC = gt.EdgeSpec("src", "dst")
LEAF_CAP = 8192  # keys per leaf (LF_CAP)


def build_with(mode, src, dst, device=True):
    old = os.environ.get("GT_BUILD")
    os.environ["GT_BUILD"] = mode
    try:
        t = gt.edge_table(np.asarray(src, np.int64), np.asarray(dst, np.int64))
        if device:
            t = t.to_device()
        return gt.table_to_graph(t, SPEC).csr()
    finally:
        if old is None:
            os.environ.pop("GT_BUILD", None)
        else:
            os.environ["GT_BUILD"] = old


@pytest.mark.parametrize("rows,n_ids,seed", [(1000, 50, 1), (300_000, 1 << 16, 2),
                                             (2_000_000, 1 << 20, 3), (1_500_000, 3000, 4)])
def test_uniform_tables(rows, n_ids, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n_ids, rows)
    dst = rng.integers(0, n_ids, rows)
    b = build_with("bucket", src, dst)
    s = build_with("sort", src, dst)
    assert_csr_equal(b, s, f"uniform {rows}x{n_ids}")


@pytest.mark.parametrize("scale,rows,permute", [(14, 400_000, False), (16, 1_500_000, True),
                                                (18, 4_000_000, True), (17, 3_000_000, False)])
def test_rmat_tables(scale, rows, permute):
    src, dst = rmat_edges(scale, rows, seed=scale, permute=permute)
    b = build_with("bucket", src, dst)
    s = build_with("sort", src, dst)
    assert_csr_equal(b, s, f"rmat s{scale}")


def test_hub_rows_and_bitmap_children():
    """A row of 3 M edges (column children larger than a leaf: bitmap path),
    rows of 20-200 K (children grouped), a hub column (the in side), and a
    single (src, dst) pair repeated 50 K times."""
    rng = np.random.default_rng(9)
    W = 1 << 20
    parts_s, parts_d = [], []
    parts_s.append(np.full(3_000_000, 7)); parts_d.append(rng.integers(0, W, 3_000_000))
    for h, d in ((11, 200_000), (12, 20_000), (13, 9_000)):
        parts_s.append(np.full(d, h)); parts_d.append(rng.integers(0, W, d))
    parts_s.append(rng.integers(0, W, 500_000)); parts_d.append(np.full(500_000, 5))
    parts_s.append(np.full(50_000, 99)); parts_d.append(np.full(50_000, 123_456))
    parts_s.append(rng.integers(0, W, 2_000_000)); parts_d.append(rng.integers(0, W, 2_000_000))
    src = np.concatenate(parts_s).astype(np.int64)
    dst = np.concatenate(parts_d).astype(np.int64)
    perm = rng.permutation(src.shape[0])
    src, dst = src[perm], dst[perm]
    b = build_with("bucket", src, dst)
    s = build_with("sort", src, dst)
    assert_csr_equal(b, s, "hubs")
    # row 7 keeps every distinct destination, sorted
    i = int(np.searchsorted(b.ids, 7))
    row = b.out_adj[b.out_off[i]:b.out_off[i + 1]]
    want = np.unique(dst[src == 7])
    assert np.array_equal(row, want)


def test_single_key_repeated_beyond_a_leaf():
    src = np.concatenate([np.full(40_000, 3), np.arange(1 << 20) % 1000]).astype(np.int64)
    dst = np.concatenate([np.full(40_000, 4), (np.arange(1 << 20) * 7) % 1000]).astype(np.int64)
    b = build_with("bucket", src, dst)
    s = build_with("sort", src, dst)
    assert_csr_equal(b, s, "repeated key")


@pytest.mark.parametrize("lo", [-(1 << 40), -5, (1 << 62), -(1 << 63)])
def test_offset_id_ranges(lo):
    rng = np.random.default_rng(3)
    n = 1_200_000
    src = (rng.integers(0, 1 << 19, n) + lo).astype(np.int64)
    dst = (rng.integers(0, 1 << 19, n) + lo).astype(np.int64)
    b = build_with("bucket", src, dst)
    s = build_with("sort", src, dst)
    assert_csr_equal(b, s, f"lo={lo}")
    assert b.ids[0] >= lo


def test_small_tables_vs_oracle():
    """Small cases forced through the bucket path (leaf-sized buckets, one
    level) against the numpy restatement of convert.py."""
    rng = np.random.default_rng(5)
    for rows, n in ((1, 1), (2, 2), (17, 5), (5000, 100), (70_000, 30_000)):
        src = rng.integers(-3, n, rows)
        dst = rng.integers(-3, n, rows)
        b = build_with("bucket", src, dst)
        assert_csr_equal(b, ref.build_csr(src.astype(np.int64), dst.astype(np.int64)),
                         f"rows={rows}")


def test_extra_isolated_nodes():
    """build_csr_nodes (graph_from_edges with extra node ids) through the
    bucket path: isolated ids get empty rows in both CSRs."""
    import torch

    from paper_1503_07881_b200 import _native

    rng = np.random.default_rng(8)
    rows = 1 << 20
    src = rng.integers(0, 1 << 19, rows).astype(np.int64)
    dst = rng.integers(0, 1 << 19, rows).astype(np.int64)
    extra = np.array([(1 << 19) + 5, -7, 12], dtype=np.int64)
    old = os.environ.get("GT_BUILD")
    os.environ["GT_BUILD"] = "bucket"
    try:
        h = _native.build_csr(src, dst, rows, False, nodes=extra)
        g = gt.graph.DeviceGraph(h)
        got = g.csr()
    finally:
        if old is None:
            os.environ.pop("GT_BUILD", None)
        else:
            os.environ["GT_BUILD"] = old
    ids = np.unique(np.concatenate([src, dst, extra]))
    assert np.array_equal(got.ids, ids)
    for x in (-7, (1 << 19) + 5):
        i = int(np.searchsorted(ids, x))
        assert got.out_off[i] == got.out_off[i + 1] and got.in_off[i] == got.in_off[i + 1]
    del torch
