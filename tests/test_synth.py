"""R-MAT / uniform generators (host side; the device twin is checked in
test_build_gpu.py)."""

import numpy as np

from paper_1503_07881_b200.synth import (
    feistel_permute,
    random_edges,
    random_edges_arrays,
    rmat_edges,
)


def test_rmat_deterministic_and_row_addressable():
    s1, d1 = rmat_edges(12, 5000, seed=3, permute=True)
    s2, d2 = rmat_edges(12, 5000, seed=3, permute=True)
    assert np.array_equal(s1, s2) and np.array_equal(d1, d2)
    s3, d3 = rmat_edges(12, 1000, seed=3, permute=True, start=4000)
    assert np.array_equal(s1[4000:], s3) and np.array_equal(d1[4000:], d3)
    s4, _ = rmat_edges(12, 5000, seed=4, permute=True)
    assert not np.array_equal(s1, s4)


def test_rmat_range_and_skew():
    s, d = rmat_edges(10, 20000, seed=1)
    assert s.min() >= 0 and d.min() >= 0 and s.max() < 1024 and d.max() < 1024
    # quadrant a (0.57) dominates: the top bit is 1 in src for ~c+d = 24% of rows
    frac = float(np.mean(s >> 9))
    assert 0.2 < frac < 0.28
    frac_d = float(np.mean(d >> 9))  # b + d = 24%
    assert 0.2 < frac_d < 0.28


def test_feistel_is_a_bijection():
    for scale in (5, 8, 11):
        x = np.arange(1 << scale, dtype=np.uint64)
        y = feistel_permute(x, scale, key=12345)
        assert np.array_equal(np.sort(y), x)
        assert not np.array_equal(y, x)


def test_random_edges_matches_numpy_generator_semantics():
    src, dst = random_edges_arrays(1000, 5000, seed=9)
    rng = np.random.default_rng(9)
    assert np.array_equal(src, rng.integers(0, 1000, size=5000, dtype=np.int64))
    assert np.array_equal(dst, rng.integers(0, 1000, size=5000, dtype=np.int64))
    t = random_edges(1000, 5000, seed=9)
    assert t.n_rows == 5000 and t.schema.names == ["src", "dst"]
