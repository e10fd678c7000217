"""Deterministic synthetic edge tables (bench and test inputs).

``random_edges`` keeps the reference's uniform generator semantics
(``synth.py:20-29``: ``np.random.default_rng(seed).integers(0, n, size)`` for
src then dst). ``rmat_edges`` is the R-MAT generator the BASELINE configs
name; the reference has none, so it is defined here once and implemented
twice — in numpy (this file, the oracle side) and in CUDA
(``csrc/rmat.cu``, ``gt_rmat_generate``) — bit for bit identical. Every row
depends only on its index, so any row range can be generated on its own.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_U64 = np.uint64
_SEED_SALT = 0x5851F42D4C957F2D
_ROUND_SALT = 0xA0761D6478BD642F
_TWO53 = 9007199254740992.0
_MASK64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = x + _U64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def _sm64_scalar(x: int) -> int:
    return int(splitmix64(np.asarray([x & _MASK64], dtype=np.uint64))[0])


@dataclass(frozen=True)
class RmatSpec:
    scale: int
    rows: int
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    seed: int = 1
    permute: bool = False


def _thresholds(a: float, b: float, c: float):
    return int(a * _TWO53), int((a + b) * _TWO53), int((a + b + c) * _TWO53)


def feistel_permute(x: np.ndarray, scale: int, key: int) -> np.ndarray:
    """Keyed bijection of [0, 2^scale): 4-round Feistel, cycle-walked."""
    h = (scale + 1) // 2
    mh = _U64((1 << h) - 1)
    limit = _U64(1 << scale)
    rk = [_sm64_scalar(key ^ ((_ROUND_SALT * (r + 1)) & _MASK64)) for r in range(4)]
    x = x.astype(np.uint64, copy=True)
    todo = np.ones(x.shape[0], dtype=bool)
    while True:
        idx = np.nonzero(todo)[0]
        if idx.size == 0:
            return x
        v = x[idx]
        left, right = v >> _U64(h), v & mh
        for r in range(4):
            left, right = right, left ^ (splitmix64(right ^ _U64(rk[r])) & mh)
        v = (left << _U64(h)) | right
        x[idx] = v
        todo[idx] = v >= limit


def rmat_edges(scale: int, rows: int, a: float = 0.57, b: float = 0.19, c: float = 0.19,
               seed: int = 1, permute: bool = False, start: int = 0,
               chunk: int = 1 << 22):
    """R-MAT rows [start, start+rows) as two int64 arrays (src, dst)."""
    if scale < 1 or scale > 40:
        raise ValueError("scale must be in [1, 40]")
    key = _sm64_scalar(seed ^ _SEED_SALT)
    ta, tab, tabc = (_U64(t) for t in _thresholds(a, b, c))
    src = np.empty(rows, dtype=np.int64)
    dst = np.empty(rows, dtype=np.int64)
    for lo in range(0, rows, chunk):
        hi = min(rows, lo + chunk)
        e = np.arange(start + lo, start + hi, dtype=np.uint64)
        base = _U64(key) + e * _U64(scale)
        s = np.zeros(hi - lo, dtype=np.uint64)
        d = np.zeros(hi - lo, dtype=np.uint64)
        for level in range(scale):
            u = splitmix64(base + _U64(level)) >> _U64(11)
            sb = (u >= tab).astype(np.uint64)
            db = (((u >= ta) & (u < tab)) | (u >= tabc)).astype(np.uint64)
            s = (s << _U64(1)) | sb
            d = (d << _U64(1)) | db
        if permute:
            s = feistel_permute(s, scale, key)
            d = feistel_permute(d, scale, key)
        src[lo:hi] = s.astype(np.int64)
        dst[lo:hi] = d.astype(np.int64)
    return src, dst


def random_edges_arrays(n_nodes: int, n_edges: int, seed: int = 0):
    """Uniform iid src/dst in [0, n_nodes) — synth.py:20-29 semantics."""
    if n_nodes < 0 or n_edges < 0:
        raise ValueError("sizes must be >= 0")
    if n_nodes == 0 and n_edges > 0:
        raise ValueError("cannot draw edges from an empty node range")
    rng = np.random.default_rng(seed)
    src = rng.integers(0, max(n_nodes, 1), size=n_edges, dtype=np.int64)
    dst = rng.integers(0, max(n_nodes, 1), size=n_edges, dtype=np.int64)
    return src, dst


_UNIFORM_SALT = 0xD1B54A32D192ED03


def _mulhi64(x: np.ndarray, n: int) -> np.ndarray:
    """High 64 bits of x * n for uint64 x and n < 2^32 (no 128-bit numpy ints)."""
    xh = x >> _U64(32)
    xl = x & _U64(0xFFFFFFFF)
    nn = _U64(n)
    return (xh * nn + ((xl * nn) >> _U64(32))) >> _U64(32)


def uniform_edges(n_nodes: int, rows: int, seed: int = 4, start: int = 0):
    """Uniform iid (src, dst) in [0, n_nodes): the counter-based stand-in for
    BASELINE config 4 (reference synth.random_edges semantics, synth.py:20-29),
    bit-identical to csrc/rmat.cu uniform_kernel. Row e: src =
    hi64(splitmix64(key + 2e) * n), dst from key + 2e + 1."""
    if not 1 <= n_nodes < (1 << 32):
        raise ValueError("n_nodes must be in [1, 2^32)")
    key = _sm64_scalar(seed ^ _UNIFORM_SALT)
    e = np.arange(start, start + rows, dtype=np.uint64)
    with np.errstate(over="ignore"):
        b = _U64(key) + _U64(2) * e
        src = _mulhi64(splitmix64(b), n_nodes).astype(np.int64)
        dst = _mulhi64(splitmix64(b + _U64(1)), n_nodes).astype(np.int64)
    return src, dst


@dataclass(frozen=True)
class UniformSpec:
    n_nodes: int
    rows: int
    seed: int = 4


# BASELINE.json configs (C3 reuses the C2 table; C4 and C5 are generated on
# the device by bench.py).
CONFIGS = {
    "c1": RmatSpec(scale=17, rows=1_048_576, seed=1, permute=False),
    "c2": RmatSpec(scale=22, rows=69_000_000, seed=2, permute=True),
    "c4": RmatSpec(scale=26, rows=1_470_000_000, seed=3, permute=True),
    "c5": UniformSpec(n_nodes=100_000_000, rows=2_000_000_000, seed=4),
}


def spec_edges(spec, rows: int | None = None, start: int = 0):
    """Host (numpy) rows [start, start+rows) of a config's table."""
    rows = spec.rows if rows is None else rows
    if isinstance(spec, UniformSpec):
        return uniform_edges(spec.n_nodes, rows, spec.seed, start)
    assert start == 0
    return rmat_edges(spec.scale, rows, spec.a, spec.b, spec.c, spec.seed, spec.permute)


def rmat_device(spec, device: str = "cuda", start: int = 0, rows: int | None = None):
    """Generate rows [start, start+rows) of a config's table (R-MAT or uniform)
    straight into HBM."""
    import torch

    from . import _native

    rows = spec.rows if rows is None else rows
    src = torch.empty(rows, dtype=torch.int64, device=device)
    dst = torch.empty(rows, dtype=torch.int64, device=device)
    if isinstance(spec, UniformSpec):
        _native.uniform_generate(spec.n_nodes, rows, spec.seed, src.data_ptr(), dst.data_ptr(),
                                 start=start)
        return src, dst
    _native.rmat_generate(spec.scale, rows, spec.a, spec.b, spec.c, spec.seed, spec.permute,
                          src.data_ptr(), dst.data_ptr(), start=start)
    return src, dst


def random_edges(n_nodes: int, n_edges: int, seed: int = 0):
    """ColumnTable of uniform random edges (reference synth.random_edges)."""
    from .tables import INT, ColumnTable, Schema

    src, dst = random_edges_arrays(n_nodes, n_edges, seed)
    return ColumnTable(Schema([("src", INT), ("dst", INT)]), [src, dst])


def rmat_table(spec: RmatSpec):
    """ColumnTable of an R-MAT spec generated on the host (numpy)."""
    from .tables import INT, ColumnTable, Schema

    src, dst = rmat_edges(spec.scale, spec.rows, spec.a, spec.b, spec.c, spec.seed,
                          spec.permute)
    return ColumnTable(Schema([("src", INT), ("dst", INT)]), [src, dst])
