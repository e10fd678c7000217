"""PageRank, triangle counting and the other CSR consumers on the device CSR.

Drop-ins for ``graphtables.algorithms.pagerank`` (algorithms.py:36-87) and
``triangle_count`` (algorithms.py:90-119): same signatures, validation and
results (PageRank fp64 within 1e-9 L1 of the reference — GPU summation order
differs, but is fixed, so runs are bitwise reproducible; triangle counts
exact). Any graph exposing ``node_ids()``/``record()`` is accepted; host
graphs are uploaded first (isolated nodes included).

SURVEY §8f next #4: ``sssp`` (BFS hop distances, algorithms.py:125-141),
``connected_components`` (:232-248) and ``k_core`` (:206-229) on the same
device CSR (csrc/traverse.cu), with the reference's results and errors.
"""

from __future__ import annotations

from collections.abc import Mapping

import numpy as np

from . import _native
from .convert import resolve_workers
from .errors import UnknownNodeError
from .graph import DeviceGraph, upload


class RankMap(Mapping):
    """Read-only ``{node id: score}`` view over two arrays (ids ascending).

    Returned instead of building a Python dict of N entries
    (algorithms.py:87): lookups are a binary search, iteration yields ids in
    ascending order, ``dict(r)`` / ``r.items()`` / ``sum(r.values())`` work.
    """

    __slots__ = ("ids", "scores")

    def __init__(self, ids: np.ndarray, scores: np.ndarray):
        self.ids = ids
        self.scores = scores

    def __getitem__(self, node):
        try:
            pos = int(np.searchsorted(self.ids, node))
        except (TypeError, OverflowError):
            raise KeyError(node) from None
        if pos >= self.ids.shape[0] or self.ids[pos] != node:
            raise KeyError(node)
        return float(self.scores[pos])

    def __len__(self):
        return int(self.ids.shape[0])

    def __iter__(self):
        return iter(self.ids.tolist())

    def __contains__(self, node):
        try:
            self[node]
            return True
        except KeyError:
            return False

    def items(self):
        return zip(self.ids.tolist(), self.scores.tolist())

    def values(self):
        return self.scores.tolist()

    def to_dict(self) -> dict:
        return dict(zip(self.ids.tolist(), self.scores.tolist()))

    def __eq__(self, other):
        if isinstance(other, RankMap):
            return np.array_equal(self.ids, other.ids) and np.array_equal(self.scores,
                                                                           other.scores)
        if isinstance(other, Mapping):
            return self.to_dict() == dict(other.items())
        return NotImplemented

    def __repr__(self):
        return f"RankMap(nodes={len(self)})"


def pagerank(g, damping: float = 0.85, iterations: int = 10,
             workers: int | None = None) -> RankMap:
    """Damped power iteration, fp64, uniform start and dangling redistribution."""
    if not 0.0 < damping < 1.0:
        raise ValueError(f"damping must be in (0, 1), got {damping}")
    if iterations < 1:
        raise ValueError(f"iterations must be >= 1, got {iterations}")
    if g.node_count == 0:
        raise ValueError("pagerank needs a non-empty graph")
    resolve_workers(workers)
    dg = upload(g)
    scores = _native.pagerank(dg.handle, dg.node_count, damping, iterations)
    ids = dg.csr().ids if dg._host is not None else _ids_only(dg)
    return RankMap(ids, scores)


def _ids_only(dg: DeviceGraph) -> np.ndarray:
    ids = _native.host_empty(dg.node_count, np.int64)
    if ids.size:
        _native.check(_native.load().gt_graph_export(dg.handle, ids.ctypes.data, None, None,
                                                     None, None), "gt_graph_export")
    ids.flags.writeable = False
    return ids


def pagerank_device(g: DeviceGraph, damping: float, iterations: int, out_ptr: int) -> None:
    """Scores straight into a device buffer of N doubles (no host copy)."""
    _native.pagerank(g.handle, g.node_count, damping, iterations, out_ptr=out_ptr)


def triangle_count(g, workers: int | None = None) -> int:
    """Unordered mutually adjacent triples of the symmetrised graph."""
    resolve_workers(workers)
    if g.node_count == 0:
        return 0
    dg = upload(g)
    return _native.triangles(dg.handle)


def pagerank_and_triangles(g, damping: float = 0.85, iterations: int = 10,
                           scores_out_ptr: int | None = None, workers: int | None = None):
    """PageRank and the triangle count of one graph, run concurrently on two
    library lanes (PageRank on lane 1, the count on lane 0): same results as
    ``pagerank(g, ...)`` and ``triangle_count(g)``. With ``scores_out_ptr``
    the scores go to that device buffer (returns (None, count)); otherwise a
    RankMap is returned."""
    resolve_workers(workers)
    if not (0.0 < damping < 1.0):
        raise ValueError(f"damping must be in (0, 1), got {damping}")
    if iterations < 1:
        raise ValueError(f"iterations must be >= 1, got {iterations}")
    if g.node_count == 0:
        raise ValueError("pagerank needs a non-empty graph")
    dg = upload(g)
    if scores_out_ptr is not None:
        fut = _native.lane_submit(1, pagerank_device, dg, damping, iterations, scores_out_ptr)
    else:
        fut = _native.lane_submit(1, pagerank, dg, damping, iterations)
    try:
        tc = triangle_count(dg)
    finally:
        pr = fut.result()
    return pr, tc


class _NodeArrayMap(Mapping):
    """Read-only ``{node id: value}`` view over (ids ascending, values)."""

    __slots__ = ("ids", "values_")

    def __init__(self, ids: np.ndarray, values: np.ndarray):
        self.ids = ids
        self.values_ = values

    def _conv(self, x):
        return int(x)

    def __getitem__(self, node):
        try:
            pos = int(np.searchsorted(self.ids, node))
        except (TypeError, OverflowError):
            raise KeyError(node) from None
        if pos >= self.ids.shape[0] or self.ids[pos] != node:
            raise KeyError(node)
        return self._conv(self.values_[pos])

    def __len__(self):
        return int(self.ids.shape[0])

    def __iter__(self):
        return iter(self.ids.tolist())

    def __contains__(self, node):
        try:
            self[node]
            return True
        except KeyError:
            return False

    def items(self):
        return zip(self.ids.tolist(), (self._conv(x) for x in self.values_.tolist()))

    def values(self):
        return [self._conv(x) for x in self.values_.tolist()]

    def to_dict(self) -> dict:
        return dict(self.items())

    def __eq__(self, other):
        if isinstance(other, Mapping):
            return self.to_dict() == dict(other.items())
        return NotImplemented

    def __repr__(self):
        return f"{type(self).__name__}(nodes={len(self)})"


class DistMap(_NodeArrayMap):
    """``{node id: hops or None}`` (algorithms.py:125-141: unreachable -> None)."""

    def _conv(self, x):
        return None if x < 0 else int(x)


class LabelMap(_NodeArrayMap):
    """``{node id: component label}``, labels dense from 0."""


def sssp(g, source: int) -> DistMap:
    """Hop distances from source along directed edges (BFS); unreachable -> None."""
    dg = upload(g) if g.node_count else None
    if dg is None:
        raise UnknownNodeError(f"node {source} not in graph")
    ids = dg.csr().ids if dg._host is not None else _ids_only(dg)
    try:
        pos = int(np.searchsorted(ids, source))
    except (TypeError, OverflowError):
        raise UnknownNodeError(f"node {source} not in graph") from None
    if pos >= ids.shape[0] or ids[pos] != source:
        raise UnknownNodeError(f"node {source} not in graph")
    return DistMap(ids, _native.bfs(dg.handle, dg.node_count, pos))


def connected_components(g) -> LabelMap:
    """Weakly connected components of the symmetrized graph; dense labels
    numbered in ascending order of each component's smallest node id."""
    if g.node_count == 0:
        return LabelMap(np.empty(0, np.int64), np.empty(0, np.int64))
    dg = upload(g)
    labels, _ = _native.connected_components(dg.handle, dg.node_count)
    ids = dg.csr().ids if dg._host is not None else _ids_only(dg)
    return LabelMap(ids, labels)


def scc(g) -> LabelMap:
    """Strongly connected components (algorithms.py:144-203); labels dense,
    numbered in ascending order of each component's smallest node id."""
    if g.node_count == 0:
        return LabelMap(np.empty(0, np.int64), np.empty(0, np.int64))
    dg = upload(g)
    labels, _ = _native.scc(dg.handle, dg.node_count)
    ids = dg.csr().ids if dg._host is not None else _ids_only(dg)
    return LabelMap(ids, labels)


def k_core(g, k: int) -> DeviceGraph:
    """Maximal subgraph whose nodes all have >= k distinct undirected
    neighbors (iterative peeling); the induced subgraph as a new graph."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    dg = upload(g)
    return DeviceGraph(_native.kcore(dg.handle, k))
