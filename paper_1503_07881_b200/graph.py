"""Graph types of the drop-in.

``DeviceGraph`` is what ``table_to_graph`` returns: an owner of the device
CSR pair built by ``gt_build_csr``. It answers the reference ``Graph`` read
API (graphs.py:62-88, 148-226: ``node_count``, ``edge_count``,
``node_ids()``, ``record()``, ``neighbors()``, ``has_edge()``,
``undirected_neighbors()``, ``__eq__``, ``check_invariants()``,
``memory_bytes()``) from a lazily exported host copy whose adjacency views
are read-only (test_convert.py:75-78). The first mutation turns it into a
host ``Graph`` and drops the device buffers, so a converted graph stays
mutable (test_convert.py:80-84).

``Graph`` is the host-side dynamic graph (dict of node records with sorted
in/out vectors, graphs.py:42-58 semantics) used for mutation and for the
sequential-replay oracle ``from_edges`` (graphs.py:229-234).
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native
from .errors import UnknownNodeError

_EMPTY = np.empty(0, dtype=np.int64)
_EMPTY.flags.writeable = False


def _frozen(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


class NodeRecord:
    """Node id plus its sorted in/out adjacency vectors (graphs.py:42-50)."""

    __slots__ = ("id", "in_nbrs", "out_nbrs")

    def __init__(self, node_id: int, in_nbrs=_EMPTY, out_nbrs=_EMPTY):
        self.id = node_id
        self.in_nbrs = in_nbrs
        self.out_nbrs = out_nbrs


def _sorted_insert(vec: np.ndarray, value: int):
    pos = int(np.searchsorted(vec, value))
    if pos < vec.shape[0] and vec[pos] == value:
        return vec, False
    return _frozen(np.insert(vec, pos, value)), True


def _sorted_remove(vec: np.ndarray, value: int):
    pos = int(np.searchsorted(vec, value))
    if pos >= vec.shape[0] or vec[pos] != value:
        return vec, False
    return _frozen(np.delete(vec, pos)), True


class _GraphReadAPI:
    """Read API shared by Graph and DeviceGraph, written against
    ``node_ids()`` / ``record()`` / ``edge_count``."""

    def neighbors(self, node_id: int, direction: str = "out") -> np.ndarray:
        rec = self.record(node_id)
        if direction == "out":
            return rec.out_nbrs
        if direction == "in":
            return rec.in_nbrs
        raise ValueError(f"direction must be 'in' or 'out', got {direction!r}")

    def out_degree(self, node_id: int) -> int:
        return int(self.record(node_id).out_nbrs.shape[0])

    def in_degree(self, node_id: int) -> int:
        return int(self.record(node_id).in_nbrs.shape[0])

    def undirected_neighbors(self, node_id: int) -> np.ndarray:
        rec = self.record(node_id)
        merged = np.union1d(rec.in_nbrs, rec.out_nbrs)
        return merged[merged != node_id]

    def has_edge(self, src: int, dst: int) -> bool:
        if not self.has_node(src):
            return False
        out = self.record(src).out_nbrs
        pos = int(np.searchsorted(out, dst))
        return pos < out.shape[0] and out[pos] == dst

    def out_csr(self):
        """(ids ascending, out offsets, out adjacency) as numpy arrays."""
        ids = np.asarray(self.node_ids(), dtype=np.int64)
        vecs = [self.record(int(i)).out_nbrs for i in ids.tolist()]
        lens = np.fromiter((v.shape[0] for v in vecs), dtype=np.int64, count=len(vecs))
        off = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
        adj = np.concatenate(vecs).astype(np.int64) if vecs else np.empty(0, np.int64)
        return ids, off, adj

    def __eq__(self, other):
        """Same node keys, edge count and out vectors (graphs.py:195-205)."""
        if not (hasattr(other, "node_ids") and hasattr(other, "record")
                and hasattr(other, "edge_count")):
            return NotImplemented
        if self.edge_count != other.edge_count or self.node_count != other.node_count:
            return False
        a_ids, a_off, a_adj = self.out_csr()
        if isinstance(other, _GraphReadAPI):
            b_ids, b_off, b_adj = other.out_csr()
        else:
            b_ids, b_off, b_adj = _GraphReadAPI.out_csr(other)
        return (np.array_equal(a_ids, b_ids) and np.array_equal(a_off, b_off)
                and np.array_equal(a_adj, b_adj))

    __hash__ = None


class Graph(_GraphReadAPI):
    """Host dynamic directed simple graph (graphs.py:53-234 semantics)."""

    def __init__(self):
        self._nodes: dict[int, NodeRecord] = {}
        self._edge_count = 0

    @property
    def node_count(self) -> int:
        return len(self._nodes)

    @property
    def edge_count(self) -> int:
        return self._edge_count

    def has_node(self, node_id: int) -> bool:
        return node_id in self._nodes

    def node_ids(self) -> list[int]:
        return sorted(self._nodes)

    def record(self, node_id: int) -> NodeRecord:
        rec = self._nodes.get(node_id)
        if rec is None:
            raise UnknownNodeError(f"node {node_id} not in graph")
        return rec

    def add_node(self, node_id: int) -> bool:
        if node_id in self._nodes:
            return False
        self._nodes[node_id] = NodeRecord(int(node_id))
        return True

    def add_edge(self, src: int, dst: int) -> bool:
        self.add_node(src)
        self.add_node(dst)
        s = self._nodes[src]
        s.out_nbrs, inserted = _sorted_insert(s.out_nbrs, dst)
        if not inserted:
            return False
        d = self._nodes[dst]
        d.in_nbrs, _ = _sorted_insert(d.in_nbrs, src)
        self._edge_count += 1
        return True

    def del_edge(self, src: int, dst: int) -> bool:
        s = self._nodes.get(src)
        if s is None:
            return False
        s.out_nbrs, removed = _sorted_remove(s.out_nbrs, dst)
        if not removed:
            return False
        d = self._nodes[dst]
        d.in_nbrs, _ = _sorted_remove(d.in_nbrs, src)
        self._edge_count -= 1
        return True

    def del_node(self, node_id: int) -> bool:
        rec = self._nodes.get(node_id)
        if rec is None:
            return False
        removed = rec.out_nbrs.shape[0]
        for v in rec.out_nbrs.tolist():
            if v != node_id:
                self._nodes[v].in_nbrs, _ = _sorted_remove(self._nodes[v].in_nbrs, node_id)
        for u in rec.in_nbrs.tolist():
            if u != node_id:
                self._nodes[u].out_nbrs, _ = _sorted_remove(self._nodes[u].out_nbrs, node_id)
                removed += 1
        del self._nodes[node_id]
        self._edge_count -= removed
        return True

    def subgraph(self, node_ids) -> "Graph":
        keep = {int(n) for n in node_ids}
        sub = Graph()
        for n in keep:
            rec = self.record(n)
            out = _frozen(np.asarray([v for v in rec.out_nbrs.tolist() if v in keep], np.int64))
            inn = _frozen(np.asarray([u for u in rec.in_nbrs.tolist() if u in keep], np.int64))
            sub._nodes[n] = NodeRecord(n, in_nbrs=inn, out_nbrs=out)
            sub._edge_count += out.shape[0]
        return sub

    def memory_bytes(self) -> int:
        total = len(self._nodes) * 120
        for rec in self._nodes.values():
            total += rec.in_nbrs.nbytes + rec.out_nbrs.nbytes
        return total

    def check_invariants(self) -> None:
        total_out = total_in = 0
        for n, rec in self._nodes.items():
            for vec in (rec.out_nbrs, rec.in_nbrs):
                if vec.shape[0] > 1:
                    assert bool(np.all(vec[1:] > vec[:-1])), f"unsorted vector at {n}"
            total_out += rec.out_nbrs.shape[0]
            total_in += rec.in_nbrs.shape[0]
            for dst in rec.out_nbrs.tolist():
                other = self._nodes[dst].in_nbrs
                pos = int(np.searchsorted(other, n))
                assert pos < other.shape[0] and other[pos] == n, \
                    f"missing in-entry for edge ({n}, {dst})"
        assert total_out == total_in == self._edge_count, \
            f"edge count {self._edge_count} != sum of degrees {total_out}/{total_in}"

    def __repr__(self):
        return f"Graph(nodes={self.node_count}, edges={self.edge_count})"


def from_edges(edges) -> Graph:
    """Sequential edge replay (graphs.py:229-234): the conversion oracle."""
    g = Graph()
    for src, dst in edges:
        g.add_edge(int(src), int(dst))
    return g


class _HostCSR:
    __slots__ = ("ids", "out_off", "out_adj", "in_off", "in_adj")

    def __init__(self, ids, out_off, out_adj, in_off, in_adj):
        self.ids, self.out_off, self.out_adj = ids, out_off, out_adj
        self.in_off, self.in_adj = in_off, in_adj
        for a in (ids, out_off, out_adj, in_off, in_adj):
            a.flags.writeable = False


def _mutating(name):
    def method(self, *args, **kwargs):
        return getattr(self._materialize(), name)(*args, **kwargs)
    method.__name__ = name
    return method


def _as_list(a):
    if a is None:
        return []
    return [int(x) for x in (a.tolist() if hasattr(a, "tolist") else a)]


def _pair_lists(p):
    if p is None:
        return [], []
    return _as_list(p[0]), _as_list(p[1])


class DeviceGraph(_GraphReadAPI):
    """Directed simple graph whose CSR pair lives in HBM (gt_graph handle)."""

    def __init__(self, handle: int):
        self._handle = handle
        self._n, self._e = _native.graph_sizes(handle)
        self._host: _HostCSR | None = None
        self._ids: np.ndarray | None = None  # ids alone, for node_ids()
        self._graph: Graph | None = None  # set once mutated
        self._finalizer = weakref.finalize(self, _native.graph_free, handle)

    # -- device side --------------------------------------------------------
    @property
    def handle(self) -> int:
        if self._graph is not None:
            raise RuntimeError("graph was mutated; its device CSR has been released")
        return self._handle

    @property
    def on_device(self) -> bool:
        return self._graph is None

    def device_views(self):
        """Device pointers (ids, out_off, out_adj[int32], in_off, in_adj[int32])."""
        return _native.graph_device_views(self.handle)

    def csr(self) -> _HostCSR:
        """Host copy in the reference's pool layout (original int64 ids)."""
        if self._host is None:
            self._host = _HostCSR(*_native.graph_export(self.handle, self._n, self._e))
        return self._host

    # -- read API -----------------------------------------------------------
    @property
    def node_count(self) -> int:
        return self._graph.node_count if self._graph is not None else self._n

    @property
    def edge_count(self) -> int:
        return self._graph.edge_count if self._graph is not None else self._e

    def node_ids(self) -> list[int]:
        if self._graph is not None:
            return self._graph.node_ids()
        if self._host is not None:
            return self._host.ids.tolist()
        if self._ids is None:  # ids only (8 B per node), not the whole CSR
            ids = np.empty(self._n, dtype=np.int64)
            _native.check(_native.load().gt_graph_export(self.handle, _native._ptr(ids), None, None,
                                                         None, None), "gt_graph_export")
            self._ids = _frozen(ids)
        return self._ids.tolist()

    @staticmethod
    def _as_id(node_id):
        try:
            x = int(node_id)
        except (TypeError, ValueError, OverflowError):
            return None
        if x != node_id or not (-(1 << 63) <= x < (1 << 63)):
            return None
        return x

    def _index(self, node_id) -> int:
        if self._host is not None:
            ids = self._host.ids
            try:
                pos = int(np.searchsorted(ids, node_id))
            except (TypeError, OverflowError):
                pos = ids.shape[0]
            if pos >= ids.shape[0] or ids[pos] != node_id:
                raise UnknownNodeError(f"node {node_id} not in graph")
            return pos
        # no host copy: binary search on the device (no O(E) transfer)
        x = self._as_id(node_id)
        pos = -1 if x is None else int(_native.graph_find(self.handle, [x])[0])
        if pos < 0:
            raise UnknownNodeError(f"node {node_id} not in graph")
        return pos

    def has_node(self, node_id: int) -> bool:
        if self._graph is not None:
            return self._graph.has_node(node_id)
        try:
            self._index(node_id)
            return True
        except UnknownNodeError:
            return False

    def record(self, node_id: int) -> NodeRecord:
        if self._graph is not None:
            return self._graph.record(node_id)
        i = self._index(node_id)
        h = self._host
        if h is None:  # one row each way from the device
            return NodeRecord(int(node_id),
                              in_nbrs=_frozen(_native.graph_row(self.handle, i, True)),
                              out_nbrs=_frozen(_native.graph_row(self.handle, i, False)))
        return NodeRecord(int(node_id), in_nbrs=h.in_adj[h.in_off[i]:h.in_off[i + 1]],
                          out_nbrs=h.out_adj[h.out_off[i]:h.out_off[i + 1]])

    def has_edge(self, src: int, dst: int) -> bool:
        if self._graph is not None or self._host is not None:
            return super().has_edge(src, dst)
        a, b = self._as_id(src), self._as_id(dst)
        if a is None or b is None:
            return False
        return _native.graph_has_edge(self.handle, a, b)

    def out_csr(self):
        if self._graph is not None:
            return self._graph.out_csr()
        h = self.csr()
        return h.ids, h.out_off, h.out_adj

    def memory_bytes(self) -> int:
        if self._graph is not None:
            return self._graph.memory_bytes()
        return 8 * self._n + 16 * (self._n + 1) + 8 * self._e  # ids, 2 offsets, 2 int32 adj

    def check_invariants(self) -> None:
        """Sortedness, in/out symmetry, edge-count identity (graphs.py:210-226)."""
        if self._graph is not None:
            return self._graph.check_invariants()
        h = self.csr()
        n, e = self._n, self._e
        assert h.out_off[0] == 0 and h.in_off[0] == 0
        assert h.out_off[-1] == e and h.in_off[-1] == e, "edge count != sum of degrees"
        for off, adj in ((h.out_off, h.out_adj), (h.in_off, h.in_adj)):
            assert np.all(np.diff(off) >= 0)
            if e > 1:
                row_start = np.zeros(e, dtype=bool)
                row_start[off[:-1][off[:-1] < e]] = True
                inc = adj[1:] > adj[:-1]  # no np.diff: int64 extremes overflow
                assert bool(np.all(inc | row_start[1:])), "unsorted adjacency vector"
        if n > 1:
            assert bool(np.all(h.ids[1:] > h.ids[:-1])), "node ids not strictly ascending"
        src = np.repeat(h.ids, np.diff(h.out_off))
        dst_of_in = np.repeat(h.ids, np.diff(h.in_off))
        a = np.lexsort((h.out_adj, src))
        b = np.lexsort((dst_of_in, h.in_adj))
        assert np.array_equal(src[a], h.in_adj[b]) and np.array_equal(h.out_adj[a],
                                                                      dst_of_in[b]), \
            "in/out adjacency are not mirror images"

    def _materialize(self) -> Graph:
        if self._graph is None:
            h = self.csr()
            g = Graph()
            ids = h.ids.tolist()
            for i, nid in enumerate(ids):
                g._nodes[nid] = NodeRecord(nid, in_nbrs=h.in_adj[h.in_off[i]:h.in_off[i + 1]],
                                           out_nbrs=h.out_adj[h.out_off[i]:h.out_off[i + 1]])
            g._edge_count = self._e
            self._graph = g
            self._finalizer()  # release the device CSR now
        return self._graph

    def apply_updates(self, add=None, delete=None, add_nodes=None, del_nodes=None) -> None:
        """Batched mutation on the device (gt_graph_update): the same result as
        the reference's calls (graphs.py:92-144) del_node(x) for x in
        del_nodes, del_edge(s, d) for (s, d) in delete, add_node(x) for x in
        add_nodes, add_edge(s, d) for (s, d) in add — in that order. ``add``
        and ``delete`` are (src ids, dst ids) pairs of equal-length arrays
        (host or device). The graph stays device-resident; a graph already
        mutated on the host applies the calls to its host records instead."""
        if self._graph is not None:
            g = self._graph
            for x in _as_list(del_nodes):
                g.del_node(x)
            for a, b in zip(*_pair_lists(delete)):
                g.del_edge(a, b)
            for x in _as_list(add_nodes):
                g.add_node(x)
            for a, b in zip(*_pair_lists(add)):
                g.add_edge(a, b)
            return
        import torch

        dev = torch.device("cuda", _native.device_ordinal())

        def col(a):
            if a is None:
                return torch.empty(0, dtype=torch.int64, device=dev)
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=torch.int64).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(dev)

        def pair(p):
            if p is None:
                return col(None), col(None)
            a, b = col(p[0]), col(p[1])
            if a.shape[0] != b.shape[0]:
                raise ValueError("src and dst arrays of an update differ in length")
            return a, b

        asrc, adst = pair(add)
        dsrc, ddst = pair(delete)
        an, dn = col(add_nodes), col(del_nodes)
        ptr = lambda t: t.data_ptr() if t.numel() else None  # noqa: E731
        new = _native.graph_update(self.handle, ptr(asrc), ptr(adst), asrc.shape[0],
                                   ptr(dsrc), ptr(ddst), dsrc.shape[0], ptr(an), an.shape[0],
                                   ptr(dn), dn.shape[0])
        self._finalizer()
        self._handle = new
        self._n, self._e = _native.graph_sizes(new)
        self._host = None
        self._ids = None
        self._finalizer = weakref.finalize(self, _native.graph_free, new)

    add_node = _mutating("add_node")
    add_edge = _mutating("add_edge")
    del_edge = _mutating("del_edge")
    del_node = _mutating("del_node")

    def subgraph(self, node_ids) -> Graph:
        if self._graph is not None:
            return self._graph.subgraph(node_ids)
        tmp = Graph()
        h = self.csr()
        for i, nid in enumerate(h.ids.tolist()):
            tmp._nodes[nid] = NodeRecord(nid, h.in_adj[h.in_off[i]:h.in_off[i + 1]],
                                         h.out_adj[h.out_off[i]:h.out_off[i + 1]])
        tmp._edge_count = self._e
        return tmp.subgraph(node_ids)

    def __repr__(self):
        where = "device" if self._graph is None else "host"
        return f"DeviceGraph(nodes={self.node_count}, edges={self.edge_count}, {where})"


def upload(g) -> DeviceGraph:
    """Device CSR of any graph exposing node_ids()/record() (isolated nodes kept)."""
    if isinstance(g, DeviceGraph) and g.on_device:
        return g
    ids, off, adj = _GraphReadAPI.out_csr(g)
    src = np.repeat(ids, np.diff(off))
    return DeviceGraph(_native.build_csr(src, adj, src.shape[0], False, nodes=ids))
