"""ToGraph: edge table -> DeviceGraph through libgtb200 (gt_build_csr).

Drop-in for ``graphtables.convert.table_to_graph`` (convert.py:128-175) and
``EdgeSpec`` (convert.py:30-42): same signature, same validation and errors,
same result (node set = distinct ids of both columns, duplicates collapse,
self-loops kept, out-vectors sorted by (src, dst), in-vectors by (dst, src)),
built on the GPU by a sort-first radix pipeline.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import TypeMismatchError
from .graph import DeviceGraph
from .tables import INT

_INT_TYPES = (INT,)


def resolve_workers(workers):
    """parallel.py:22-28 contract: None or >= 1 (the GPU ignores the count)."""
    if workers is not None and workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    return workers


@dataclass(frozen=True)
class EdgeSpec:
    """Names of the edge source and destination columns."""

    src_col: str
    dst_col: str

    def validate(self, table) -> None:
        for name in (self.src_col, self.dst_col):
            typ = table.schema.type_of(name)  # UnknownColumnError if absent
            if typ not in _INT_TYPES:
                raise TypeMismatchError(
                    f"edge column {name!r} must be integer-typed, got {typ}")


def _device_ptr(col):
    if getattr(col, "is_cuda", False):
        import torch

        if col.dtype != torch.int64:
            col = col.to(torch.int64)
        col = col.contiguous()
        return col, col.data_ptr()
    iface = getattr(col, "__cuda_array_interface__", None)
    if iface is not None:
        if np.dtype(iface["typestr"]) != np.int64 or iface.get("strides") not in (None, (8,)):
            raise TypeMismatchError("device edge columns must be contiguous int64")
        return col, int(iface["data"][0])
    return None, None


def table_to_graph(table, spec: EdgeSpec, workers: int | None = None) -> DeviceGraph:
    """Build the directed simple graph of an edge table on the GPU.

    Accepts this package's ColumnTable (host or device-resident columns) or
    any object with ``schema.type_of`` and ``column`` — the reference's own
    ColumnTable included. Input columns are never written.
    """
    spec.validate(table)
    resolve_workers(workers)
    if hasattr(table, "_await_ready"):
        table._await_ready()
    src = table.column(spec.src_col)
    dst = table.column(spec.dst_col)
    s_keep, s_ptr = _device_ptr(src)
    d_keep, d_ptr = _device_ptr(dst)
    rows = int(src.shape[0])
    if s_ptr is not None and d_ptr is not None:
        handle = _native.build_csr(s_ptr, d_ptr, rows, True)
        del s_keep, d_keep
    else:
        if s_ptr is not None:
            src = src.cpu().numpy()
        if d_ptr is not None:
            dst = dst.cpu().numpy()
        handle = _native.build_csr(np.asarray(src), np.asarray(dst), rows, False)
    return DeviceGraph(handle)


# ------------------------------------------------------------ graph -> table
# the step after the path in the paper's workflow
# (demo.py:45-46). Device kernels in libgtb200 (gt_graph_edge_table /
# gt_graph_node_table); host graphs are uploaded first.

def graph_to_edge_table(g, workers: int | None = None, device: bool = False):
    """Edges as a two-column table sorted by (src, dst) (convert.py:178-197).

    ``device=True`` leaves the columns in HBM (torch tensors)."""
    from .graph import upload
    from .tables import ColumnTable, Schema

    resolve_workers(workers)
    dg = upload(g)
    e = dg.edge_count
    schema = Schema([("src", INT), ("dst", INT)])
    if device:
        import torch

        src = torch.empty(e, dtype=torch.int64, device="cuda")
        dst = torch.empty(e, dtype=torch.int64, device="cuda")
        _native.graph_edge_table(dg.handle, src.data_ptr(), dst.data_ptr(), True)
    else:
        src = np.empty(e, dtype=np.int64)
        dst = np.empty(e, dtype=np.int64)
        _native.graph_edge_table(dg.handle, src, dst, False)
    return ColumnTable(schema, [src, dst])


def graph_to_node_table(g, values=None, value_name: str = "value"):
    """Per-node table (node, out_deg, in_deg[, value]), ascending by id
    (convert.py:200-217); ``values`` must cover exactly the node set
    (CoverageError otherwise)."""
    from .errors import CoverageError
    from .graph import upload
    from .tables import FLOAT, ColumnTable, Schema

    dg = upload(g)
    n = dg.node_count
    node = np.empty(n, dtype=np.int64)
    out_deg = np.empty(n, dtype=np.int64)
    in_deg = np.empty(n, dtype=np.int64)
    _native.graph_node_table(dg.handle, node, out_deg, in_deg)
    cols = [node, out_deg, in_deg]
    schema_cols = [("node", INT), ("out_deg", INT), ("in_deg", INT)]
    if values is not None:
        vals = _values_in_id_order(values, node)
        if vals is None:
            raise CoverageError(
                "values mapping must cover exactly the node set "
                f"({len(values)} values for {n} nodes)")
        cols.append(vals)
        schema_cols.append((value_name, FLOAT))
    return ColumnTable(Schema(schema_cols), cols)


def _values_in_id_order(values, node):
    """float64 values aligned with `node` (ascending ids), or None when the
    key set differs from the node set."""
    ids = getattr(values, "ids", None)
    if ids is not None and hasattr(values, "scores"):  # RankMap: already (ids, scores)
        if np.array_equal(np.asarray(ids), node):
            return np.asarray(values.scores, dtype=np.float64)
        return None
    if len(values) != node.shape[0]:
        return None
    try:
        return np.asarray([float(values[int(i)]) for i in node.tolist()], dtype=np.float64)
    except KeyError:
        return None
