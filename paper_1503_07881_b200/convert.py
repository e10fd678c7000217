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
