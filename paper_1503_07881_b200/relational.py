"""Device-resident Select / Project / Join feeding ToGraph.

Mirrors the reference's relational operators (``tables.py``): ``Predicate``
(:94-125), ``select`` (:325-344, with ``_check_predicate`` :313-322 and
``_take`` :232-240), ``project`` (:347-356), ``join`` (:397-426, with
``_suffixed_schema`` :359-364, ``_merge_pools`` :367-382, ``_paired_table``
:385-394) — same names, argument meaning, errors, output row order and row
ids. The row work runs in libgtb200 (``gt_select_rows``, ``gt_gather_u64``,
``gt_join_build``); host tables are moved to HBM first and results stay
there, ready for ``table_to_graph``. Only O(pool) string bookkeeping (pool
merge, string-ordering lookup tables) is done on the host. There is no CPU
fallback: without the library every call raises ``NativeError``.
"""

from __future__ import annotations

import math
import operator
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import SchemaError, TypeMismatchError
from .tables import FLOAT, INT, STRING, ColumnTable, Schema, _is_device

_OPS = {"=": 0, "!=": 1, "<": 2, "<=": 3, ">": 4, ">=": 5}
_PY_CMP = {"=": operator.eq, "!=": operator.ne, "<": operator.lt, "<=": operator.le,
           ">": operator.gt, ">=": operator.ge}
_I64_MIN, _I64_MAX = -(1 << 63), (1 << 63) - 1


@dataclass(frozen=True)
class Predicate:
    """Comparison of one column against a constant (tables.py:94-125)."""

    column: str
    op: str
    value: object

    def __post_init__(self):
        if self.op not in _OPS:
            raise ValueError(f"unknown comparison operator {self.op!r}")

    @classmethod
    def parse(cls, text: str, schema: Schema) -> "Predicate":
        """Parse 'Tag=Java' / 'age>=30' style predicates against a schema."""
        for op in ("<=", ">=", "!=", "=", "<", ">"):
            if op in text:
                col, _, raw = text.partition(op)
                col = col.strip()
                raw = raw.strip()
                typ = schema.type_of(col)
                if typ == INT:
                    value = int(raw)
                elif typ == FLOAT:
                    value = float(raw)
                else:
                    value = raw
                return cls(col, op, value)
        raise ValueError(f"no comparison operator found in {text!r}")


def _check_predicate(table: ColumnTable, pred: Predicate) -> str:
    typ = table.schema.type_of(pred.column)
    v = pred.value
    if typ == STRING and not isinstance(v, str):
        raise TypeMismatchError(
            f"predicate on string column {pred.column!r} needs a string, got {v!r}")
    if typ in (INT, FLOAT) and isinstance(v, (str, bool)):
        raise TypeMismatchError(
            f"predicate on numeric column {pred.column!r} needs a number, got {v!r}")
    return typ


# ---------------------------------------------------------------- device I/O --

def _torch():
    import torch

    return torch


def _device_of(*tables):
    for t in tables:
        for c in t.columns:
            if _is_device(c):
                return c.device
    _native.ensure_init()
    return _torch().device("cuda", _native.device_ordinal())


def _dev(col, typ, device):
    """The column as a contiguous 8-byte device tensor (int64 / float64)."""
    torch = _torch()
    dt = torch.float64 if typ == FLOAT else torch.int64
    if _is_device(col):
        t = col if isinstance(col, torch.Tensor) else torch.as_tensor(col, device=device)
        return t.to(device=device, dtype=dt).contiguous()
    arr = np.ascontiguousarray(col, dtype=np.float64 if typ == FLOAT else np.int64)
    return torch.from_numpy(arr).to(device)


def _gather(col, idx, n: int, remap=None):
    """col[idx] (idx None: identity) on the device, optionally through remap."""
    torch = _torch()
    out = torch.empty(max(n, 1), dtype=col.dtype, device=col.device)
    if n:
        _native.gather_u64(col.data_ptr(), None if idx is None else idx.data_ptr(), n,
                           None if remap is None else remap.data_ptr(), out.data_ptr())
    return out[:n]


# -------------------------------------------------------------------- select --

def _int_predicate(op: str, v):
    """(kind, op, ival) for an INT column against any numeric constant, with
    numpy's comparison results (non-integral, infinite, NaN, beyond-int64)."""
    all_rows = (0, _OPS[">="], _I64_MIN)
    no_rows = (2, _OPS["="], 0)  # empty lookup table: nothing matches
    if isinstance(v, float):
        if math.isnan(v):
            return all_rows if op == "!=" else no_rows
        if math.isinf(v):
            below = v > 0  # every int64 is below +inf
            if op == "!=" or (below and op in ("<", "<=")) or (not below and op in (">", ">=")):
                return all_rows
            return no_rows
        if not v.is_integer():
            if op == "=":
                return no_rows
            if op == "!=":
                return all_rows
            if op in ("<", "<="):
                return (0, _OPS["<="], math.floor(v)) if math.floor(v) <= _I64_MAX else all_rows
            return (0, _OPS[">="], math.ceil(v)) if math.ceil(v) >= _I64_MIN else all_rows
        v = int(v)
    v = int(v)
    if v > _I64_MAX:
        return all_rows if op in ("<", "<=", "!=") else no_rows
    if v < _I64_MIN:
        return all_rows if op in (">", ">=", "!=") else no_rows
    return (0, _OPS[op], v)


def select(table: ColumnTable, pred: Predicate, in_place: bool = False) -> ColumnTable:
    """Rows satisfying pred, ids and order preserved; optionally in place
    (tables.py:325-344). The result is device-resident."""
    typ = _check_predicate(table, pred)
    table._await_ready()
    torch = _torch()
    device = _device_of(table)
    n = table.n_rows
    col = _dev(table.column(pred.column), typ, device)
    lut = None
    fval = 0.0
    if typ == STRING:
        if pred.op in ("=", "!="):
            code = table.encode_value(pred.value)
            kind, op, ival = 0, _OPS[pred.op], -1 if code is None else code
        else:  # ordering comparisons go through the decoded strings (tables.py:339-341)
            cmp = _PY_CMP[pred.op]
            flags = np.fromiter((cmp(s, pred.value) for s in table.pool), dtype=np.uint8,
                                count=len(table.pool))
            lut = torch.from_numpy(flags).to(device) if flags.size else None
            kind, op, ival = 2, _OPS["="], 0
    elif typ == INT:
        kind, op, ival = _int_predicate(pred.op, pred.value)
    else:
        kind, op, ival, fval = 1, _OPS[pred.op], 0, float(pred.value)
    idx = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    lut_n = 0 if lut is None else int(lut.numel())
    m = _native.select_rows(col.data_ptr() if n else None, n, kind, op, ival, fval,
                            None if lut is None else lut.data_ptr(), lut_n, idx.data_ptr())
    sel = idx[:m]
    cols = [_gather(_dev(c, t, device), sel, m) for c, (_, t) in
            zip(table.columns, table.schema.columns)]
    ids = _gather(_dev(table.row_ids, INT, device), sel, m)
    if in_place:
        table.columns = cols
        table._row_ids = ids
        return table
    return ColumnTable(table.schema, cols, pool=table.pool, row_ids=ids,
                       next_row_id=table._next_row_id)


def project(table: ColumnTable, names) -> ColumnTable:
    """Restrict to the named columns in the given order; row ids preserved
    (tables.py:347-356)."""
    names = list(names)
    if not names:
        raise SchemaError("projection onto zero columns is not allowed")
    idxs = [table.schema.index_of(n) for n in names]
    schema = Schema([table.schema.columns[i] for i in idxs])
    return ColumnTable(schema, [table.columns[i] for i in idxs], pool=table.pool,
                       row_ids=table.row_ids, next_row_id=table._next_row_id)


# ---------------------------------------------------------------------- join --

def _suffixed_schema(left: Schema, right: Schema) -> Schema:
    """Concatenate schemas, suffixing colliding names by origin (-1 left, -2 right)."""
    collisions = set(left.names) & set(right.names)
    cols = [(f"{n}-1" if n in collisions else n, t) for n, t in left.columns]
    cols += [(f"{n}-2" if n in collisions else n, t) for n, t in right.columns]
    return Schema(cols)


def _merge_pools(left: ColumnTable, right: ColumnTable):
    """Combined pool plus the code remap of the right table's pool."""
    pool = list(left.pool)
    if not right.pool:
        return pool, np.empty(0, dtype=np.int64)
    index = {s: i for i, s in enumerate(pool)}
    remap = np.empty(len(right.pool), dtype=np.int64)
    for code, s in enumerate(right.pool):
        new = index.get(s)
        if new is None:
            new = index[s] = len(pool)
            pool.append(s)
        remap[code] = new
    return pool, remap


def join(left: ColumnTable, right: ColumnTable, left_col: str, right_col: str) -> ColumnTable:
    """Equi-join building on the smaller input (tables.py:397-426): left
    schema then right schema with collisions suffixed -1/-2, rows in probe
    order then build order, fresh row ids. The result is device-resident."""
    lt = left.schema.type_of(left_col)
    rt = right.schema.type_of(right_col)
    if lt != rt:
        raise TypeMismatchError(
            f"join columns {left_col!r} ({lt}) and {right_col!r} ({rt}) differ in type")
    left._await_ready()
    right._await_ready()
    torch = _torch()
    device = _device_of(left, right)
    schema = _suffixed_schema(left.schema, right.schema)
    pool, remap = _merge_pools(left, right)
    remap_d = torch.from_numpy(remap).to(device) if remap.size else None
    nl, nr = left.n_rows, right.n_rows
    lkeys = _dev(left.column(left_col), lt, device)
    rkeys = _dev(right.column(right_col), rt, device)
    if lt == STRING and remap_d is not None and nr:
        rkeys = _gather(rkeys, None, nr, remap_d)
    li, ri = _native.join_pairs(lkeys.data_ptr() if nl else None, nl,
                                rkeys.data_ptr() if nr else None, nr, 1 if lt == FLOAT else 0,
                                lambda k: torch.empty(max(k, 1), dtype=torch.int64,
                                                      device=device)[:k])
    m = int(li.shape[0])
    cols = [_gather(_dev(c, t, device), li, m) for c, (_, t) in
            zip(left.columns, left.schema.columns)]
    for c, (_, t) in zip(right.columns, right.schema.columns):
        rm = remap_d if (t == STRING and remap_d is not None) else None
        cols.append(_gather(_dev(c, t, device), ri, m, rm))
    return ColumnTable(schema, cols, pool=pool)
