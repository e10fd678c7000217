"""Column tables for the ToGraph path: schema-typed int64 columns that can
live in host memory (numpy) or in HBM (torch CUDA tensors).

Mirrors the parts of the reference's ``tables.py`` the path touches:
``Schema`` (tables.py:44-90, incl. ``parse``), ``ColumnTable.column`` /
``n_rows`` (tables.py:128-186) and ``load_tsv`` (tables.py:246-284: headerless
UTF-8 TSV, exact field count, ``ParseError`` carrying line and column).
``ColumnTable.to_device()`` is new: it makes the int columns device-resident
once, so every later ToGraph reads them straight from HBM.
"""

from __future__ import annotations

import numpy as np

from .errors import ParseError, SchemaError, TypeMismatchError, UnknownColumnError

INT, FLOAT, STRING = "int", "float", "str"
_TYPES = (INT, FLOAT, STRING)


class Schema:
    """Ordered (name, type) pairs; types are int, float or str."""

    def __init__(self, columns):
        cols = [(str(n), t) for n, t in columns]
        if not cols:
            raise SchemaError("schema must have at least one column")
        names = [n for n, _ in cols]
        if len(set(names)) != len(names):
            raise SchemaError(f"duplicate column names in {names}")
        for name, typ in cols:
            if not name:
                raise SchemaError("column names must be non-empty")
            if typ not in _TYPES:
                raise SchemaError(f"unknown column type {typ!r} for {name!r}")
        self.columns = cols
        self._index = {n: i for i, n in enumerate(names)}

    def __len__(self):
        return len(self.columns)

    def __eq__(self, other):
        return isinstance(other, Schema) and self.columns == other.columns

    def __repr__(self):
        return "Schema(%s)" % ", ".join(f"{n}:{t}" for n, t in self.columns)

    @property
    def names(self):
        return [n for n, _ in self.columns]

    def index_of(self, name: str) -> int:
        try:
            return self._index[name]
        except KeyError:
            raise UnknownColumnError(f"no column named {name!r} (have {self.names})") from None

    def type_of(self, name: str) -> str:
        return self.columns[self.index_of(name)][1]

    @classmethod
    def parse(cls, text: str) -> "Schema":
        """'src:int,dst:int' -> Schema."""
        cols = []
        for part in text.split(","):
            name, _, typ = part.partition(":")
            cols.append((name.strip(), typ.strip()))
        return cls(cols)


def _is_device(col) -> bool:
    return getattr(col, "is_cuda", False) or hasattr(col, "__cuda_array_interface__")


def _length(col) -> int:
    return int(col.shape[0])


class ColumnTable:
    """Schema-typed columns of equal length (host numpy or device tensors);
    every row carries a persistent id (tables.py:136-150): fresh tables
    number their rows 0..n-1, ``select`` keeps the ids of the surviving rows."""

    def __init__(self, schema: Schema, columns, pool=None, row_ids=None, next_row_id=None):
        if len(columns) != len(schema):
            raise SchemaError("column count does not match schema")
        cols = [c if _is_device(c) else np.asarray(c) for c in columns]
        lengths = {_length(c) for c in cols}
        if len(lengths) > 1:
            raise SchemaError(f"ragged column lengths {sorted(lengths)}")
        self.schema = schema
        self.columns = cols
        self.pool = pool if pool is not None else []
        self._pool_index = None
        n = _length(cols[0]) if cols else 0
        if row_ids is not None and _length(row_ids) != n:
            raise SchemaError("row_ids length does not match the columns")
        self._row_ids = row_ids
        self._ready = None  # pending prefetch (event, device tensors)
        if next_row_id is None:
            next_row_id = n if row_ids is None else (int(row_ids.max()) + 1 if n else 0)
        self._next_row_id = int(next_row_id)

    @classmethod
    def from_rows(cls, schema: Schema, rows) -> "ColumnTable":
        """Table from python row tuples, strings given decoded and pooled by
        first occurrence (tables.py:158-178)."""
        pool: list[str] = []
        index: dict[str, int] = {}
        cols = []
        for j, (_, typ) in enumerate(schema.columns):
            vals = [r[j] for r in rows]
            if typ == STRING:
                codes = np.empty(len(vals), dtype=np.int64)
                for i, v in enumerate(vals):
                    code = index.get(v)
                    if code is None:
                        code = index[v] = len(pool)
                        pool.append(v)
                    codes[i] = code
                cols.append(codes)
            else:
                cols.append(np.asarray(vals, dtype=np.float64 if typ == FLOAT else np.int64))
        return cls(schema, cols, pool=pool)

    @property
    def row_ids(self):
        """Persistent row ids (int64, same residency as the first column)."""
        if self._row_ids is None:
            n = self.n_rows
            if self.columns and _is_device(self.columns[0]):
                import torch

                self._row_ids = torch.arange(n, dtype=torch.int64, device=self.columns[0].device)
            else:
                self._row_ids = np.arange(n, dtype=np.int64)
        return self._row_ids

    def decoded(self, name: str):
        """Host column values with string codes decoded through the pool
        (tables.py:193-199)."""
        idx = self.schema.index_of(name)
        col = self.columns[idx]
        col = col.cpu().numpy() if _is_device(col) else col
        if self.schema.columns[idx][1] == STRING:
            return (np.asarray(self.pool, dtype=object)[col] if col.size
                    else np.empty(0, dtype=object))
        return col

    def encode_value(self, value: str):
        """Pool code of a string, or None when it is not pooled (tables.py:201-205)."""
        if self._pool_index is None:
            self._pool_index = {v: i for i, v in enumerate(self.pool)}
        return self._pool_index.get(value)

    def cell_equal(self, other: "ColumnTable") -> bool:
        """Same schema and decoded cells row by row, row ids ignored (tables.py:219-223)."""
        return (self.schema == other.schema and self.n_rows == other.n_rows
                and self.to_rows() == other.to_rows())

    @property
    def n_rows(self) -> int:
        return _length(self.columns[0]) if self.columns else 0

    def column(self, name: str):
        return self.columns[self.schema.index_of(name)]

    def is_device_resident(self, name: str) -> bool:
        return _is_device(self.column(name))

    def to_device(self, device="cuda", all_columns=False) -> "ColumnTable":
        """Copy of the table whose int columns (every column with
        ``all_columns``: str codes as int64, floats as float64) live in HBM."""
        import torch

        cols = []
        for (name, typ), col in zip(self.schema.columns, self.columns):
            if (typ == INT or all_columns) and not _is_device(col):
                dt = np.float64 if typ == FLOAT else np.int64
                col = torch.from_numpy(np.ascontiguousarray(col, dtype=dt)).to(device)
            cols.append(col)
        ids = self._row_ids
        if ids is not None and all_columns and not _is_device(ids):
            ids = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64)).to(device)
        return ColumnTable(self.schema, cols, pool=self.pool, row_ids=ids,
                           next_row_id=self._next_row_id)

    def prefetch(self, device=None) -> "ColumnTable":
        """Device-resident copy of the table whose host→device transfer runs on
        a side stream and returns at once. The library waits for the copy only
        when a call first uses the table (``_await_ready``), so a copy issued
        while the library is busy overlaps that work (pipelined ingest of a
        stream of tables). Host columns should be pinned for the copy to be
        asynchronous; str codes travel as int64, floats as float64. The copy
        engine's writes go through L2 and evict what kernels running meanwhile
        keep there: measured on B200 at C4, issuing the next table's copy at
        the start of a step (under the build and PageRank) costs ~1 %, issuing
        it under the triangle count ~20 % of the count
        (scripts/probe_e2e.py, profiles/r2_e2e_probe.txt)."""
        import torch

        from . import _native

        dev = torch.device("cuda", _native.device_ordinal()) if device is None \
            else torch.device(device)
        side = _copy_stream(dev)
        cols = []
        with torch.cuda.stream(side):
            for (_, typ), col in zip(self.schema.columns, self.columns):
                if _is_device(col):
                    cols.append(col)
                    continue
                dt = np.float64 if typ == FLOAT else np.int64
                t = col if isinstance(col, torch.Tensor) else \
                    torch.from_numpy(np.ascontiguousarray(col, dtype=dt))
                cols.append(t.to(dev, non_blocking=True))
        ev = torch.cuda.Event()
        ev.record(side)
        out = ColumnTable(self.schema, cols, pool=self.pool, row_ids=None,
                          next_row_id=self._next_row_id)
        if self._row_ids is not None:
            out._row_ids = self._row_ids
        out._ready = (ev, [c for c in cols if c.device == dev])
        return out

    def _await_ready(self) -> None:
        """Make the library stream wait for a pending prefetch of this table."""
        ready = getattr(self, "_ready", None)
        if ready is None:
            return
        import torch

        from . import _native

        ev, tensors = ready
        dev = tensors[0].device if tensors else torch.device("cuda", _native.device_ordinal())
        lib = torch.cuda.ExternalStream(_native.stream_handle(), device=dev)
        lib.wait_event(ev)
        for t in tensors:
            t.record_stream(lib)
        self._ready = None

    def to_host(self) -> "ColumnTable":
        cols = [c.cpu().numpy() if _is_device(c) else c for c in self.columns]
        ids = self._row_ids
        if ids is not None and _is_device(ids):
            ids = ids.cpu().numpy()
        return ColumnTable(self.schema, cols, pool=self.pool, row_ids=ids,
                           next_row_id=self._next_row_id)

    def to_rows(self) -> list[tuple]:
        host = self.to_host()
        out = []
        for i in range(self.n_rows):
            row = []
            for (_, typ), col in zip(self.schema.columns, host.columns):
                v = col[i]
                row.append(self.pool[int(v)] if typ == STRING else
                           (int(v) if typ == INT else float(v)))
            out.append(tuple(row))
        return out

    def memory_bytes(self) -> int:
        return int(sum(c.nbytes if hasattr(c, "nbytes") else c.element_size() * c.numel()
                       for c in self.columns))

    def __repr__(self):
        return f"ColumnTable({self.schema!r}, rows={self.n_rows})"


_COPY_STREAMS: dict = {}


def _copy_stream(dev):
    import torch

    key = str(dev)
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[key]


def load_tsv(path, schema: Schema, device=None) -> ColumnTable:
    """Headerless TSV, one row per line, fields per schema (tables.py:246-284).

    ``device="cuda"`` parses an all-int ASCII file on the GPU (gt_tsv_parse_int64,
    SURVEY §8f next #2) and returns HBM-resident columns — the same values and
    the same ParseError / OverflowError as the host parser, which stays the
    default (``device=None``) and handles str / float columns and non-ASCII
    text."""
    if device is not None:
        return _load_tsv_device(path, schema, device)
    return _load_tsv_host(path, schema)


def load_tsv_frontend(path, schema: Schema) -> ColumnTable:
    """LoadTableTSV's ingest (front-end __init__.py:126-128 -> tables.py:246-284):
    all-int schemas of ASCII text are parsed on the GPU into HBM-resident
    columns (the hot path's input: ToGraph, Select, Join read them in place);
    str / float columns and non-ASCII text keep the host parser, which is the
    reference's own semantics for those types (Python int()/float() on
    Unicode, string pools). Values and errors are identical either way
    (tests/test_tsv_gpu.py, goldens of the real reference in tsv.npz)."""
    from . import _native

    if all(t == INT for _, t in schema.columns) and len(schema.columns) <= 16:
        try:
            import torch

            cuda = torch.cuda.is_available()
        except Exception:  # pragma: no cover - torch is a hard dependency
            cuda = False
        if cuda:
            try:
                return _load_tsv_device(path, schema, f"cuda:{_native.device_ordinal()}")
            except TypeMismatchError:
                pass  # non-ASCII text: Python int() semantics on Unicode digits
    return _load_tsv_host(path, schema)


def _line_bounds(data: np.ndarray, k: int):
    """Byte range of the k-th line (0-based) under universal newlines."""
    nl = data == 10
    cr = data == 13
    lf_after = np.zeros_like(cr)
    lf_after[:-1] = nl[1:]
    ends = np.flatnonzero(nl | (cr & ~lf_after))
    start = 0 if k == 0 else int(ends[k - 1]) + 1
    end = int(ends[k]) if k < ends.shape[0] else data.shape[0]
    if end > start and end < data.shape[0] and data[end] == 10 and data[end - 1] == 13:
        end -= 1
    return start, end


def _load_tsv_device(path, schema: Schema, device) -> ColumnTable:
    import ctypes

    import torch

    from . import _native

    types = [t for _, t in schema.columns]
    data = np.fromfile(path, dtype=np.uint8)
    if any(t != INT for t in types) or len(types) > 16 or (data.size and data.max() >= 0x80):
        raise TypeMismatchError("device TSV ingest takes all-int schemas (<= 16 columns) of "
                                "ASCII text; use device=None for the host parser")
    dev = torch.device(device)
    buf = torch.from_numpy(data).to(dev) if data.size else torch.empty(1, dtype=torch.uint8,
                                                                        device=dev)
    lib = _native.ensure_init()
    n_lines = ctypes.c_int64()
    _native.check(lib.gt_tsv_count_lines(buf.data_ptr(), data.size, ctypes.byref(n_lines)),
                  "gt_tsv_count_lines")
    n = int(n_lines.value)
    cols = [torch.empty(max(n, 1), dtype=torch.int64, device=dev) for _ in types]
    ptrs = (ctypes.c_void_p * len(cols))(*[c.data_ptr() for c in cols])
    err_line, err_col, overflow = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
    _native.check(lib.gt_tsv_parse_int64(buf.data_ptr(), data.size, len(cols), ptrs,
                                         ctypes.byref(n_lines), ctypes.byref(err_line),
                                         ctypes.byref(err_col), ctypes.byref(overflow)),
                  "gt_tsv_parse_int64")
    if err_line.value >= 0:
        lineno = int(err_line.value) + 1
        a, b = _line_bounds(data, int(err_line.value))
        fields = data[a:b].tobytes().decode("ascii").split("\t")
        if err_col.value < 0:
            raise ParseError(f"line {lineno}: expected {len(types)} fields, got {len(fields)}",
                             line=lineno)
        name = schema.columns[err_col.value][0]
        raise ParseError(f"line {lineno}, column {name!r}: {fields[err_col.value]!r} is not "
                         "an integer", line=lineno, column=name)
    if overflow.value:
        raise OverflowError("Python int too large to convert to C long")
    return ColumnTable(schema, [c[:n] for c in cols])


def _load_tsv_host(path, schema: Schema) -> ColumnTable:
    n_cols = len(schema)
    raw = [[] for _ in range(n_cols)]
    pool: list[str] = []
    codes: dict[str, int] = {}
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            fields = line.rstrip("\n").split("\t")
            if len(fields) != n_cols:
                raise ParseError(f"line {lineno}: expected {n_cols} fields, got {len(fields)}",
                                 line=lineno)
            for j, (name, typ) in enumerate(schema.columns):
                field = fields[j]
                if typ == STRING:
                    code = codes.get(field)
                    if code is None:
                        code = codes[field] = len(pool)
                        pool.append(field)
                    raw[j].append(code)
                    continue
                conv = int if typ == INT else float
                try:
                    raw[j].append(conv(field))
                except ValueError:
                    kind = "an integer" if typ == INT else "a float"
                    raise ParseError(f"line {lineno}, column {name!r}: {field!r} is not {kind}",
                                     line=lineno, column=name) from None
    arrays = [np.asarray(raw[j], dtype=np.float64 if t == FLOAT else np.int64)
              for j, (_, t) in enumerate(schema.columns)]
    return ColumnTable(schema, arrays, pool=pool)


def save_tsv(table: ColumnTable, path) -> None:
    """Inverse of load_tsv for int/float/str columns."""
    rows = table.to_rows()
    with open(path, "w", encoding="utf-8") as fh:
        for row in rows:
            parts = []
            for v, (_, typ) in zip(row, table.schema.columns):
                if typ == STRING and ("\t" in v or "\n" in v):
                    raise TypeMismatchError(f"string value {v!r} contains a tab or newline")
                parts.append(repr(v) if typ == FLOAT else str(v))
            fh.write("\t".join(parts) + "\n")


def edge_table(src, dst, names=("src", "dst")) -> ColumnTable:
    """Two-int-column edge table from arrays (host or device)."""
    return ColumnTable(Schema([(names[0], INT), (names[1], INT)]), [src, dst])


def table_from_map(pairs, key_name: str, val_name: str) -> ColumnTable:
    """Two-column (int key, float value) table sorted ascending by key
    (tables.py:662-670). A PageRank ``RankMap`` is already (ids ascending,
    scores): its arrays become the columns without a Python pass."""
    schema = Schema([(key_name, INT), (val_name, FLOAT)])
    ids = getattr(pairs, "ids", None)
    if ids is not None and hasattr(pairs, "scores"):
        return ColumnTable(schema, [np.asarray(ids, dtype=np.int64).copy(),
                                    np.asarray(pairs.scores, dtype=np.float64).copy()])
    items = sorted((int(k), float(v)) for k, v in pairs.items())
    if not items:
        return ColumnTable(schema, [np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float64)])
    keys, vals = zip(*items)
    return ColumnTable(schema, [np.asarray(keys, dtype=np.int64),
                                np.asarray(vals, dtype=np.float64)])
