"""ctypes binding of libgtb200.so (declared in include/gtb200.h).

The library is the only compute path: if it is missing or cannot initialise
a B200, every call raises :class:`NativeError` — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import CapacityError, NativeError

LIB_PATH = Path(__file__).resolve().parent / "libgtb200.so"
if os.environ.get("GT_LIB_VARIANT"):  # build-knob sweeps (scripts/sweep_*.sh) only
    LIB_PATH = LIB_PATH.with_name(f"libgtb200_{os.environ['GT_LIB_VARIANT']}.so")

GT_OK, GT_EINVAL, GT_ENOMEM, GT_ECUDA, GT_ENCCL, GT_ECAPACITY, GT_ENODEV = range(7)

# Every symbol include/gtb200.h declares, with its ctypes signature.
_I64P = ctypes.POINTER(ctypes.c_int64)
_VP = ctypes.c_void_p
SIGNATURES = {
    "gt_init": (ctypes.c_int, [ctypes.c_int]),
    "gt_version": (ctypes.c_char_p, []),
    "gt_stream": (_VP, []),
    "gt_last_error": (ctypes.c_char_p, []),
    "gt_set_lane": (ctypes.c_int, [ctypes.c_int]),
    "gt_release_workspace": (ctypes.c_int, []),
    "gt_build_csr": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int,
                                    ctypes.POINTER(_VP)]),
    "gt_build_csr_nodes": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP, ctypes.c_int64,
                                          ctypes.c_int, ctypes.POINTER(_VP)]),
    "gt_graph_sizes": (ctypes.c_int, [_VP, _I64P, _I64P]),
    "gt_graph_export": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "gt_graph_device_views": (ctypes.c_int, [_VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP),
                                             ctypes.POINTER(_VP), ctypes.POINTER(_VP),
                                             ctypes.POINTER(_VP)]),
    "gt_graph_free": (None, [_VP]),
    "gt_graph_find": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP]),
    "gt_graph_row": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int, _VP, ctypes.c_int64, _I64P]),
    "gt_graph_has_edge": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.POINTER(ctypes.c_int)]),
    "gt_pagerank": (ctypes.c_int, [_VP, ctypes.c_double, ctypes.c_int, _VP, ctypes.c_int]),
    "gt_graph_edge_table": (ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int]),
    "gt_tsv_count_lines": (ctypes.c_int, [_VP, ctypes.c_int64, _I64P]),
    "gt_tsv_parse_int64": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_void_p), _I64P, _I64P,
                                          ctypes.POINTER(ctypes.c_int),
                                          ctypes.POINTER(ctypes.c_int)]),
    "gt_graph_node_table": (ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int]),
    "gt_triangles": (ctypes.c_int, [_VP, _I64P]),
    "gt_triangle_orientation": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _I64P]),
    "gt_bfs": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, ctypes.c_int]),
    "gt_connected_components": (ctypes.c_int, [_VP, _VP, ctypes.c_int, _I64P]),
    "gt_kcore": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(_VP)]),
    "gt_scc": (ctypes.c_int, [_VP, _VP, ctypes.c_int, _I64P]),
    "gt_graph_update": (ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int64, _VP, _VP, ctypes.c_int64,
                                       _VP, ctypes.c_int64, _VP, ctypes.c_int64,
                                       ctypes.POINTER(_VP)]),
    "gt_rmat_generate": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                        ctypes.c_int, _VP, _VP]),
    "gt_rmat_generate_range": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_uint64, ctypes.c_int, _VP, _VP]),
    "gt_uniform_generate_range": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                 ctypes.c_uint64, _VP, _VP]),
    "gt_id_minmax": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP]),
    "gt_id_presence": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      _VP]),
    "gt_id_rankmap": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, _I64P]),
    "gt_id_list": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int64, _VP]),
    "gt_pack_keys": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int64, _VP, ctypes.c_int,
                                    _VP]),
    "gt_sort_keys": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int)]),
    "gt_unique_keys": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, _I64P]),
    "gt_merge_runs": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int)]),
    "gt_key_bucket_counts": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                            _VP]),
    "gt_key_lower_bounds": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, ctypes.c_int, _VP]),
    "gt_swap_key_halves": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int, _VP]),
    "gt_csr_from_keys": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_int64, _VP, _VP, _VP]),
    "gt_graph_from_csr": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _VP, _VP, _VP, _VP, _VP,
                                         ctypes.POINTER(_VP)]),
    "gt_inv_degree": (ctypes.c_int, [_VP, ctypes.c_int64, _VP]),
    "gt_remap_padded": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, ctypes.c_int, ctypes.c_int64,
                                       _VP]),
    "gt_pagerank_init": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, _VP]),
    "gt_pagerank_step": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        _VP, _VP, _VP, ctypes.c_double, ctypes.c_int, _VP, _VP,
                                        _VP]),
    "gt_triangles_part": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, _I64P]),
    "gt_tc_undirected_keys": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int, _VP, _I64P]),
    "gt_tc_degree_rank": (ctypes.c_int, [_VP, ctypes.c_int64, _VP]),
    "gt_tc_orient_keys": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int64, _VP,
                                         ctypes.c_int, _VP, _I64P]),
    "gt_triangles_oriented_part": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int64,
                                                  ctypes.c_int, ctypes.c_int, _I64P]),
    "gt_graph_undirected_edges": (ctypes.c_int, [_VP, _I64P]),
    "gt_select_rows": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int64, ctypes.c_double, _VP, ctypes.c_int64, _VP,
                                      _I64P]),
    "gt_gather_u64": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP, _VP]),
    "gt_join_build": (ctypes.c_int, [_VP, ctypes.c_int64, _VP, ctypes.c_int64, ctypes.c_int,
                                     ctypes.POINTER(_VP), _I64P]),
    "gt_join_export": (ctypes.c_int, [_VP, _VP, _VP]),
    "gt_join_free": (None, [_VP]),
    "gt_launch_count": (ctypes.c_int64, []),
    "gt_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "gt_profile_reset": (ctypes.c_int, []),
    "gt_profile_read": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                       ctypes.POINTER(ctypes.c_double), _I64P,
                                       ctypes.POINTER(ctypes.c_double)]),
}

_lib = None
_lock = threading.Lock()
_initialised = False


def load():
    """dlopen libgtb200.so and declare every entry point (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (the CUDA library is the only compute path)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def _raise(rc: int, what: str):
    msg = load().gt_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == GT_EINVAL:
        raise ValueError(text)
    if rc == GT_ECAPACITY:
        raise CapacityError(text)
    if rc == GT_ENOMEM:
        raise MemoryError(text)
    raise NativeError(text)


def check(rc: int, what: str):
    if rc != GT_OK:
        _raise(rc, what)


def device_ordinal() -> int:
    for var in ("GT_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var):
            return int(os.environ[var])
    return 0


def ensure_init():
    global _initialised
    lib = load()
    if not _initialised:
        check(lib.gt_init(device_ordinal()), "gt_init")
        _initialised = True
    order_after_torch()
    return lib


def order_after_torch():
    """Order the library stream after the caller's torch stream.

    The library's streams are blocking streams, so they already run after
    everything queued on torch's default (legacy) stream. When the caller
    works on another torch stream (``with torch.cuda.stream(s)``), make the
    library stream wait on it here, so that buffers written by torch ops are
    complete before a library kernel reads them. Called by every entry point
    (via ``ensure_init``)."""
    import sys

    torch = sys.modules.get("torch")
    if torch is None or not torch.cuda.is_initialized():
        return
    cur = torch.cuda.current_stream()
    if cur.cuda_stream == 0:
        return
    torch.cuda.ExternalStream(load().gt_stream(), device=cur.device).wait_stream(cur)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def build_csr(src, dst, rows: int, on_device: bool, nodes=None) -> int:
    """-> opaque gt_graph* (int). src/dst: device pointers or numpy int64."""
    lib = ensure_init()
    out = ctypes.c_void_p()
    if on_device:
        s, d = int(src), int(dst)
        keep = ()
    else:
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        s, d, keep = _ptr(src), _ptr(dst), (src, dst)
    if nodes is None:
        rc = lib.gt_build_csr(s, d, int(rows), int(on_device), ctypes.byref(out))
    else:
        if on_device:
            nptr, nn = int(nodes[0]), int(nodes[1])
        else:
            nodes = np.ascontiguousarray(nodes, dtype=np.int64)
            nptr, nn = _ptr(nodes), int(nodes.shape[0])
        rc = lib.gt_build_csr_nodes(s, d, int(rows), nptr, nn, int(on_device),
                                    ctypes.byref(out))
    del keep
    check(rc, "gt_build_csr")
    return int(out.value)


def graph_sizes(handle: int):
    n, e = ctypes.c_int64(), ctypes.c_int64()
    check(load().gt_graph_sizes(handle, ctypes.byref(n), ctypes.byref(e)), "gt_graph_sizes")
    return int(n.value), int(e.value)


def graph_export(handle: int, n: int, e: int):
    ids = np.empty(n, dtype=np.int64)
    out_off = np.empty(n + 1, dtype=np.int64)
    out_adj = np.empty(e, dtype=np.int64)
    in_off = np.empty(n + 1, dtype=np.int64)
    in_adj = np.empty(e, dtype=np.int64)
    check(load().gt_graph_export(handle, _ptr(ids), _ptr(out_off), _ptr(out_adj), _ptr(in_off),
                                 _ptr(in_adj)), "gt_graph_export")
    return ids, out_off, out_adj, in_off, in_adj


def graph_device_views(handle: int):
    ptrs = [ctypes.c_void_p() for _ in range(5)]
    check(load().gt_graph_device_views(handle, *[ctypes.byref(p) for p in ptrs]),
          "gt_graph_device_views")
    return [int(p.value or 0) for p in ptrs]


def graph_find(handle: int, node_ids) -> np.ndarray:
    """Dense index of each node id (-1 when absent), searched on the device."""
    lib = ensure_init()
    q = np.ascontiguousarray(node_ids, dtype=np.int64)
    out = np.empty(q.shape[0], dtype=np.int64)
    check(lib.gt_graph_find(handle, _ptr(q), q.shape[0], _ptr(out)), "gt_graph_find")
    return out


def graph_row(handle: int, index: int, in_side: bool) -> np.ndarray:
    """One adjacency row (original ids) copied from the device."""
    lib = ensure_init()
    n = ctypes.c_int64()
    check(lib.gt_graph_row(handle, int(index), int(in_side), None, 0, ctypes.byref(n)),
          "gt_graph_row")
    out = np.empty(n.value, dtype=np.int64)
    if n.value:
        check(lib.gt_graph_row(handle, int(index), int(in_side), _ptr(out), n.value,
                               ctypes.byref(n)), "gt_graph_row")
    return out


def graph_has_edge(handle: int, src: int, dst: int) -> bool:
    lib = ensure_init()
    r = ctypes.c_int()
    check(lib.gt_graph_has_edge(handle, int(src), int(dst), ctypes.byref(r)), "gt_graph_has_edge")
    return bool(r.value)


def graph_free(handle: int):
    if handle and _lib is not None:
        _lib.gt_graph_free(handle)


_PINNED_MAX = 1 << 30  # bytes; larger one-off outputs stay pageable


def host_empty(n: int, dtype) -> np.ndarray:
    """Uninitialised host array for a device->host result. Node-sized results
    (scores, ids) come from torch's caching pinned-host allocator: the copy
    runs at full link rate into pages that are already mapped, and the block
    returns to the cache when the array is freed (a pageable buffer costs a
    staging copy plus first-touch page faults: ~5 ms per 19 MB at C2)."""
    dtype = np.dtype(dtype)
    if 0 < n * dtype.itemsize <= _PINNED_MAX:
        try:
            import torch

            if torch.cuda.is_available():
                tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
                       np.dtype(np.int32): torch.int32}.get(dtype)
                if tdt is not None:
                    return torch.empty(n, dtype=tdt, pin_memory=True).numpy()
        except Exception:
            pass
    return np.empty(n, dtype=dtype)


def pagerank(handle: int, n: int, damping: float, iterations: int, out_ptr: int | None = None):
    lib = ensure_init()
    if out_ptr is not None:
        check(lib.gt_pagerank(handle, float(damping), int(iterations), int(out_ptr), 1),
              "gt_pagerank")
        return None
    scores = host_empty(n, np.float64)
    check(lib.gt_pagerank(handle, float(damping), int(iterations), _ptr(scores), 0),
          "gt_pagerank")
    return scores


def triangles(handle: int) -> int:
    lib = ensure_init()
    c = ctypes.c_int64()
    check(lib.gt_triangles(handle, ctypes.byref(c)), "gt_triangles")
    return int(c.value)


def undirected_edges(handle: int) -> int:
    """m of the last triangle count on this graph (-1 before the first)."""
    m = ctypes.c_int64()
    check(load().gt_graph_undirected_edges(handle, ctypes.byref(m)), "gt_graph_undirected_edges")
    return int(m.value)


def bfs(handle: int, n: int, source_index: int) -> np.ndarray:
    """-> dist[N] int32 (-1 = unreachable)."""
    lib = ensure_init()
    dist = host_empty(n, np.int32)
    check(lib.gt_bfs(handle, int(source_index), _ptr(dist), 0), "gt_bfs")
    return dist


def connected_components(handle: int, n: int):
    """-> (labels[N] int64, number of components)."""
    lib = ensure_init()
    labels = host_empty(n, np.int64)
    count = ctypes.c_int64()
    check(lib.gt_connected_components(handle, _ptr(labels) if n else None, 0, ctypes.byref(count)),
          "gt_connected_components")
    return labels, int(count.value)


def scc(handle: int, n: int):
    """-> (labels[N] int64, number of strongly connected components)."""
    lib = ensure_init()
    labels = host_empty(n, np.int64)
    count = ctypes.c_int64()
    check(lib.gt_scc(handle, _ptr(labels) if n else None, 0, ctypes.byref(count)), "gt_scc")
    return labels, int(count.value)


def graph_update(handle: int, add_src, add_dst, n_add: int, del_src, del_dst, n_del: int,
                 add_nodes, n_add_nodes: int, del_nodes, n_del_nodes: int) -> int:
    """Device pointers in -> handle of the updated graph (caller owns it)."""
    lib = ensure_init()
    out = _VP()
    check(lib.gt_graph_update(handle, add_src, add_dst, int(n_add), del_src, del_dst, int(n_del),
                              add_nodes, int(n_add_nodes), del_nodes, int(n_del_nodes),
                              ctypes.byref(out)), "gt_graph_update")
    return out.value or 0


def kcore(handle: int, k: int) -> int:
    """-> handle of the k-core graph (caller owns it)."""
    lib = ensure_init()
    out = _VP()
    check(lib.gt_kcore(handle, int(k), ctypes.byref(out)), "gt_kcore")
    return out.value or 0


def triangle_orientation(handle: int, n: int):
    """-> (deg[N], rank[N], off_p[N+1], adj_p[m]): the rank-space orientation."""
    lib = ensure_init()
    m = ctypes.c_int64()
    deg = np.empty(n, dtype=np.int32)
    rank = np.empty(n, dtype=np.int32)
    off_p = np.empty(n + 1, dtype=np.int64)
    check(lib.gt_triangle_orientation(handle, _ptr(deg), _ptr(rank), _ptr(off_p), None,
                                      ctypes.byref(m)), "gt_triangle_orientation")
    adj_p = np.empty(int(m.value), dtype=np.int32)
    check(lib.gt_triangle_orientation(handle, None, None, None, _ptr(adj_p), ctypes.byref(m)),
          "gt_triangle_orientation")
    return deg, rank, off_p, adj_p


def select_rows(col_ptr: int, n: int, kind: int, op: int, ival: int, fval: float,
                lut_ptr: int | None, lut_n: int, out_ptr: int) -> int:
    """Device select -> number of selected rows (indices written to out_ptr)."""
    lib = ensure_init()
    m = ctypes.c_int64()
    check(lib.gt_select_rows(col_ptr or None, int(n), int(kind), int(op), int(ival), float(fval),
                             lut_ptr or None, int(lut_n), out_ptr or None, ctypes.byref(m)),
          "gt_select_rows")
    return int(m.value)


def gather_u64(src_ptr: int, idx_ptr: int | None, n: int, remap_ptr: int | None,
               out_ptr: int) -> None:
    lib = ensure_init()
    check(lib.gt_gather_u64(src_ptr or None, idx_ptr or None, int(n), remap_ptr or None,
                            out_ptr or None), "gt_gather_u64")


def join_pairs(left_ptr: int, nl: int, right_ptr: int, nr: int, kind: int, alloc):
    """Device equi-join -> (left rows, right rows) as two int64 device buffers
    obtained from ``alloc(n)``."""
    lib = ensure_init()
    h = _VP()
    m = ctypes.c_int64()
    check(lib.gt_join_build(left_ptr or None, int(nl), right_ptr or None, int(nr), int(kind),
                            ctypes.byref(h), ctypes.byref(m)), "gt_join_build")
    try:
        n = int(m.value)
        li, ri = alloc(n), alloc(n)
        check(lib.gt_join_export(h, li.data_ptr() if n else None, ri.data_ptr() if n else None),
              "gt_join_export")
        return li, ri
    finally:
        lib.gt_join_free(h)


def graph_edge_table(handle: int, src, dst, on_device: bool):
    lib = ensure_init()
    if on_device:
        check(lib.gt_graph_edge_table(handle, int(src), int(dst), 1), "gt_graph_edge_table")
    else:
        check(lib.gt_graph_edge_table(handle, _ptr(src), _ptr(dst), 0), "gt_graph_edge_table")


def graph_node_table(handle: int, node, out_deg, in_deg):
    lib = ensure_init()
    check(lib.gt_graph_node_table(handle, _ptr(node), _ptr(out_deg), _ptr(in_deg), 0),
          "gt_graph_node_table")


def uniform_generate(n_nodes, rows, seed, src_ptr, dst_ptr, start=0):
    lib = ensure_init()
    check(lib.gt_uniform_generate_range(int(n_nodes), int(start), int(rows), int(seed),
                                        int(src_ptr), int(dst_ptr)), "gt_uniform_generate_range")


def rmat_generate(scale, rows, a, b, c, seed, permute, src_ptr, dst_ptr, start=0):
    lib = ensure_init()
    check(lib.gt_rmat_generate_range(int(scale), int(start), int(rows), float(a), float(b),
                                     float(c), int(seed) & ((1 << 64) - 1), int(bool(permute)),
                                     int(src_ptr), int(dst_ptr)), "gt_rmat_generate_range")


_LANE_POOLS: dict = {}


def lane_submit(lane: int, fn, *args, **kwargs):
    """Run fn(*args, **kwargs) on a worker thread bound to library lane `lane`
    (its own stream and workspace): independent calls on one graph overlap on
    the GPU. Returns a concurrent.futures.Future."""
    from concurrent.futures import ThreadPoolExecutor

    ensure_init()
    pool = _LANE_POOLS.get(lane)
    if pool is None:
        def bind():
            check(load().gt_set_lane(int(lane)), "gt_set_lane")

        pool = _LANE_POOLS[lane] = ThreadPoolExecutor(1, initializer=bind)
    return pool.submit(fn, *args, **kwargs)


def stream_handle() -> int:
    return int(ensure_init().gt_stream() or 0)


def launch_count() -> int:
    return int(load().gt_launch_count())


def profile_enable(on: bool = True):
    ensure_init().gt_profile_enable(int(on))


def profile_reset():
    check(load().gt_profile_reset(), "gt_profile_reset")


def profile_read():
    """-> {phase: (total_ms, launches, algorithmic_bytes)}"""
    lib = load()
    cap = 64
    names = (ctypes.c_char_p * cap)()
    ms = (ctypes.c_double * cap)()
    launches = (ctypes.c_int64 * cap)()
    nbytes = (ctypes.c_double * cap)()
    k = lib.gt_profile_read(cap, names, ms, launches, nbytes)
    if k < 0:
        _raise(-k, "gt_profile_read")
    return {names[i].decode(): (ms[i], int(launches[i]), nbytes[i]) for i in range(min(k, cap))}
