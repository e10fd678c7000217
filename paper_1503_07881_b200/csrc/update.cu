// update.cu — batched dynamic updates of a device graph.
//
// The reference mutates its Graph one call at a time (graphs.py:92-144):
// add_node, add_edge (creates endpoints, ignores present edges), del_edge
// (nodes stay), del_node (drops the node and every incident edge). A batch
// here is defined as those calls in this order:
//     del_node(x) for x in del_nodes; del_edge(s, d) for (s, d) in deletions;
//     add_node(x) for x in add_nodes; add_edge(s, d) for (s, d) in additions
// and is applied on the device:
//   1. dead[N]: deleted node ids located by binary search in ids
//   2. gone[E]: deleted edges located by binary search (row of s, then d in
//      the sorted out-row)
//   3. warp per row: keep flag of every edge (row alive, edge not gone,
//      destination alive)
//   4. stream compaction of the kept (src id, dst id) pairs and of the live
//      node ids, additions appended
//   5. gt_build_csr's pipeline on the result (sort, dedupe, both CSRs), with
//      the live node ids and add_nodes as extra nodes so isolated nodes stay.
// Cost: one pass over the old CSR plus a build — HBM-rate batch updates
// instead of per-edge sorted-vector inserts.
#include "graph.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"

#include <algorithm>
#include <string>

namespace gt {
gt_graph* build_csr(const int64_t* src, const int64_t* dst, int64_t rows, const int64_t* extra,
                    int64_t n_extra, bool on_device);
}

namespace gtd {

constexpr int UP_TILE = 2048;  // 256 threads x 8

__device__ __forceinline__ int64_t up_find(const int64_t* __restrict__ ids, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ids[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && ids[lo] == x ? lo : -1;
}

__global__ void __launch_bounds__(256) up_dead_kernel(const int64_t* __restrict__ ids, int64_t n,
                                                      const int64_t* __restrict__ del, int64_t m,
                                                      uint8_t* __restrict__ dead) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t v = up_find(ids, n, del[i]);
  if (v >= 0) dead[v] = 1;
}

__global__ void __launch_bounds__(256) up_gone_kernel(const int64_t* __restrict__ ids, int64_t n,
                                                      const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ adj,
                                                      const int64_t* __restrict__ ds,
                                                      const int64_t* __restrict__ dd, int64_t m,
                                                      uint8_t* __restrict__ gone) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t s = up_find(ids, n, ds[i]);
  const int64_t d = s >= 0 ? up_find(ids, n, dd[i]) : -1;
  if (d < 0) return;
  int64_t lo = off[s], hi = off[s + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (adj[mid] < d) lo = mid + 1;
    else hi = mid;
  }
  if (lo < off[s + 1] && adj[lo] == d) gone[lo] = 1;
}

// keep[e] for every edge: warp per row, lanes over the row.
__global__ void __launch_bounds__(256) up_keep_kernel(const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ adj, int64_t n,
                                                      const uint8_t* __restrict__ dead,
                                                      uint8_t* __restrict__ keep) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
    const bool row_dead = dead[r] != 0;
    for (int64_t e = off[r] + lane, b = off[r + 1]; e < b; e += 32)
      keep[e] = (!row_dead && !keep[e] && !dead[adj[e]]) ? 1 : 0;  // keep[] holds gone[] on entry
  }
}

// Stream compaction by a byte flag: per-tile counts, then ordered writes of
// (a[i], b[i]) for flagged i (b may be null).
__global__ void __launch_bounds__(256) up_count_kernel(const uint8_t* __restrict__ flag, int64_t n,
                                                       bool invert, int64_t* __restrict__ counts) {
  __shared__ int64_t s_red[8];
  const int64_t r0 = int64_t(blockIdx.x) * UP_TILE + threadIdx.x;
  int64_t c = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + i * 256;
    if (r < n && ((flag[r] != 0) != invert)) ++c;
  }
  c = block_sum_256(c, s_red);
  if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

__global__ void __launch_bounds__(256) up_write_kernel(const uint8_t* __restrict__ flag, int64_t n,
                                                       bool invert, const int64_t* __restrict__ offs,
                                                       const int64_t* __restrict__ a,
                                                       const int64_t* __restrict__ b,
                                                       int64_t* __restrict__ oa,
                                                       int64_t* __restrict__ ob) {
  __shared__ uint32_t s_w[8][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = int64_t(blockIdx.x) * UP_TILE + threadIdx.x;
  uint32_t hit = 0, below[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + i * 256;
    const bool h = r < n && ((flag[r] != 0) != invert);
    const uint32_t bb = __ballot_sync(0xffffffffu, h);
    below[i] = __popc(bb & ((1u << lane) - 1u));
    if (lane == 0) s_w[i][warp] = __popc(bb);
    hit |= uint32_t(h) << i;
  }
  __syncthreads();
  int64_t base = offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t before = 0, slab = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t c = s_w[i][w];
      before += w < warp ? c : 0u;
      slab += c;
    }
    if ((hit >> i) & 1u) {
      const int64_t r = r0 + i * 256;
      oa[base + before + below[i]] = a[r];
      if (b) ob[base + before + below[i]] = b[r];
    }
    base += slab;
  }
}

}  // namespace gtd

namespace gt {

// Compact (a, b)[flag != invert] into (oa, ob); returns the count.
static int64_t compact(const uint8_t* flag, int64_t n, bool invert, const int64_t* a,
                       const int64_t* b, int64_t* oa, int64_t* ob, int64_t* scratch_counts,
                       int64_t* total) {
  if (n == 0) return 0;
  const int64_t tiles = ceil_div64(n, gtd::UP_TILE);
  GT_LAUNCH(gtd::up_count_kernel, static_cast<int>(tiles), 256, 0, flag, n, invert,
            scratch_counts);
  exclusive_scan_i64(scratch_counts, tiles, total);
  GT_LAUNCH(gtd::up_write_kernel, static_cast<int>(tiles), 256, 0, flag, n, invert,
            scratch_counts, a, b, oa, ob);
  int64_t m = 0;
  d2h(&m, total, 8);
  sync();
  return m;
}

static gt_graph* graph_update(const gt_graph* g, const int64_t* add_src, const int64_t* add_dst,
                              int64_t n_add, const int64_t* del_src, const int64_t* del_dst,
                              int64_t n_del, const int64_t* add_nodes, int64_t n_add_nodes,
                              const int64_t* del_nodes, int64_t n_del_nodes) {
  require_init();
  const int64_t n = g->n, e = g->e;
  cudaStream_t s = ctx().stream;
  // scratch owned here (the build below uses every workspace slot)
  const size_t bytes = size_t(n) + size_t(e) + 16 + 8 * (size_t(ceil_div64(std::max(n, e), 2048)) + 4) +
                       8 * 2 * size_t(e + n_add) + 8 * size_t(n + n_add_nodes) + 64;
  char* base = static_cast<char*>(dalloc(bytes));
  char* p = base;
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  uint8_t* dead = reinterpret_cast<uint8_t*>(carve(size_t(n) + 1));
  uint8_t* keep = reinterpret_cast<uint8_t*>(carve(size_t(e) + 1));
  int64_t* counts = reinterpret_cast<int64_t*>(carve(8 * (size_t(ceil_div64(std::max(n, e), 2048)) + 2)));
  int64_t* total = reinterpret_cast<int64_t*>(carve(16));
  int64_t* src = reinterpret_cast<int64_t*>(carve(8 * size_t(e + n_add)));
  int64_t* dst = reinterpret_cast<int64_t*>(carve(8 * size_t(e + n_add)));
  int64_t* nodes = reinterpret_cast<int64_t*>(carve(8 * size_t(n + n_add_nodes)));
  gt_graph* out = nullptr;
  try {
    int64_t kept = 0, live = 0;
    {
      Phase ph("update.filter", 1.0 * n + 2.0 * e + 4.0 * e + 16.0 * (n + 1));
      if (n) GT_CUDA(cudaMemsetAsync(dead, 0, size_t(n), s));
      if (e) GT_CUDA(cudaMemsetAsync(keep, 0, size_t(e), s));
      if (n && n_del_nodes)
        GT_LAUNCH(gtd::up_dead_kernel, ceil_div(n_del_nodes, 256), 256, 0, g->ids, n, del_nodes,
                  n_del_nodes, dead);
      if (e && n_del)
        GT_LAUNCH(gtd::up_gone_kernel, ceil_div(n_del, 256), 256, 0, g->ids, n, g->out_off,
                  g->out_adj, del_src, del_dst, n_del, keep);
      if (e)
        GT_LAUNCH(gtd::up_keep_kernel,
                  static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div64(n, 8),
                                                                            16LL * ctx().sm_count))),
                  256, 0, g->out_off, g->out_adj, n, dead, keep);
    }
    if (e) {
      // the old edges as (src id, dst id) in (src, dst) order, then compacted
      int64_t* es = ws_n<int64_t>(WS_TMP2, size_t(2 * e));
      int64_t* ed = es + e;
      if (gt_graph_edge_table(g, es, ed, 1) != GT_OK) {
        const std::string msg = gt_last_error();
        fail(GT_ECUDA, msg.c_str());
      }
      Phase ph("update.compact", 17.0 * e);
      kept = compact(keep, e, false, es, ed, src, dst, counts, total);
    }
    if (n) {
      Phase ph("update.compact", 9.0 * n);
      live = compact(dead, n, true, g->ids, nullptr, nodes, nullptr, counts, total);
    }
    if (n_add) {
      GT_CUDA(cudaMemcpyAsync(src + kept, add_src, size_t(n_add) * 8, cudaMemcpyDeviceToDevice, s));
      GT_CUDA(cudaMemcpyAsync(dst + kept, add_dst, size_t(n_add) * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (n_add_nodes)
      GT_CUDA(cudaMemcpyAsync(nodes + live, add_nodes, size_t(n_add_nodes) * 8,
                              cudaMemcpyDeviceToDevice, s));
    out = build_csr(src, dst, kept + n_add, nodes, live + n_add_nodes, true);
  } catch (...) {
    sync();
    dfree(base);
    throw;
  }
  sync();
  dfree(base);
  return out;
}

}  // namespace gt

using namespace gt;

extern "C" int gt_graph_update(const gt_graph* g, const int64_t* d_add_src,
                               const int64_t* d_add_dst, int64_t n_add, const int64_t* d_del_src,
                               const int64_t* d_del_dst, int64_t n_del,
                               const int64_t* d_add_nodes, int64_t n_add_nodes,
                               const int64_t* d_del_nodes, int64_t n_del_nodes, gt_graph** out) {
  GT_API_BEGIN
  if (!g || !out) fail(GT_EINVAL, "null graph or output");
  if (n_add < 0 || n_del < 0 || n_add_nodes < 0 || n_del_nodes < 0)
    fail(GT_EINVAL, "update sizes must be >= 0");
  if ((n_add && (!d_add_src || !d_add_dst)) || (n_del && (!d_del_src || !d_del_dst)) ||
      (n_add_nodes && !d_add_nodes) || (n_del_nodes && !d_del_nodes))
    fail(GT_EINVAL, "null update array");
  *out = graph_update(g, d_add_src, d_add_dst, n_add, d_del_src, d_del_dst, n_del, d_add_nodes,
                      n_add_nodes, d_del_nodes, n_del_nodes);
  GT_API_END
}
