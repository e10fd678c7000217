// triangles.cu — exact triangle count of the symmetrised graph.
//
// Reference (algorithms.py:90-119): undirected neighbourhoods = union of in-
// and out-neighbours minus self (graphs.py:163-167); rank nodes by
// (undirected degree, id) (algorithms.py:103-106); keep only higher-ranked
// neighbours (algorithms.py:108); total = sum over oriented arcs (u,v) of
// |N+(u) ∩ N+(v)| (algorithms.py:110-116).
//
// Device pipeline:
//   und_keys_kernel    out-CSR arcs -> (min,max) packed keys, self-loops -> sentinel
//   radix_sort         2k bits
//   und_dedupe_kernel  unique undirected pairs (m) + undirected degrees
//   orient_kernel      pair -> arc from lower to higher (degree, id) rank
//   radix_sort         2k bits
//   segment<plain>     oriented CSR (off_p, adj_p), rows ascending by id
//   tc_items_kernel    work items (u, block of 32 out-neighbours)
//   tc_count_kernel    warp per item: N+(u) staged in shared memory; the
//                      warp flattens the (v, w in N+(v)) pairs of its 32 v's
//                      across lanes and binary-searches each w in N+(u)
//                      (or N+(v) elements searched in N+(u) when shorter).
// All counts are integers -> exact and order independent.
#include "graph.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "segment.cuh"

#include <algorithm>

namespace gtd {

constexpr int TC_TILE = 2048;
constexpr int TC_CAP = 1024;  // N+(u) staged in shared memory up to this size

// Largest r in [lo, hi] with off[r] <= e (the row holding edge e).
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ off, int64_t lo, int64_t hi,
                                          int64_t e) {
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) und_keys_kernel(const int64_t* __restrict__ off,
                                                       const int32_t* __restrict__ adj, int64_t n,
                                                       int64_t e, int kbits, SortPlan plan,
                                                       unsigned long long* __restrict__ hist,
                                                       uint64_t* __restrict__ keys) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  __shared__ int64_t s_r[2];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  const int64_t e0 = int64_t(blockIdx.x) * TC_TILE;
  const int64_t e1 = min(e, e0 + TC_TILE);
  if (threadIdx.x == 0) {
    s_r[0] = row_of(off, 0, n - 1, e0);
    s_r[1] = row_of(off, s_r[0], n - 1, e1 - 1);
  }
  __syncthreads();
  constexpr int PER = TC_TILE / 256;
  const int64_t my0 = e0 + int64_t(threadIdx.x) * PER;
  if (my0 < e1) {
    int64_t r = row_of(off, s_r[0], s_r[1], my0);
    int64_t rend = off[r + 1];
    for (int i = 0; i < PER; ++i) {
      const int64_t ei = my0 + i;
      if (ei >= e1) break;
      while (ei >= rend) { ++r; rend = off[r + 1]; }
      const uint64_t u = uint64_t(r), v = uint64_t(adj[ei]);
      uint64_t key;
      if (u == v) key = ~0ull;
      else key = u < v ? ((u << kbits) | v) : ((v << kbits) | u);
      keys[ei] = key;
      plan_hist_add(sh, plan, key);
    }
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

// Unique undirected pairs (drop repeats and self-loop sentinels) + degrees.
__global__ void __launch_bounds__(256) und_dedupe_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                         int kbits, uint64_t* __restrict__ out,
                                                         int32_t* __restrict__ deg,
                                                         uint64_t* __restrict__ status,
                                                         uint32_t* __restrict__ counter,
                                                         uint32_t epoch,
                                                         int64_t* __restrict__ total_out) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = int(s_tile);
  const int64_t wbase = int64_t(tile) * SEG_TILE + int64_t(warp) * 32 * SEG_KPT;
  const uint64_t mask2 = (kbits >= 32) ? ~0ull : ((1ull << (2 * kbits)) - 1ull);
  uint64_t k[SEG_KPT];
  uint32_t keep_bits = 0, before[SEG_KPT], run = 0;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    k[i] = idx < n ? keys[idx] : ~0ull;
    const bool keep = idx < n && (k[i] & mask2) != mask2 && (idx == 0 || keys[idx - 1] != k[i]);
    keep_bits |= uint32_t(keep) << i;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    before[i] = run + __popc(bal & lt);
    run += __popc(bal);
  }
  if (lane == 0) s_warp[warp] = run;
  __syncthreads();
  uint32_t wpre = 0, tcount = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t c = s_warp[w];
    if (w < warp) wpre += c;
    tcount += c;
  }
  if (tid == 0) {
    s_excl = lookback_single(status, tile, epoch, tcount);
    if (int64_t(tile) == (n - 1) / SEG_TILE) *total_out = int64_t(s_excl) + tcount;
  }
  __syncthreads();
  const int64_t base = int64_t(s_excl) + wpre;
  const uint64_t low = (1ull << kbits) - 1ull;
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    if ((keep_bits >> i) & 1u) {
      out[base + before[i]] = k[i];
      atomicAdd(&deg[k[i] >> kbits], 1);
      atomicAdd(&deg[k[i] & low], 1);
    }
  }
}

__global__ void __launch_bounds__(256) orient_kernel(const uint64_t* __restrict__ pairs, int64_t m,
                                                     int kbits, const int32_t* __restrict__ deg,
                                                     SortPlan plan,
                                                     unsigned long long* __restrict__ hist,
                                                     uint64_t* __restrict__ arcs) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t low = (1ull << kbits) - 1ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint64_t p = pairs[i];
    const uint64_t a = p >> kbits, b = p & low;  // a < b by id
    const int32_t da = deg[a], db = deg[b];
    const bool a_low = da <= db;  // equal degree: the lower id (a) ranks lower
    const uint64_t arc = a_low ? p : ((b << kbits) | a);
    arcs[i] = arc;
    plan_hist_add(sh, plan, arc);
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

// Items: (u, first index of a block of 32 out-neighbours) for d+(u) >= 2.
__global__ void __launch_bounds__(256) tc_item_count_kernel(const int64_t* __restrict__ off, int64_t n,
                                                            int64_t* __restrict__ cnt) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t d = off[u + 1] - off[u];
  cnt[u] = d >= 2 ? (d + 31) / 32 : 0;
}

__global__ void __launch_bounds__(256) tc_item_fill_kernel(const int64_t* __restrict__ item_off,
                                                           int64_t n, int2* __restrict__ items) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t a = item_off[u], b = item_off[u + 1];
  for (int64_t i = a; i < b; ++i) items[i] = make_int2(int(u), int(i - a));
}

__device__ __forceinline__ bool bsearch_in(const int32_t* list, int len, int32_t x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (list[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && list[lo] == x;
}

__global__ void __launch_bounds__(256) tc_count_kernel(const int64_t* __restrict__ off,
                                                       const int32_t* __restrict__ adj,
                                                       const int2* __restrict__ items, int64_t n_items,
                                                       unsigned int* __restrict__ next_item,
                                                       unsigned long long* __restrict__ total) {
  __shared__ int32_t s_list[8][TC_CAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long acc = 0;
  int32_t* my = s_list[warp];
  while (true) {
    unsigned int it = 0;
    if (lane == 0) it = atomicAdd(next_item, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (int64_t(it) >= n_items) break;
    const int2 item = items[it];
    const int64_t u = item.x;
    const int64_t ou = off[u];
    const int du = int(off[u + 1] - ou);
    const int32_t* lu;
    if (du <= TC_CAP) {
      for (int j = lane; j < du; j += 32) my[j] = adj[ou + j];
      __syncwarp();
      lu = my;
    } else {
      lu = adj + ou;
    }
    // this item's 32 v's
    const int j = item.y * 32 + lane;
    int32_t v = -1;
    int64_t ov = 0;
    int dv = 0;
    if (j < du) {
      v = lu[j];
      ov = off[v];
      dv = int(off[v + 1] - ov);
    }
    const int incl = warp_incl_scan(dv);
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - dv;
    unsigned int cnt = 0;
    for (int t0 = 0; t0 < tot; t0 += 32) {
      const int t = t0 + lane;
      // owner lane: largest l with excl_l <= t
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int cand = lo + step;
        const int ex = __shfl_sync(0xffffffffu, excl, cand & 31);
        if (cand < 32 && ex <= t) lo = cand;
      }
      const int64_t ovl = __shfl_sync(0xffffffffu, ov, lo);
      const int exl = __shfl_sync(0xffffffffu, excl, lo);
      if (t < tot) {
        const int32_t w = adj[ovl + (t - exl)];
        cnt += bsearch_in(lu, du, w) ? 1u : 0u;
      }
    }
    acc += warp_sum(cnt);
    __syncwarp();
  }
  if (lane == 0 && acc) atomicAdd(total, acc);
}

}  // namespace gtd

namespace gt {

int64_t triangles(const gt_graph* g) {
  require_init();
  if (!g) fail(GT_EINVAL, "null graph");
  const int64_t n = g->n, e = g->e;
  if (n == 0 || e == 0) return 0;
  cudaStream_t s = ctx().stream;
  const int kb = g->kbits;
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(e));
  uint64_t* kbuf = ws_n<uint64_t>(WS_KEYS_B, size_t(e));

  // 1. undirected pair keys from the out-CSR
  SortPlan plan = make_plan(0, 2 * kb);
  SortHist h0 = sort_hist_begin(0);
  {
    Phase ph("tc.und_keys", 4.0 * e + 8.0 * n + 8.0 * e);
    GT_LAUNCH(gtd::und_keys_kernel, ceil_div(e, gtd::TC_TILE), 256, 0, g->out_off, g->out_adj, n, e,
              kb, plan, h0.hist, ka);
  }
  uint64_t* sorted = radix_sort(ka, kbuf, e, plan, h0, "tc.sort");
  uint64_t* other = sorted == ka ? kbuf : ka;

  // 2. unique undirected pairs + degrees
  int32_t* deg = ws_n<int32_t>(WS_TMP2, size_t(n));
  GT_CUDA(cudaMemsetAsync(deg, 0, size_t(n) * 4, s));
  {
    Phase ph("tc.und_dedupe", 8.0 * e);
    const int64_t tiles = ceil_div64(e, gtd::SEG_TILE);
    uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) * 256);
    GT_CUDA(cudaMemsetAsync(counters + 20, 0, 4, s));
    GT_LAUNCH(gtd::und_dedupe_kernel, static_cast<int>(tiles), 256, 0, sorted, e, kb, other, deg,
              status, counters + 20, next_epoch(), small + 4);
  }
  int64_t m = 0;
  d2h(&m, small + 4, 8);
  sync();
  profile_add_bytes("tc.und_dedupe", 8.0 * m + 8.0 * m);
  if (m == 0) return 0;

  // 3. orient by (degree, id) and sort arcs
  SortHist h1 = sort_hist_begin(1);
  {
    Phase ph("tc.orient", 16.0 * m);
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div64(m, 1024), 8LL * ctx().sm_count));
    GT_LAUNCH(gtd::orient_kernel, grid, 256, 0, other, m, kb, deg, plan, h1.hist, sorted);
  }
  uint64_t* arcs = radix_sort(sorted, other, m, plan, h1, "tc.sort");

  // 4. oriented CSR
  const size_t need = size_t(n + 1) * 8 * 2 + size_t(m) * 4 + 64;
  char* p = static_cast<char*>(ws_get(WS_TMP3, need));
  int64_t* off_p = reinterpret_cast<int64_t*>(p);
  int64_t* item_off = off_p + (n + 1);
  int32_t* adj_p = reinterpret_cast<int32_t*>(item_off + (n + 1));
  {
    Phase ph("tc.oriented_csr", 12.0 * m + 8.0 * n);
    GT_LAUNCH(gtd::segment_kernel<false>, ceil_div(m, gtd::SEG_TILE), 256, 0, arcs, m, kb, n, adj_p,
              off_p, (uint64_t*)nullptr, SortPlan(), (unsigned long long*)nullptr,
              (uint64_t*)nullptr, (uint32_t*)nullptr, 0u, (int64_t*)nullptr);
  }

  // 5. work items: (u, block of 32 out-neighbours) for every u with d+(u) >= 2
  int64_t n_items = 0;
  {
    Phase ph("tc.items", 16.0 * n);
    GT_LAUNCH(gtd::tc_item_count_kernel, ceil_div(n, 256), 256, 0, off_p, n, item_off);
    exclusive_scan_i64(item_off, n, small + 5);
  }
  d2h(&n_items, small + 5, 8);
  sync();
  unsigned long long* total = reinterpret_cast<unsigned long long*>(small + 6);
  GT_CUDA(cudaMemsetAsync(total, 0, 8, s));
  if (n_items > 0) {
    if (n_items >= (int64_t(1) << 32)) fail(GT_ECAPACITY, "triangle work list too long");
    int2* items = ws_n<int2>(WS_TMP0, size_t(n_items));
    GT_CUDA(cudaMemsetAsync(counters + 21, 0, 4, s));
    {
      Phase ph("tc.items", 8.0 * n_items);
      GT_LAUNCH(gtd::tc_item_fill_kernel, ceil_div(n, 256), 256, 0, item_off, n, items);
    }
    Phase ph("tc.count", 4.0 * m);
    GT_LAUNCH(gtd::tc_count_kernel, ctx().sm_count * 8, 256, 0, off_p, adj_p, items, n_items,
              counters + 21, total);
  }
  int64_t result = 0;
  d2h(&result, total, 8);
  sync();
  return result;
}

}  // namespace gt

using namespace gt;

extern "C" int gt_triangles(const gt_graph* g, int64_t* count) {
  GT_API_BEGIN
  if (!count) fail(GT_EINVAL, "count must not be NULL");
  *count = triangles(g);
  GT_API_END
}
