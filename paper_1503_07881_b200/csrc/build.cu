// build.cu — ToGraph on the device: edge table -> out-CSR + in-CSR.
//
// Reference algorithm (convert.py:128-175): dense ids by np.unique
// (convert.py:45-59), pack (src,dst) into a 64-bit key (convert.py:62-63),
// sort + drop adjacent duplicates (convert.py:71-80), re-sort by (dst,src)
// for the in-pool (convert.py:150-151), bincount/cumsum offsets
// (convert.py:154-157), scatter into per-node pools (convert.py:92-125).
//
// Device pipeline (one stream, three small host syncs for sizes):
//   minmax_kernel      16 B/row   id range -> dense or sparse id map
//   presence_kernel    16 B/row   1 bit per id in the range (dense path)
//   word_prefix_kernel W*8 B      popcount prefix -> rank of every present id
//   ids_kernel         W*8 + 8N   sorted distinct ids
//   pack_kernel        24 B/row   key = rank(src)<<k | rank(dst), k = ceil(log2 N),
//                                 + digit histograms of every radix pass
//   radix_sort         16 B/row/pass over 2k bits
//   segment<dedupe>    8R + 12E + 8N  drop duplicate keys, out_adj, out_off,
//                                 in-keys (dst<<k|src) + their digit histograms
//   radix_sort         16 B/edge/pass over the k dst bits only (stable:
//                                 src stays ascending within each dst)
//   segment<plain>     8E + 4E + 8N   in_adj, in_off
// Sparse ids (range wider than 32 ids per row) take the sort-unique path of
// convert.py:59 instead: radix sort of the 2R ids + unique + binary search.
#include "graph.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "segment.cuh"

#include <algorithm>
#include <cstring>

namespace gtd {

using gt::SortPlan;

__global__ void __launch_bounds__(256) minmax_kernel(const int64_t* __restrict__ src,
                                                     const int64_t* __restrict__ dst, int64_t n,
                                                     long long* __restrict__ out) {
  __shared__ long long smin[8], smax[8];
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long a = ld_stream_s64(src + i), b = ld_stream_s64(dst + i);
    mn = min(mn, min(a, b));
    mx = max(mx, max(a, b));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { smin[w] = mn; smax[w] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < int(blockDim.x >> 5); ++i) { mn = min(mn, smin[i]); mx = max(mx, smax[i]); }
    atomicMin(&out[0], mn);
    atomicMax(&out[1], mx);
  }
}

// Rank map word: presence bits of 32 consecutive ids + number of present ids
// below the word (exclusive popcount prefix).
// The check goes through the non-coherent L1 path: a stale 0 only costs a
// redundant atomicOr (bits are only ever set), and hub ids — most rows on
// R-MAT — then skip the L2 atomic entirely.
__device__ __forceinline__ void mark_present(uint2* __restrict__ words, uint64_t off) {
  unsigned int* p = &words[off >> 5].x;
  const unsigned int bit = 1u << (off & 31);
  if ((__ldg(p) & bit) == 0) atomicOr(p, bit);
}

__global__ void __launch_bounds__(256) presence_kernel(const int64_t* __restrict__ src,
                                                       const int64_t* __restrict__ dst, int64_t n,
                                                       int64_t lo, uint2* __restrict__ words) {
  // U rows per thread per step: all 2U id loads, then all 2U word checks, are
  // in flight before the first conditional atomic
  constexpr int U = 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint64_t off[2 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      off[2 * u] = uint64_t(ld_stream_s64(src + i + u * stride)) - uint64_t(lo);
      off[2 * u + 1] = uint64_t(ld_stream_s64(dst + i + u * stride)) - uint64_t(lo);
    }
    unsigned int seen[2 * U];
#pragma unroll
    for (int u = 0; u < 2 * U; ++u) seen[u] = __ldg(&words[off[u] >> 5].x);
#pragma unroll
    for (int u = 0; u < 2 * U; ++u) {
      const unsigned int bit = 1u << (off[u] & 31);
      if ((seen[u] & bit) == 0) atomicOr(&words[off[u] >> 5].x, bit);
    }
  }
  for (; i < n; i += stride) {
    mark_present(words, uint64_t(ld_stream_s64(src + i)) - uint64_t(lo));
    mark_present(words, uint64_t(ld_stream_s64(dst + i)) - uint64_t(lo));
  }
}

// Blocked exclusive popcount scan over the rank-map words (16 words/thread).
__global__ void __launch_bounds__(256) word_prefix_kernel(uint2* __restrict__ words, int64_t nw,
                                                          uint64_t* __restrict__ status,
                                                          uint32_t* __restrict__ counter,
                                                          uint32_t epoch,
                                                          int64_t* __restrict__ total_out) {
  __shared__ uint32_t s_tile;
  __shared__ int64_t s_scan[8];
  __shared__ uint64_t s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = int(s_tile);
  const int64_t first = (int64_t(tile) * 256 + threadIdx.x) * 16;
  uint32_t c[16];
  int64_t sum = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    c[j] = (first + j < nw) ? __popc(words[first + j].x) : 0u;
    sum += c[j];
  }
  int64_t tot;
  int64_t ex = block_excl_scan_256<int64_t>(sum, s_scan, tot);
  if (threadIdx.x == 0) s_excl = lookback_single(status, tile, epoch, uint64_t(tot));
  __syncthreads();
  int64_t run = int64_t(s_excl) + ex;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (first + j < nw) words[first + j].y = uint32_t(run);
    run += c[j];
  }
  if (first <= nw - 1 && nw - 1 < first + 16) *total_out = run;  // thread holding the last word
}

__global__ void __launch_bounds__(256) ids_kernel(const uint2* __restrict__ words, int64_t nw,
                                                  int64_t lo, int64_t* __restrict__ ids) {
  const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint2 v = words[w];
  uint32_t bits = v.x;
  int64_t pos = v.y;
  while (bits) {
    const int b = __ffs(bits) - 1;
    bits &= bits - 1;
    ids[pos++] = lo + (w << 5) + b;
  }
}

__device__ __forceinline__ uint32_t rank_dense(const uint2* __restrict__ words, int64_t x,
                                               int64_t lo) {
  const uint64_t off = uint64_t(x) - uint64_t(lo);
  const uint2 w = words[off >> 5];
  return w.y + __popc(w.x & ((1u << (off & 31)) - 1u));
}

__device__ __forceinline__ uint32_t rank_search(const int64_t* __restrict__ ids, int64_t n,
                                                int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ids[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return uint32_t(lo);
}

template <bool DENSE>
__global__ void __launch_bounds__(256) pack_kernel(const int64_t* __restrict__ src,
                                                   const int64_t* __restrict__ dst, int64_t n,
                                                   int64_t lo, const uint2* __restrict__ words,
                                                   const int64_t* __restrict__ ids, int64_t n_ids,
                                                   int kbits, SortPlan plan,
                                                   unsigned long long* __restrict__ hist,
                                                   uint64_t* __restrict__ keys) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  // U rows per thread per step: all 2U column loads, then all 2U rank
  // lookups, are in flight before the first key is formed (the single-row
  // loop was latency-bound: 2.3 TB/s at C4)
  constexpr int U = 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int64_t a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = ld_stream_s64(src + i + u * stride);
      b[u] = ld_stream_s64(dst + i + u * stride);
    }
    uint32_t ra[U], rb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (DENSE) {
        ra[u] = rank_dense(words, a[u], lo);
        rb[u] = rank_dense(words, b[u], lo);
      } else {
        ra[u] = rank_search(ids, n_ids, a[u]);
        rb[u] = rank_search(ids, n_ids, b[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t key = (uint64_t(ra[u]) << kbits) | rb[u];
      __stcs(keys + i + u * stride, key);
      plan_hist_add(sh, plan, key);
    }
  }
  for (; i < n; i += stride) {
    const int64_t a = ld_stream_s64(src + i), b = ld_stream_s64(dst + i);
    uint32_t ra, rb;
    if (DENSE) {
      ra = rank_dense(words, a, lo);
      rb = rank_dense(words, b, lo);
    } else {
      ra = rank_search(ids, n_ids, a);
      rb = rank_search(ids, n_ids, b);
    }
    const uint64_t key = (uint64_t(ra) << kbits) | rb;
    keys[i] = key;
    plan_hist_add(sh, plan, key);
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

// Sparse path: ids shifted to unsigned offsets from lo, for a sort of 2R keys.
__global__ void __launch_bounds__(256) idkeys_kernel(const int64_t* __restrict__ src,
                                                     const int64_t* __restrict__ dst, int64_t n,
                                                     int64_t lo, SortPlan plan,
                                                     unsigned long long* __restrict__ hist,
                                                     uint64_t* __restrict__ keys) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t a = uint64_t(ld_stream_s64(src + i)) - uint64_t(lo);
    const uint64_t b = uint64_t(ld_stream_s64(dst + i)) - uint64_t(lo);
    keys[i] = a;
    keys[n + i] = b;
    plan_hist_add(sh, plan, a);
    plan_hist_add(sh, plan, b);
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

// Sparse path: sorted id offsets -> distinct ids (lo + offset).
__global__ void __launch_bounds__(256) unique_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                     int64_t lo, int64_t* __restrict__ ids,
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
  uint64_t k[SEG_KPT];
  uint32_t keep_bits = 0, before[SEG_KPT], run = 0;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    k[i] = idx < n ? keys[idx] : 0ull;
    const bool keep = idx < n && (idx == 0 || keys[idx - 1] != k[i]);
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
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i)
    if ((keep_bits >> i) & 1u) ids[base + before[i]] = lo + int64_t(k[i]);
}

__global__ void __launch_bounds__(256) gather_ids_kernel(const int32_t* __restrict__ adj, int64_t n,
                                                         const int64_t* __restrict__ ids,
                                                         int64_t* __restrict__ out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = ids[adj[i]];
}


// ---- per-node lookups (Graph.record / has_node / has_edge, graphs.py:62-88,
// 148-167) without exporting the CSR: binary searches on the device, one
// row gathered and copied back.
__device__ __forceinline__ int64_t gl_find(const int64_t* __restrict__ ids, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (ids[m] < x) lo = m + 1;
    else hi = m;
  }
  return (lo < n && ids[lo] == x) ? lo : -1;
}

__global__ void gl_find_kernel(const int64_t* __restrict__ ids, int64_t n,
                               const int64_t* __restrict__ q, int64_t k, int64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < k) out[i] = gl_find(ids, n, q[i]);
}

__global__ void gl_has_edge_kernel(const int64_t* __restrict__ ids, int64_t n,
                                   const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                                   int64_t src, int64_t dst, int64_t* __restrict__ out) {
  const int64_t a = gl_find(ids, n, src), b = gl_find(ids, n, dst);
  int64_t r = 0;
  if (a >= 0 && b >= 0) {
    int64_t lo = off[a], hi = off[a + 1];
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (adj[m] < int32_t(b)) lo = m + 1;
      else hi = m;
    }
    r = (lo < off[a + 1] && adj[lo] == int32_t(b)) ? 1 : 0;
  }
  out[0] = r;
}

__global__ void gl_row_kernel(const int64_t* __restrict__ ids, const int32_t* __restrict__ adj,
                              int64_t begin, int64_t len, int64_t* __restrict__ out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += stride)
    out[i] = ids[adj[begin + i]];
}
// Kept (distinct) keys per SEG_TILE tile of the sorted out-keys (scanned into
// segment_kernel<true>'s tile bases), and the in-sort digit counts of the
// dropped copies (see in_hist_kernel). Tiles are independent: no look-back.
__global__ void __launch_bounds__(256) dedupe_count_kernel(const uint64_t* __restrict__ keys,
                                                           int64_t n, int kbits, SortPlan in_plan,
                                                           unsigned long long* __restrict__ dup_hist,
                                                           int64_t* __restrict__ tile_cnt) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  __shared__ uint32_t s_w[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < in_plan.passes * 256; i += 256) sh[i] = 0;
  __syncthreads();
  const int64_t wbase = int64_t(blockIdx.x) * SEG_TILE + int64_t(warp) * 32 * SEG_KPT;
  const uint64_t lowmask = (1ull << kbits) - 1ull;
  uint64_t k[SEG_KPT];
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    k[i] = idx < n ? ld_stream_u64(keys + idx) : 0ull;
  }
  uint64_t first_prev = 0;
  if (lane == 0 && wbase > 0 && wbase - 1 < n) first_prev = keys[wbase - 1];
  const unsigned lt = lanemask_lt();
  uint32_t kept = 0;
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    uint64_t prev = __shfl_up_sync(0xffffffffu, k[i], 1);
    const uint64_t last_prev = __shfl_sync(0xffffffffu, i > 0 ? k[i > 0 ? i - 1 : 0] : first_prev, 31);
    if (lane == 0) prev = (i == 0) ? first_prev : last_prev;
    const bool valid = idx < n;
    const bool keep = valid && (idx == 0 || k[i] != prev);
    kept += __popc(__ballot_sync(0xffffffffu, keep));
    // Copies of one key are adjacent lanes: the last lane of each run of
    // dropped lanes adds the run length (equal addresses would serialise).
    const uint32_t dropped = __ballot_sync(0xffffffffu, valid && !keep);
    if (dropped && ((dropped >> lane) & 1u) && (lane == 31 || !((dropped >> (lane + 1)) & 1u))) {
      const uint32_t below = ~dropped & lt;
      const uint32_t cnt = uint32_t(lane) - (below ? uint32_t(31 - __clz(below)) : ~0u);
      const uint64_t ik = ((k[i] & lowmask) << kbits) | (k[i] >> kbits);
#pragma unroll
      for (int q = 0; q < gt::RS_MAX_PASSES; ++q)
        if (q < in_plan.passes)
          atomicAdd(&sh[q * 256 + (uint32_t(ik >> in_plan.shift[q]) & ((1u << in_plan.bits[q]) - 1u))],
                    cnt);
    }
  }
  if (lane == 0) s_w[warp] = kept;
  __syncthreads();
  if (tid == 0) {
    int64_t t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_w[w];
    tile_cnt[blockIdx.x] = t;
  }
  plan_hist_flush(sh, in_plan, dup_hist);
}

// The in-sort digit histograms without a per-key pass: the in-plan's digits
// are the out-plan's digits restricted to the dst bits [0, kbits) (an in-key
// is dst << kbits | src), so each in-histogram is a fold of one out-sort
// histogram — counted by pack_kernel over every row — minus the digit counts
// of the duplicates segment_kernel<true> dropped. grid = in passes.
__global__ void __launch_bounds__(256) in_hist_kernel(const unsigned long long* __restrict__ out_hist,
                                                      SortPlan in_plan, SortPlan src_pass,
                                                      const unsigned long long* __restrict__ dup_hist,
                                                      unsigned long long* __restrict__ in_hist) {
  const int q = blockIdx.x;
  const int b = in_plan.bits[q];
  const int p = src_pass.shift[q];  // the out pass holding in-digit q (low bits of its digit)
  const int w = src_pass.bits[q];   // that out digit's width
  const uint32_t x = threadIdx.x;
  if (x >= (1u << b)) {
    if (x < 256) in_hist[q * 256 + x] = 0;
    return;
  }
  unsigned long long c = 0;
  for (uint32_t hi = 0; hi < (1u << (w - b)); ++hi) c += out_hist[p * 256 + (hi << b | x)];
  in_hist[q * 256 + x] = c - dup_hist[q * 256 + x];
}

}  // namespace gtd

namespace gt {

// Out-sort digits (LSD first) for keys src << kb | dst: the dst bits in
// near-equal digits, the last of them widened to 8 bits into the src bits,
// then the rest of the src bits. The in-sort digits are the out digits cut to
// the dst bits (in_hist_kernel), so this keeps them near-equal too (C4: out
// 7,7,6,8,8,8,8 -> in 7,7,6,6) without adding a pass over make_plan.
static SortPlan make_out_plan(int kb) {
  SortPlan full = make_plan(0, 2 * kb);
  if (kb <= 0) return full;
  SortPlan p;
  const int nd = (kb + 7) / 8;
  int shift = 0;
  for (int q = 0; q < nd; ++q) {
    int b = kb / nd + (q < kb % nd ? 1 : 0);
    if (q == nd - 1) b = std::min(8, 2 * kb - shift);
    p.shift[p.passes] = shift;
    p.bits[p.passes++] = b;
    shift += b;
  }
  const int rest = 2 * kb - shift;
  const int nr = (rest + 7) / 8;
  for (int q = 0; q < nr; ++q) {
    const int b = rest / nr + (q < rest % nr ? 1 : 0);
    p.shift[p.passes] = shift;
    p.bits[p.passes++] = b;
    shift += b;
  }
  return p.passes <= full.passes ? p : full;
}

}  // namespace gt

namespace gt {

static int grid_for(int64_t n, int per_thread = 1) {
  const int64_t want = ceil_div64(n, 256LL * per_thread);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(ctx().sm_count) * 8)));
}

static int64_t read_i64(const int64_t* d) {
  int64_t h = 0;
  d2h(&h, d, sizeof h);
  sync();
  return h;
}

static gt_graph* empty_graph() {
  gt_graph* g = new gt_graph();
  g->out_off = dalloc_n<int64_t>(1);
  g->in_off = dalloc_n<int64_t>(1);
  GT_CUDA(cudaMemsetAsync(g->out_off, 0, 8, ctx().stream));
  GT_CUDA(cudaMemsetAsync(g->in_off, 0, 8, ctx().stream));
  sync();
  return g;
}

// Shared with bucket_build.cu.
void launch_presence(const int64_t* a, const int64_t* b, int64_t n, int64_t lo, uint2* words) {
  if (n) GT_LAUNCH(gtd::presence_kernel, grid_for(n, 4), 256, 0, a, b, n, lo, words);
}
void launch_word_prefix(uint2* words, int64_t nw, int64_t* total_out) {
  const int64_t tiles = ceil_div64(nw, 256 * 16);
  uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) * 256);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  GT_CUDA(cudaMemsetAsync(counters + 16, 0, 4, ctx().stream));
  GT_LAUNCH(gtd::word_prefix_kernel, static_cast<int>(tiles), 256, 0, words, nw, status,
            counters + 16, next_epoch(), total_out);
}
void launch_ids(const uint2* words, int64_t nw, int64_t lo, int64_t* ids) {
  GT_LAUNCH(gtd::ids_kernel, ceil_div(nw, 256), 256, 0, words, nw, lo, ids);
}
bool bucket_build_applies(int64_t rows, uint64_t span);
void bucket_build(const int64_t* src, const int64_t* dst, int64_t rows, const int64_t* extra,
                  int64_t n_extra, int64_t lo, uint64_t span, gt_graph* g);

void graph_free(gt_graph* g) {
  if (!g) return;
  dfree(g->ids);
  dfree(g->out_off);
  dfree(g->out_adj);
  dfree(g->in_off);
  dfree(g->in_adj);
  delete g;
}

gt_graph* build_csr(const int64_t* src, const int64_t* dst, int64_t rows, const int64_t* extra,
                    int64_t n_extra, bool on_device) {
  require_init();
  if (rows < 0 || n_extra < 0) fail(GT_EINVAL, "rows must be >= 0");
  if (n_extra > 0 && !extra) fail(GT_EINVAL, "extra node ids must not be NULL");
  if (rows == 0 && n_extra == 0) return empty_graph();
  cudaStream_t s = ctx().stream;

  if (!on_device) {
    int64_t* cols = ws_n<int64_t>(WS_COLS, size_t(2) * rows + size_t(n_extra));
    Phase ph("build.h2d", 16.0 * rows + 8.0 * n_extra);
    h2d(cols, src, size_t(rows) * 8);
    h2d(cols + rows, dst, size_t(rows) * 8);
    h2d(cols + 2 * rows, extra, size_t(n_extra) * 8);
    src = cols;
    dst = cols + rows;
    extra = cols + 2 * rows;
  }

  gt_graph* g = new gt_graph();
  try {
    int64_t* small = ws_n<int64_t>(WS_SMALL, 16);  // [0]=min [1]=max [2]=N [3]=E
    {
      long long init[2] = {LLONG_MAX, LLONG_MIN};
      h2d(small, init, sizeof init);
      Phase ph("build.minmax", 16.0 * rows);
      if (rows)
        GT_LAUNCH(gtd::minmax_kernel, grid_for(rows, 4), 256, 0, src, dst, rows,
                  reinterpret_cast<long long*>(small));
      if (n_extra)
        GT_LAUNCH(gtd::minmax_kernel, grid_for(n_extra, 4), 256, 0, extra, extra, n_extra,
                  reinterpret_cast<long long*>(small));
    }
    int64_t mm[2];
    d2h(mm, small, sizeof mm);
    sync();
    const int64_t lo = mm[0], hi = mm[1];
    const uint64_t span = uint64_t(hi) - uint64_t(lo);  // width - 1, no overflow
    // Dense rank map when its 8 bytes per 32 ids cost no more than one column.
    const bool dense = span < (uint64_t(1) << 36) &&
                       (span + 1) <= std::max<uint64_t>(uint64_t(1) << 26, uint64_t(rows) * 32);

    if (dense && bucket_build_applies(rows, span)) {
      bucket_build(src, dst, rows, extra, n_extra, lo, span, g);
      return g;
    }
    uint2* words = nullptr;
    int64_t nw = 0;
    int64_t n_nodes = 0;
    const size_t key_cap = dense ? size_t(rows) : size_t(2) * (rows + n_extra);
    uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, key_cap);
    uint64_t* kb = ws_n<uint64_t>(WS_KEYS_B, key_cap);
    uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);

    if (dense) {
      nw = int64_t((span + 1 + 31) / 32);
      words = ws_n<uint2>(WS_RANKMAP, size_t(nw));
      GT_CUDA(cudaMemsetAsync(words, 0, size_t(nw) * sizeof(uint2), s));
      {
        Phase ph("build.presence", 16.0 * rows);
        if (rows)
          GT_LAUNCH(gtd::presence_kernel, grid_for(rows, 4), 256, 0, src, dst, rows, lo, words);
        if (n_extra)
          GT_LAUNCH(gtd::presence_kernel, grid_for(n_extra, 4), 256, 0, extra, extra, n_extra, lo,
                    words);
      }
      {
        Phase ph("build.rank_prefix", 16.0 * nw);
        const int64_t tiles = ceil_div64(nw, 256 * 16);
        uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) * 256);
        GT_CUDA(cudaMemsetAsync(counters + 16, 0, 4, s));
        GT_LAUNCH(gtd::word_prefix_kernel, static_cast<int>(tiles), 256, 0, words, nw, status,
                  counters + 16, next_epoch(), small + 2);
      }
      n_nodes = read_i64(small + 2);
      if (n_nodes >= (int64_t(1) << 31))
        fail(GT_ECAPACITY, "graph has >= 2^31 distinct node ids");
      g->ids = dalloc_n<int64_t>(n_nodes);
      {
        Phase ph("build.ids", 8.0 * nw + 8.0 * n_nodes);
        GT_LAUNCH(gtd::ids_kernel, ceil_div(nw, 256), 256, 0, words, nw, lo, g->ids);
      }
    } else {
      // Sort-unique of the 2R ids (convert.py:59 searchsorted analogue).
      const int64_t m = 2 * (rows + n_extra);
      SortPlan idplan = make_plan(0, 64 - __builtin_clzll(span | 1));
      SortHist hh = sort_hist_begin(0);
      {
        Phase ph("build.idkeys", 32.0 * (rows + n_extra));
        if (rows)
          GT_LAUNCH(gtd::idkeys_kernel, grid_for(rows, 4), 256, 0, src, dst, rows, lo, idplan,
                    hh.hist, ka);
        if (n_extra)
          GT_LAUNCH(gtd::idkeys_kernel, grid_for(n_extra, 4), 256, 0, extra, extra, n_extra, lo,
                    idplan, hh.hist, ka + 2 * rows);
      }
      uint64_t* sorted = radix_sort(ka, kb, m, idplan, hh, "build.id_sort");
      int64_t* tmp_ids = reinterpret_cast<int64_t*>(sorted == ka ? kb : ka);
      {
        Phase ph("build.unique", 8.0 * m);
        const int64_t tiles = ceil_div64(m, gtd::SEG_TILE);
        uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) * 256);
        GT_CUDA(cudaMemsetAsync(counters + 17, 0, 4, s));
        GT_LAUNCH(gtd::unique_kernel, static_cast<int>(tiles), 256, 0, sorted, m, lo, tmp_ids,
                  status, counters + 17, next_epoch(), small + 2);
      }
      n_nodes = read_i64(small + 2);
      if (n_nodes >= (int64_t(1) << 31))
        fail(GT_ECAPACITY, "graph has >= 2^31 distinct node ids");
      g->ids = dalloc_n<int64_t>(n_nodes);
      GT_CUDA(cudaMemcpyAsync(g->ids, tmp_ids, size_t(n_nodes) * 8, cudaMemcpyDeviceToDevice, s));
    }
    g->n = n_nodes;
    const int kb_bits = bits_for(n_nodes);
    g->kbits = kb_bits;
    if (rows == 0) {  // isolated nodes only
      g->out_off = dalloc_n<int64_t>(n_nodes + 1);
      g->in_off = dalloc_n<int64_t>(n_nodes + 1);
      GT_CUDA(cudaMemsetAsync(g->out_off, 0, size_t(n_nodes + 1) * 8, s));
      GT_CUDA(cudaMemsetAsync(g->in_off, 0, size_t(n_nodes + 1) * 8, s));
      sync();
      return g;
    }

    // ---- out pass: pack -> sort (src,dst) -> dedupe/out-CSR/in-keys --------
    SortPlan out_plan = make_out_plan(kb_bits);
    SortHist ho = sort_hist_begin(0);
    {
      Phase ph("build.pack", 24.0 * rows);
      if (dense)
        GT_LAUNCH(gtd::pack_kernel<true>, grid_for(rows, 4), 256, 0, src, dst, rows, lo, words,
                  (const int64_t*)nullptr, int64_t(0), kb_bits, out_plan, ho.hist, ka);
      else
        GT_LAUNCH(gtd::pack_kernel<false>, grid_for(rows, 4), 256, 0, src, dst, rows, lo,
                  (const uint2*)nullptr, g->ids, n_nodes, kb_bits, out_plan, ho.hist, ka);
    }
    uint64_t* sorted = radix_sort(ka, kb, rows, out_plan, ho, "build.out_sort",
                                  /*first_unstable=*/true);
    uint64_t* other = sorted == ka ? kb : ka;

    g->out_adj = dalloc_n<int32_t>(rows);  // E <= rows; exact E known after dedupe
    g->out_off = dalloc_n<int64_t>(n_nodes + 1);
    // in-plan digits = out-plan digits restricted to the dst bits (see in_hist_kernel)
    SortPlan in_plan, src_pass;
    for (int p = 0; p < out_plan.passes && out_plan.shift[p] < kb_bits; ++p) {
      const int q = in_plan.passes++;
      in_plan.shift[q] = kb_bits + out_plan.shift[p];
      in_plan.bits[q] = std::min(out_plan.shift[p] + out_plan.bits[p], kb_bits) - out_plan.shift[p];
      src_pass.shift[q] = p;
      src_pass.bits[q] = out_plan.bits[p];
    }
    SortHist hi_ = sort_hist_begin(1);
    {
      Phase ph("build.dedupe", 16.0 * rows);
      const int64_t tiles = ceil_div64(rows, gtd::SEG_TILE);
      int64_t* tile_base = ws_n<int64_t>(WS_TMP3, size_t(tiles) + 1);
      unsigned long long* dup = ws_n<unsigned long long>(WS_TMP4, RS_MAX_PASSES * 256);
      GT_CUDA(cudaMemsetAsync(dup, 0, RS_MAX_PASSES * 256 * 8, s));
      GT_LAUNCH(gtd::dedupe_count_kernel, static_cast<int>(tiles), 256, 0, sorted, rows, kb_bits,
                in_plan, dup, tile_base);
      exclusive_scan_i64(tile_base, tiles, small + 3);
      GT_LAUNCH(gtd::segment_kernel<true>, static_cast<int>(tiles), 256, 0, sorted, rows, kb_bits,
                n_nodes, g->out_adj, g->out_off, other, tile_base);
      if (in_plan.passes)
        GT_LAUNCH(gtd::in_hist_kernel, in_plan.passes, 256, 0, ho.hist, in_plan, src_pass, dup,
                  hi_.hist);
    }
    const int64_t n_edges = read_i64(small + 3);
    g->e = n_edges;
    profile_add_bytes("build.dedupe", 12.0 * n_edges + 8.0 * (n_nodes + 1));

    // ---- in pass: stable sort of in-keys by dst bits -> in-CSR -------------
    uint64_t* in_sorted = radix_sort(other, sorted, n_edges, in_plan, hi_, "build.in_sort");
    g->in_adj = dalloc_n<int32_t>(n_edges);
    g->in_off = dalloc_n<int64_t>(n_nodes + 1);
    {
      Phase ph("build.in_segment", 12.0 * n_edges + 8.0 * n_nodes);
      const int64_t tiles = ceil_div64(n_edges, gtd::SEG_TILE);
      GT_LAUNCH(gtd::segment_kernel<false>, static_cast<int>(tiles), 256, 0, in_sorted, n_edges,
                kb_bits, n_nodes, g->in_adj, g->in_off, (uint64_t*)nullptr, (const int64_t*)nullptr);
    }
    sync();
    return g;
  } catch (...) {
    graph_free(g);
    throw;
  }
}

void graph_export(const gt_graph* g, int64_t* ids, int64_t* out_off, int64_t* out_adj,
                  int64_t* in_off, int64_t* in_adj) {
  require_init();
  if (!g) fail(GT_EINVAL, "null graph");
  if (ids && g->n) d2h(ids, g->ids, size_t(g->n) * 8);
  if (out_off) d2h(out_off, g->out_off, size_t(g->n + 1) * 8);
  if (in_off) d2h(in_off, g->in_off, size_t(g->n + 1) * 8);
  if ((out_adj || in_adj) && g->e) {
    int64_t* tmp = ws_n<int64_t>(WS_TMP0, size_t(g->e));
    if (out_adj) {
      GT_LAUNCH(gtd::gather_ids_kernel, grid_for(g->e, 4), 256, 0, g->out_adj, g->e, g->ids, tmp);
      d2h(out_adj, tmp, size_t(g->e) * 8);
      sync();
    }
    if (in_adj) {
      GT_LAUNCH(gtd::gather_ids_kernel, grid_for(g->e, 4), 256, 0, g->in_adj, g->e, g->ids, tmp);
      d2h(in_adj, tmp, size_t(g->e) * 8);
    }
  }
  sync();
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_build_csr(const int64_t* src, const int64_t* dst, int64_t rows, int cols_are_device,
                 gt_graph** out) {
  GT_API_BEGIN
  if (!out) fail(GT_EINVAL, "out must not be NULL");
  *out = nullptr;
  if (rows > 0 && (!src || !dst)) fail(GT_EINVAL, "src/dst must not be NULL");
  *out = build_csr(src, dst, rows, nullptr, 0, cols_are_device != 0);
  GT_API_END
}

int gt_build_csr_nodes(const int64_t* src, const int64_t* dst, int64_t rows, const int64_t* nodes,
                       int64_t n_nodes, int cols_are_device, gt_graph** out) {
  GT_API_BEGIN
  if (!out) fail(GT_EINVAL, "out must not be NULL");
  *out = nullptr;
  if (rows > 0 && (!src || !dst)) fail(GT_EINVAL, "src/dst must not be NULL");
  *out = build_csr(src, dst, rows, nodes, n_nodes, cols_are_device != 0);
  GT_API_END
}

int gt_graph_sizes(const gt_graph* g, int64_t* n_nodes, int64_t* n_edges) {
  GT_API_BEGIN
  if (!g) fail(GT_EINVAL, "null graph");
  if (n_nodes) *n_nodes = g->n;
  if (n_edges) *n_edges = g->e;
  GT_API_END
}

int gt_graph_export(const gt_graph* g, int64_t* h_ids, int64_t* h_out_off, int64_t* h_out_adj,
                    int64_t* h_in_off, int64_t* h_in_adj) {
  GT_API_BEGIN
  graph_export(g, h_ids, h_out_off, h_out_adj, h_in_off, h_in_adj);
  GT_API_END
}

int gt_graph_device_views(const gt_graph* g, const int64_t** d_ids, const int64_t** d_out_off,
                          const int32_t** d_out_adj, const int64_t** d_in_off,
                          const int32_t** d_in_adj) {
  GT_API_BEGIN
  if (!g) fail(GT_EINVAL, "null graph");
  if (d_ids) *d_ids = g->ids;
  if (d_out_off) *d_out_off = g->out_off;
  if (d_out_adj) *d_out_adj = g->out_adj;
  if (d_in_off) *d_in_off = g->in_off;
  if (d_in_adj) *d_in_adj = g->in_adj;
  GT_API_END
}

int gt_graph_find(const gt_graph* g, const int64_t* h_ids, int64_t k, int64_t* h_index) {
  GT_API_BEGIN
  require_init();
  if (!g || k < 0 || (k > 0 && (!h_ids || !h_index))) fail(GT_EINVAL, "bad arguments");
  if (k == 0) return GT_OK;
  int64_t* d = ws_n<int64_t>(WS_SMALL, size_t(2 * k) + 16);
  h2d(d, h_ids, size_t(k) * 8);
  GT_LAUNCH(gtd::gl_find_kernel, ceil_div(k, 256), 256, 0, g->ids, g->n, d, k, d + k);
  d2h(h_index, d + k, size_t(k) * 8);
  sync();
  GT_API_END
}

int gt_graph_row(const gt_graph* g, int64_t index, int in_side, int64_t* h_nbrs, int64_t cap,
                 int64_t* h_len) {
  GT_API_BEGIN
  require_init();
  if (!g || !h_len || index < 0 || index >= g->n) fail(GT_EINVAL, "bad arguments");
  const int64_t* off = in_side ? g->in_off : g->out_off;
  const int32_t* adj = in_side ? g->in_adj : g->out_adj;
  int64_t be[2];
  d2h(be, off + index, 16);
  sync();
  const int64_t len = be[1] - be[0];
  *h_len = len;
  if (!h_nbrs || cap < len || len == 0) return GT_OK;
  int64_t* d = ws_n<int64_t>(WS_TMP4, size_t(len));
  GT_LAUNCH(gtd::gl_row_kernel, std::max(1, std::min(ceil_div(len, 256), 4 * ctx().sm_count)), 256,
            0, g->ids, adj, be[0], len, d);
  d2h(h_nbrs, d, size_t(len) * 8);
  sync();
  GT_API_END
}

int gt_graph_has_edge(const gt_graph* g, int64_t src_id, int64_t dst_id, int* h_result) {
  GT_API_BEGIN
  require_init();
  if (!g || !h_result) fail(GT_EINVAL, "bad arguments");
  int64_t* d = ws_n<int64_t>(WS_SMALL, 16);
  if (g->n == 0) { *h_result = 0; return GT_OK; }
  GT_LAUNCH(gtd::gl_has_edge_kernel, 1, 1, 0, g->ids, g->n, g->out_off, g->out_adj, src_id, dst_id,
            d + 15);
  int64_t r = 0;
  d2h(&r, d + 15, 8);
  sync();
  *h_result = int(r);
  GT_API_END
}

void gt_graph_free(gt_graph* g) {
  try {
    graph_free(g);
  } catch (...) {
  }
}

}  // extern "C"

// ============================================================================
// Primitives of the multi-GPU build (paper_1503_07881_b200/distributed.py).
// One process per GPU; the host-side orchestration exchanges data with
// torch.distributed (NCCL) between these calls. All pointers are device
// pointers on the calling process's GPU; every call is stream-synchronous.
// ============================================================================
namespace gtd {

__global__ void __launch_bounds__(256) presence_flags_kernel(const int64_t* __restrict__ src,
                                                             const int64_t* __restrict__ dst,
                                                             int64_t n, int64_t lo,
                                                             uint8_t* __restrict__ flags) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    flags[ld_stream_s64(src + i) - lo] = 1;
    flags[ld_stream_s64(dst + i) - lo] = 1;
  }
}

// 32 byte flags -> one presence word (prefix filled by word_prefix_kernel).
__global__ void __launch_bounds__(256) flags_to_words_kernel(const uint8_t* __restrict__ flags,
                                                             int64_t span, uint2* __restrict__ words,
                                                             int64_t nw) {
  const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint32_t bits = 0;
  const int64_t b0 = w * 32;
  for (int j = 0; j < 32; ++j)
    if (b0 + j < span && flags[b0 + j]) bits |= 1u << j;
  words[w] = make_uint2(bits, 0u);
}

// keys - (row_lo << kbits): rows become local indices for segment_kernel.
__global__ void __launch_bounds__(256) rebase_keys_kernel(const uint64_t* __restrict__ in, int64_t n,
                                                          uint64_t sub, uint64_t* __restrict__ out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = in[i] - sub;
}

// (a << k | b) -> (b << k | a)
__global__ void __launch_bounds__(256) swap_halves_kernel(const uint64_t* __restrict__ in, int64_t n,
                                                          int kbits, uint64_t* __restrict__ out) {
  const uint64_t low = (1ull << kbits) - 1ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = in[i];
    out[i] = ((k & low) << kbits) | (k >> kbits);
  }
}

constexpr int BUCKETS_MAX = 4096;
__global__ void __launch_bounds__(256) bucket_count_kernel(const uint64_t* __restrict__ keys,
                                                           int64_t n, int shift, int nb,
                                                           unsigned long long* __restrict__ out) {
  __shared__ uint32_t sh[BUCKETS_MAX];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t b = keys[i] >> shift;
    atomicAdd(&sh[b < uint64_t(nb) ? b : uint64_t(nb - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (sh[i]) atomicAdd(&out[i], (unsigned long long)sh[i]);
}

__global__ void lower_bounds_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                    const uint64_t* __restrict__ bounds, int nb,
                                    int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const uint64_t x = bounds[i];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  out[i] = lo;
}

}  // namespace gtd

namespace gt {

static int64_t to_host_i64(const int64_t* d) { return read_i64(d); }

}  // namespace gt

extern "C" {

int gt_id_minmax(const int64_t* d_src, const int64_t* d_dst, int64_t rows, int64_t* d_out2) {
  GT_API_BEGIN
  require_init();
  if (rows < 0 || !d_out2) fail(GT_EINVAL, "bad arguments");
  const long long init[2] = {LLONG_MAX, LLONG_MIN};
  h2d(d_out2, init, sizeof init);
  if (rows > 0)
    GT_LAUNCH(gtd::minmax_kernel, grid_for(rows, 4), 256, 0, d_src, d_dst, rows,
              reinterpret_cast<long long*>(d_out2));
  sync();
  GT_API_END
}

int gt_id_presence(const int64_t* d_src, const int64_t* d_dst, int64_t rows, int64_t lo,
                   int64_t span, uint8_t* d_flags) {
  GT_API_BEGIN
  require_init();
  if (rows < 0 || span < 0 || (span > 0 && !d_flags)) fail(GT_EINVAL, "bad arguments");
  if (span) GT_CUDA(cudaMemsetAsync(d_flags, 0, size_t(span), ctx().stream));
  if (rows > 0)
    GT_LAUNCH(gtd::presence_flags_kernel, grid_for(rows, 4), 256, 0, d_src, d_dst, rows, lo,
              d_flags);
  sync();
  GT_API_END
}

int gt_id_rankmap(const uint8_t* d_flags, int64_t span, void* d_words, int64_t* n_nodes) {
  GT_API_BEGIN
  require_init();
  if (span <= 0 || !d_words || !n_nodes) fail(GT_EINVAL, "bad arguments");
  const int64_t nw = (span + 31) / 32;
  uint2* words = static_cast<uint2*>(d_words);
  GT_LAUNCH(gtd::flags_to_words_kernel, ceil_div(nw, 256), 256, 0, d_flags, span, words, nw);
  const int64_t tiles = ceil_div64(nw, 256 * 16);
  uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) + 1);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  GT_CUDA(cudaMemsetAsync(counters + 16, 0, 4, ctx().stream));
  GT_LAUNCH(gtd::word_prefix_kernel, static_cast<int>(tiles), 256, 0, words, nw, status,
            counters + 16, next_epoch(), small + 2);
  *n_nodes = to_host_i64(small + 2);
  GT_API_END
}

int gt_id_list(const void* d_words, int64_t span, int64_t lo, int64_t* d_ids) {
  GT_API_BEGIN
  require_init();
  const int64_t nw = (span + 31) / 32;
  if (nw > 0)
    GT_LAUNCH(gtd::ids_kernel, ceil_div(nw, 256), 256, 0, static_cast<const uint2*>(d_words), nw,
              lo, d_ids);
  sync();
  GT_API_END
}

int gt_pack_keys(const int64_t* d_src, const int64_t* d_dst, int64_t rows, int64_t lo,
                 const void* d_words, int kbits, uint64_t* d_keys) {
  GT_API_BEGIN
  require_init();
  if (kbits < 1 || kbits > 31) fail(GT_EINVAL, "kbits must be in [1, 31]");
  if (rows > 0)
    GT_LAUNCH(gtd::pack_kernel<true>, grid_for(rows, 4), 256, 0, d_src, d_dst, rows, lo,
              static_cast<const uint2*>(d_words), (const int64_t*)nullptr, int64_t(0), kbits,
              SortPlan(), (unsigned long long*)nullptr, d_keys);
  sync();
  GT_API_END
}

int gt_sort_keys(uint64_t* d_keys, uint64_t* d_tmp, int64_t n, int lo_bit, int hi_bit,
                 int* result_in_tmp) {
  GT_API_BEGIN
  require_init();
  if (!result_in_tmp || lo_bit < 0 || hi_bit > 64 || lo_bit > hi_bit) fail(GT_EINVAL, "bad arguments");
  SortPlan plan = make_plan(lo_bit, hi_bit);
  SortHist h = sort_hist_begin(0);
  sort_histogram(d_keys, n, plan, h);
  uint64_t* out = radix_sort(d_keys, d_tmp, n, plan, h, "dist.sort");
  *result_in_tmp = out == d_tmp ? 1 : 0;
  sync();
  GT_API_END
}

int gt_unique_keys(const uint64_t* d_in, int64_t n, uint64_t* d_out, int64_t* m) {
  GT_API_BEGIN
  require_init();
  if (!m) fail(GT_EINVAL, "m must not be NULL");
  *m = 0;
  if (n > 0) {
    const int64_t tiles = ceil_div64(n, gtd::SEG_TILE);
    uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) + 1);
    uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
    int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
    GT_CUDA(cudaMemsetAsync(counters + 17, 0, 4, ctx().stream));
    GT_LAUNCH(gtd::unique_kernel, static_cast<int>(tiles), 256, 0, d_in, n, int64_t(0),
              reinterpret_cast<int64_t*>(d_out), status, counters + 17, next_epoch(), small + 3);
    *m = to_host_i64(small + 3);
  }
  GT_API_END
}

int gt_key_bucket_counts(const uint64_t* d_keys, int64_t n, int shift, int nbuckets,
                         int64_t* d_counts) {
  GT_API_BEGIN
  require_init();
  if (nbuckets < 1 || nbuckets > gtd::BUCKETS_MAX || shift < 0 || shift > 63)
    fail(GT_EINVAL, "nbuckets must be in [1, 4096]");
  GT_CUDA(cudaMemsetAsync(d_counts, 0, size_t(nbuckets) * 8, ctx().stream));
  if (n > 0)
    GT_LAUNCH(gtd::bucket_count_kernel, grid_for(n, 8), 256, 0, d_keys, n, shift, nbuckets,
              reinterpret_cast<unsigned long long*>(d_counts));
  sync();
  GT_API_END
}

int gt_key_lower_bounds(const uint64_t* d_sorted, int64_t n, const uint64_t* h_bounds, int nb,
                        int64_t* h_out) {
  GT_API_BEGIN
  require_init();
  if (nb < 1 || nb > 4096 || !h_bounds || !h_out) fail(GT_EINVAL, "bad arguments");
  uint64_t* db = reinterpret_cast<uint64_t*>(ws_n<int64_t>(WS_TMP4, size_t(2 * nb)));
  int64_t* dout = reinterpret_cast<int64_t*>(db + nb);
  h2d(db, h_bounds, size_t(nb) * 8);
  GT_LAUNCH(gtd::lower_bounds_kernel, ceil_div(nb, 256), 256, 0, d_sorted, n, db, nb, dout);
  d2h(h_out, dout, size_t(nb) * 8);
  sync();
  GT_API_END
}

int gt_swap_key_halves(const uint64_t* d_in, int64_t n, int kbits, uint64_t* d_out) {
  GT_API_BEGIN
  require_init();
  if (n > 0) GT_LAUNCH(gtd::swap_halves_kernel, grid_for(n, 4), 256, 0, d_in, n, kbits, d_out);
  sync();
  GT_API_END
}

int gt_csr_from_keys(const uint64_t* d_sorted, int64_t m, int kbits, int64_t row_lo,
                     int64_t rows, uint64_t* d_tmp, int64_t* d_off, int32_t* d_adj) {
  GT_API_BEGIN
  require_init();
  if (rows < 0 || m < 0 || !d_off) fail(GT_EINVAL, "bad arguments");
  if (m == 0) {
    GT_CUDA(cudaMemsetAsync(d_off, 0, size_t(rows + 1) * 8, ctx().stream));
  } else {
    const uint64_t* keys = d_sorted;
    if (row_lo != 0) {
      GT_LAUNCH(gtd::rebase_keys_kernel, grid_for(m, 4), 256, 0, d_sorted, m,
                uint64_t(row_lo) << kbits, d_tmp);
      keys = d_tmp;
    }
    GT_LAUNCH(gtd::segment_kernel<false>, ceil_div(m, gtd::SEG_TILE), 256, 0, keys, m, kbits,
              rows, d_adj, d_off, (uint64_t*)nullptr, (const int64_t*)nullptr);
  }
  sync();
  GT_API_END
}

int gt_graph_from_csr(int64_t n, int64_t e, const int64_t* d_ids, const int64_t* d_out_off,
                      const int32_t* d_out_adj, const int64_t* d_in_off, const int32_t* d_in_adj,
                      gt_graph** out) {
  GT_API_BEGIN
  require_init();
  if (!out || n < 0 || e < 0) fail(GT_EINVAL, "bad arguments");
  *out = nullptr;
  if (n >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "graph has >= 2^31 nodes");
  gt_graph* g = new gt_graph();
  try {
    cudaStream_t s = ctx().stream;
    g->n = n;
    g->e = e;
    g->kbits = bits_for(n);
    g->ids = dalloc_n<int64_t>(n);
    g->out_off = dalloc_n<int64_t>(n + 1);
    g->in_off = dalloc_n<int64_t>(n + 1);
    g->out_adj = dalloc_n<int32_t>(e);
    g->in_adj = dalloc_n<int32_t>(e);
    GT_CUDA(cudaMemcpyAsync(g->ids, d_ids, size_t(n) * 8, cudaMemcpyDeviceToDevice, s));
    GT_CUDA(cudaMemcpyAsync(g->out_off, d_out_off, size_t(n + 1) * 8, cudaMemcpyDeviceToDevice, s));
    GT_CUDA(cudaMemcpyAsync(g->in_off, d_in_off, size_t(n + 1) * 8, cudaMemcpyDeviceToDevice, s));
    GT_CUDA(cudaMemcpyAsync(g->out_adj, d_out_adj, size_t(e) * 4, cudaMemcpyDeviceToDevice, s));
    GT_CUDA(cudaMemcpyAsync(g->in_adj, d_in_adj, size_t(e) * 4, cudaMemcpyDeviceToDevice, s));
    sync();
  } catch (...) {
    graph_free(g);
    throw;
  }
  *out = g;
  GT_API_END
}

}  // extern "C"

// ============================================================================
// Graph -> table (convert.py:178-217): the out-CSR
// expanded back into an edge table sorted by (src, dst), and the per-node
// table (node, out_deg, in_deg). Pure bandwidth: per edge 4 B adjacency +
// two id gathers in, 16 B out.
// ============================================================================
namespace gtd {

// Edge tiles of 2048 (coalesced: edge e0 + 256*q + tid): the tile's row
// offsets are staged in shared memory, each edge finds its row by a short
// binary search there, dst = ids[adj] is a gather from L2, src = ids[row]
// hits L1 (consecutive edges share rows).
constexpr int EXPORT_TILE = 2048;
constexpr int EXPORT_ROWS = EXPORT_TILE + 2;

__global__ void __launch_bounds__(256) export_tile_rows_kernel(const int64_t* __restrict__ off,
                                                               int64_t n, int64_t e,
                                                               int64_t tiles,
                                                               int64_t* __restrict__ tile_row) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > tiles) return;
  const int64_t x = t < tiles ? t * EXPORT_TILE : e - 1;  // row holding edge x
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  tile_row[t] = lo;
}

__global__ void __launch_bounds__(256) edge_table_kernel(const int64_t* __restrict__ ids,
                                                         const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ adj,
                                                         int64_t e,
                                                         const int64_t* __restrict__ tile_row,
                                                         int64_t* __restrict__ src,
                                                         int64_t* __restrict__ dst) {
  __shared__ int64_t s_off[EXPORT_ROWS];
  const int64_t t = blockIdx.x;
  const int64_t e0 = t * EXPORT_TILE;
  const int64_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const int64_t nr = r1 - r0 + 2;
  const bool staged = nr <= EXPORT_ROWS;
  if (staged)
    for (int i = threadIdx.x; i < int(nr); i += 256) s_off[i] = off[r0 + i];
  __syncthreads();
#pragma unroll 4
  for (int q = 0; q < EXPORT_TILE / 256; ++q) {
    const int64_t k = e0 + q * 256 + threadIdx.x;
    if (k >= e) break;
    int64_t lo = r0, hi = r1;  // largest r with off[r] <= k
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if ((staged ? s_off[mid - r0] : off[mid]) <= k) lo = mid;
      else hi = mid - 1;
    }
    src[k] = ids[lo];
    dst[k] = ids[__ldcs(adj + k)];
  }
}

__global__ void __launch_bounds__(256) node_table_kernel(const int64_t* __restrict__ out_off,
                                                         const int64_t* __restrict__ in_off,
                                                         int64_t n, int64_t* __restrict__ out_deg,
                                                         int64_t* __restrict__ in_deg) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out_deg[i] = out_off[i + 1] - out_off[i];
  in_deg[i] = in_off[i + 1] - in_off[i];
}

}  // namespace gtd

extern "C" {

int gt_graph_edge_table(const gt_graph* g, int64_t* src, int64_t* dst, int out_is_device) {
  GT_API_BEGIN
  require_init();
  if (!g) fail(GT_EINVAL, "null graph");
  if (g->e == 0) return GT_OK;
  if (!src || !dst) fail(GT_EINVAL, "output pointers must not be NULL");
  int64_t* ds = src;
  int64_t* dd = dst;
  if (!out_is_device) {
    ds = ws_n<int64_t>(WS_TMP0, size_t(2 * g->e));
    dd = ds + g->e;
  }
  {
    Phase ph("export.edges", 4.0 * g->e + 16.0 * g->e + 8.0 * g->n * 2);
    const int64_t tiles = ceil_div64(g->e, gtd::EXPORT_TILE);
    int64_t* tile_row = ws_n<int64_t>(WS_TMP1, size_t(tiles) + 1);
    GT_LAUNCH(gtd::export_tile_rows_kernel, ceil_div(tiles + 1, 256), 256, 0, g->out_off, g->n,
              g->e, tiles, tile_row);
    GT_LAUNCH(gtd::edge_table_kernel, static_cast<int>(tiles), 256, 0, g->ids, g->out_off,
              g->out_adj, g->e, tile_row, ds, dd);
  }
  if (!out_is_device) {
    d2h(src, ds, size_t(g->e) * 8);
    d2h(dst, dd, size_t(g->e) * 8);
  }
  sync();
  GT_API_END
}

int gt_graph_node_table(const gt_graph* g, int64_t* node, int64_t* out_deg, int64_t* in_deg,
                        int out_is_device) {
  GT_API_BEGIN
  require_init();
  if (!g) fail(GT_EINVAL, "null graph");
  if (g->n == 0) return GT_OK;
  if (!node || !out_deg || !in_deg) fail(GT_EINVAL, "output pointers must not be NULL");
  int64_t* od = out_deg;
  int64_t* id = in_deg;
  if (!out_is_device) {
    od = ws_n<int64_t>(WS_TMP0, size_t(2 * g->n));
    id = od + g->n;
  }
  {
    Phase ph("export.nodes", 8.0 * (g->n + 1) * 2 + 16.0 * g->n);
    GT_LAUNCH(gtd::node_table_kernel, ceil_div(g->n, 256), 256, 0, g->out_off, g->in_off, g->n,
              od, id);
  }
  if (out_is_device) {
    GT_CUDA(cudaMemcpyAsync(node, g->ids, size_t(g->n) * 8, cudaMemcpyDeviceToDevice,
                            ctx().stream));
  } else {
    d2h(node, g->ids, size_t(g->n) * 8);
    d2h(out_deg, od, size_t(g->n) * 8);
    d2h(in_deg, id, size_t(g->n) * 8);
  }
  sync();
  GT_API_END
}

}  // extern "C"
