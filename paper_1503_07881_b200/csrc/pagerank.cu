// pagerank.cu — pull-based PageRank over the in-CSR, fp64.
//
// Reference (algorithms.py:36-87):
//   contrib = score * inv_out                 (inv_out = 1/outdeg, 0 if dangling)
//   dangling = sum(score[outdeg == 0])
//   base = (1 - d)/N + d * dangling/N
//   new[v] = base + d * sum_{u in in(v)} contrib[u]      (np.bincount, algorithms.py:77-84)
//
// Device schedule per iteration (no host sync, no fp64 atomics => bitwise
// deterministic run to run):
//   pr_spmv_kernel   edge tiles of PR_TILE in-edges. The tile gathers
//                    contrib[in_adj[e]] once into shared memory (coalesced
//                    index loads, PR_TILE independent gathers in flight), then
//                    sums every row segment of the tile with a group of G lanes
//                    (G = 1..32 chosen from the tile's mean row length — the
//                    degree binning). Rows completed inside the tile are
//                    finalised in place (score/contrib/dangling partial); the
//                    partial sums of rows crossing tile edges go to head/tail.
//   pr_fixup_kernel  finishes the rows that span tiles (tail + heads of the
//                    following tiles, fixed order) and reduces the dangling
//                    mass of the new scores (fixed tree + last-block combine).
// Source relabelling (setup, once per call): nodes are renumbered by
// descending out-degree (pos[v]); the in-adjacency is rewritten in that
// numbering and the contrib vector is kept in it, so the contributions of the
// hub sources — which R-MAT puts behind most edges (C2: the top 16K sources
// feed 41% of the edges) — sit in a few hundred KB that stays in L1/L2
// instead of being spread over the whole vector. Scores stay in id order.
// HBM traffic per iteration (algorithmic): 4E (in_adj) + 8E (contrib gathers)
// + 8(N+1) (in_off) + 8N (inv_out) + 8N (contrib write) [+ 8N score, last
// iteration only].
#include "graph.cuh"
#include "radix_sort.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace gtd {

// Gathers: the head of contrib (the PR_HOT highest out-degree sources after
// the relabelling) through the L1-allocating non-coherent path, the tail with
// L1::no_allocate. Measured (scripts/sweep_const.sh): spmv C2 7.75 -> 7.48 ms,
// C4 203 -> 172 ms against __ldg for all; the split point itself did not
// matter (0 .. 2^20 within noise), while a plain no_allocate load for every
// gather compiled to a slower schedule (C2 10.7 ms).
#ifndef GT_PR_HOT_LOG
#define GT_PR_HOT_LOG 15
#endif
constexpr int PR_HOT = 1 << GT_PR_HOT_LOG;
__device__ __forceinline__ double pr_gather(const double* contrib, int32_t u) {
  if (u < PR_HOT) return __ldg(contrib + u);
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(contrib + u));
  return v;
}

// Same, with an L2 cache policy on the tail loads (createpolicy.range: the
// hot head of contrib evict_last, the rest evict_first) — L2 residency for
// the hot sources without a persisting set-aside, whose set-up and release
// (cudaDeviceSetLimit, cudaCtxResetPersistingL2Cache) synchronise the device.
__device__ __forceinline__ double pr_gather_pol(const double* contrib, int32_t u, uint64_t pol) {
  if (u < PR_HOT) return __ldg(contrib + u);
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(contrib + u), "l"(pol));
  return v;
}

// (build-time knobs for sweeps: -DGT_PR_TILE=..., -DGT_PR_MIN_BLOCKS=...)
#ifndef GT_PR_TILE
#define GT_PR_TILE 2048
#endif
#ifndef GT_PR_MIN_BLOCKS
#define GT_PR_MIN_BLOCKS 6
#endif
constexpr int PR_THREADS = 256;
constexpr int PR_TILE = GT_PR_TILE;
constexpr int PR_MIN_BLOCKS = GT_PR_MIN_BLOCKS;  // resident CTAs per SM the register budget is sized for

// Last-block deterministic reduction of one double per block.
__device__ __forceinline__ void grid_reduce_last(double block_val, double* partials,
                                                 unsigned int* ticket, double* out) {
  __shared__ bool s_last;
  __shared__ double s_red[8];
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = block_val;
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < int(gridDim.x); i += blockDim.x)
    v += *reinterpret_cast<volatile double*>(&partials[i]);
  v = block_sum_256(v, s_red);
  if (threadIdx.x == 0) {
    *out = v;
    *ticket = 0u;
  }
}

__global__ void __launch_bounds__(256) pr_init_kernel(const int64_t* __restrict__ out_off, int64_t n,
                                                      const int32_t* __restrict__ pos,
                                                      double* __restrict__ inv_out,
                                                      double* __restrict__ contrib,
                                                      double* __restrict__ partials,
                                                      unsigned int* __restrict__ ticket,
                                                      double* __restrict__ dangling0) {
  __shared__ double s_red[8];
  const double s0 = 1.0 / double(n);
  double dang = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int64_t deg = out_off[v + 1] - out_off[v];
    const double inv = deg ? 1.0 / double(deg) : 0.0;
    inv_out[v] = inv;
    contrib[pos[v]] = s0 * inv;
    if (deg == 0) dang += s0;
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling0);
}

// Relabelling keys: (max_deg - outdeg(v)) << kbits | v  -> ascending sort =
// descending out-degree, ties by id.
__global__ void __launch_bounds__(256) pr_relabel_keys_kernel(const int64_t* __restrict__ out_off,
                                                              int64_t n, int64_t max_deg, int kbits,
                                                              gt::SortPlan plan,
                                                              unsigned long long* __restrict__ hist,
                                                              uint64_t* __restrict__ keys) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const uint64_t k = (uint64_t(max_deg - (out_off[v + 1] - out_off[v])) << kbits) | uint64_t(v);
    keys[v] = k;
    plan_hist_add(sh, plan, k);
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

__global__ void __launch_bounds__(256) pr_pos_kernel(const uint64_t* __restrict__ sorted, int64_t n,
                                                     uint64_t lowmask, int32_t* __restrict__ pos) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n) pos[sorted[p] & lowmask] = int32_t(p);
}

__global__ void __launch_bounds__(256) pr_remap_kernel(const int32_t* __restrict__ in_adj, int64_t e,
                                                       const int32_t* __restrict__ pos,
                                                       int32_t* __restrict__ out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e; i += stride)
    out[i] = pos[__ldcs(in_adj + i)];
}

__global__ void __launch_bounds__(256) pr_max_outdeg_kernel(const int64_t* __restrict__ out_off,
                                                            int64_t n,
                                                            unsigned long long* __restrict__ out) {
  unsigned long long mx = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    mx = max(mx, (unsigned long long)(out_off[v + 1] - out_off[v]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// tile_row[c] = first row whose in-edges start at or after c*PR_TILE.
__global__ void __launch_bounds__(256) pr_tile_rows_kernel(const int64_t* __restrict__ in_off,
                                                           int64_t n, int64_t tiles,
                                                           int64_t* __restrict__ tile_row) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c > tiles) return;
  if (c == tiles) { tile_row[c] = n; return; }
  const int64_t e = c * PR_TILE;
  int64_t lo = 0, hi = n;  // lower_bound over in_off[0..n)
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (in_off[mid] < e) lo = mid + 1;
    else hi = mid;
  }
  tile_row[c] = lo;
}

constexpr int PR_ROWCAP = 512;   // rows of a tile whose metadata is staged on chip

// Per-tile row metadata in shared memory: relative start of every segment
// (clamped to the tile), 1/outdeg and the relabelled position of its row.
struct PrRows {
  uint16_t off[PR_ROWCAP + 1];
  double inv[PR_ROWCAP];
  int32_t pos[PR_ROWCAP];
};

// Row segments of a tile, summed from the gathered values in shared memory:
// segments shorter than PR_LONG by one thread each (serial, no shuffles),
// longer ones by a whole warp (strided + butterfly). The order of every sum
// is fixed, so results are bitwise reproducible.
constexpr int PR_LONG = 32;

__device__ __forceinline__ void pr_finish(int64_t s, double sum, const PrRows& sr,
                                          int64_t first_row, int64_t nseg, bool has_head,
                                          bool has_tail, int64_t c, double base, double damping,
                                          const double* __restrict__ inv_out,
                                          const int32_t* __restrict__ pos,
                                          double* __restrict__ score,
                                          double* __restrict__ contrib_next,
                                          double* __restrict__ head, double* __restrict__ tail,
                                          int64_t* __restrict__ tail_row, bool last_iter,
                                          double& dang) {
  const int64_t row = first_row + s;
  if (has_head && s == 0) {
    head[c] = sum;
  } else if (has_tail && s == nseg - 1) {
    tail[c] = sum;
    tail_row[c] = row;
  } else {
    const double sc = base + damping * sum;
    const double inv = s < PR_ROWCAP ? sr.inv[s] : inv_out[row];
    if (!last_iter)
      contrib_next[s < PR_ROWCAP ? sr.pos[s] : (pos ? int64_t(pos[row]) : row)] = sc * inv;
    else score[row] = sc;
    if (inv == 0.0) dang += sc;
  }
}

__device__ __forceinline__ void pr_rows(const double* vals, const PrRows& sr,
                                        const int64_t* __restrict__ in_off, int64_t e0, int ne,
                                        int64_t first_row, int64_t nseg, bool has_head,
                                        bool has_tail, int64_t c, double base, double damping,
                                        const double* __restrict__ inv_out,
                                        const int32_t* __restrict__ pos,
                                        double* __restrict__ score, double* __restrict__ contrib_next,
                                        double* __restrict__ head, double* __restrict__ tail,
                                        int64_t* __restrict__ tail_row, bool last_iter,
                                        double& dang, int ltid) {
  const int warp = ltid >> 5, lane = ltid & 31;
  auto off_at = [&](int64_t r) -> int {
    if (r < PR_ROWCAP + 1) return sr.off[r];
    const int64_t x = in_off[first_row + r] - e0;
    return int(x < 0 ? 0 : (x > ne ? ne : x));
  };
  // short segments: thread per segment
  for (int64_t s = ltid; s < nseg; s += PR_THREADS) {
    const int a = off_at(s), b = off_at(s + 1);
    if (b - a >= PR_LONG) continue;
    double sum = 0.0;
    for (int j = a; j < b; ++j) sum += vals[j];
    pr_finish(s, sum, sr, first_row, nseg, has_head, has_tail, c, base, damping, inv_out, pos,
              score, contrib_next, head, tail, tail_row, last_iter, dang);
  }
  // long segments: warp per segment
  for (int64_t s = warp; s < nseg; s += PR_THREADS / 32) {
    const int a = off_at(s), b = off_at(s + 1);
    if (b - a < PR_LONG) continue;  // warp-uniform
    double sum = 0.0;
    for (int j = a + lane; j < b; j += 32) sum += vals[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0)
      pr_finish(s, sum, sr, first_row, nseg, has_head, has_tail, c, base, damping, inv_out, pos,
                score, contrib_next, head, tail, tail_row, last_iter, dang);
  }
}

// One tile of PR_TILE in-edges, processed by a group of PR_THREADS threads
// (ltid = thread index in the group, bar() = the group's barrier). Gathers
// come from contrib through pr_gather.
template <typename Bar>
__device__ __forceinline__ void pr_tile(
    int64_t c, int ltid, Bar bar, double* vals, PrRows& sr,
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_adj, int64_t n, int64_t e,
    const int64_t* __restrict__ tile_row, const double* __restrict__ contrib,
    const double* __restrict__ inv_out, const int32_t* __restrict__ pos, double base,
    double damping, double* __restrict__ score, double* __restrict__ contrib_next,
    double* __restrict__ head, double* __restrict__ tail, int64_t* __restrict__ tail_row,
    double* __restrict__ dpart, bool last, uint32_t hot_bytes, uint32_t total_bytes) {
  const int64_t e0 = c * PR_TILE;
  const int64_t e1 = min(e, e0 + PR_TILE);
  const int ne = e1 > e0 ? int(e1 - e0) : 0;
  const int64_t ra = tile_row[c], rb = tile_row[c + 1];
  if (ltid == 0) tail_row[c] = -1;
  // segments: the head row ra-1 (starts before the tile) when it reaches
  // into it, then rows ra..rb-1 (start inside); the last may run past e1
  const bool has_head = ne > 0 && (ra == n || in_off[ra] > e0);
  const int64_t first_row = has_head ? ra - 1 : ra;
  const int64_t nseg = rb - first_row;
  const bool has_tail = nseg > 0 && in_off[rb] > e1 && !(has_head && nseg == 1);

  // Gather phase: PR_TILE/PR_THREADS independent loads per thread in flight,
  // and the tile's row metadata staged alongside (independent of the gathers).
  constexpr int PER = PR_TILE / PR_THREADS;
  int32_t idx[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = i * PR_THREADS + ltid;
    idx[i] = j < ne ? __ldcs(in_adj + e0 + j) : 0;
  }
  const int64_t nstage = min(nseg + 1, int64_t(PR_ROWCAP + 1));
  for (int64_t r = ltid; r < nstage; r += PR_THREADS) {
    const int64_t row = first_row + r;
    const int64_t x = in_off[row] - e0;
    sr.off[r] = uint16_t(x < 0 ? 0 : (x > ne ? ne : x));
    if (r < nseg && r < PR_ROWCAP) {
      sr.inv[r] = inv_out[row];
      sr.pos[r] = pos ? pos[row] : int32_t(row);
    }
  }
  if (hot_bytes) {
    uint64_t pol;
    asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
                 : "=l"(pol) : "l"(contrib), "r"(hot_bytes), "r"(total_bytes));
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = i * PR_THREADS + ltid;
      if (j < ne) vals[j] = pr_gather_pol(contrib, idx[i], pol);
    }
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = i * PR_THREADS + ltid;
      if (j < ne) vals[j] = pr_gather(contrib, idx[i]);
    }
  }
  bar();

  double dang = 0.0;
  pr_rows(vals, sr, in_off, e0, ne, first_row, nseg, has_head, has_tail, c, base, damping,
          inv_out, pos, score, contrib_next, head, tail, tail_row, last, dang, ltid);
  // per-warp dangling partials (summed in a fixed order by the fixup kernel):
  // no barrier at the end of the tile
  dang = warp_sum(dang);
  if ((ltid & 31) == 0) dpart[c * (PR_THREADS / 32) + (ltid >> 5)] = dang;
}

__global__ void __launch_bounds__(PR_THREADS, PR_MIN_BLOCKS) pr_spmv_kernel(
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_adj, int64_t n, int64_t e,
    int64_t n_total, const int64_t* __restrict__ tile_row, const double* __restrict__ contrib,
    const double* __restrict__ inv_out, const int32_t* __restrict__ pos,
    const double* __restrict__ dangling_prev, double damping,
    double* __restrict__ score, double* __restrict__ contrib_next, double* __restrict__ head,
    double* __restrict__ tail, int64_t* __restrict__ tail_row, double* __restrict__ dpart,
    int last_iter, uint32_t hot_bytes, uint32_t total_bytes, int pf_dist) {
  __shared__ double vals[PR_TILE];
  __shared__ PrRows sr;
  const double base =
      (1.0 - damping) / double(n_total) + damping * (*dangling_prev / double(n_total));
  // GT_PR_PF (off by default, measured no gain): CTAs start in blockIdx order;
  // the indices of a tile pf_dist ahead are pulled into L2
  if (threadIdx.x == 0 && pf_dist > 0 && (int64_t(blockIdx.x) + pf_dist + 1) * PR_TILE <= e)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                     in_adj + (int64_t(blockIdx.x) + pf_dist) * PR_TILE),
                 "r"(PR_TILE * 4)
                 : "memory");
  pr_tile(int64_t(blockIdx.x), int(threadIdx.x), [] { __syncthreads(); }, vals, sr, in_off,
          in_adj, n, e, tile_row, contrib, inv_out, pos, base, damping, score, contrib_next, head,
          tail, tail_row, dpart, last_iter != 0, hot_bytes, total_bytes);
}

__global__ void __launch_bounds__(256) pr_fixup_kernel(
    const int64_t* __restrict__ in_off, int64_t n, int64_t n_total, int64_t tiles,
    const double* __restrict__ inv_out, const int32_t* __restrict__ pos,
    const double* __restrict__ dangling_prev, double damping,
    const double* __restrict__ head, const double* __restrict__ tail,
    const int64_t* __restrict__ tail_row, const double* __restrict__ dpart,
    double* __restrict__ score, double* __restrict__ contrib_next, int last_iter,
    double* __restrict__ partials, unsigned int* __restrict__ ticket,
    double* __restrict__ dangling_next) {
  __shared__ double s_red[8];
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const double base =
      (1.0 - damping) / double(n_total) + damping * (*dangling_prev / double(n_total));
  double dang = 0.0;
  if (c < tiles) {
#pragma unroll
    for (int w = 0; w < PR_THREADS / 32; ++w) dang += dpart[c * (PR_THREADS / 32) + w];
    const int64_t v = tail_row[c];
    if (v >= 0) {
      const int64_t c_last = (in_off[v + 1] - 1) / PR_TILE;
      double sum = tail[c];
      for (int64_t c2 = c + 1; c2 <= c_last; ++c2) sum += head[c2];
      const double sc = base + damping * sum;
      const double inv = inv_out[v];
      if (last_iter) score[v] = sc;
      else contrib_next[pos ? int64_t(pos[v]) : v] = sc * inv;
      if (inv == 0.0) dang += sc;
    }
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling_next);
}

// ============================================================================
// Cache-blocked pull (contrib larger than L2): the relabelled sources are cut
// into segments of SEG = 2^sb positions (SEG * 8 B <= half of L2). Each
// segment's in-edges are kept as a doubly-compressed CSR — only the dst rows
// that have an in-edge from the segment (drow[h], dstart[h]) — so a pass
// over a segment touches its edges and those rows only. Per iteration the
// segments run in order: every gather hits the L2-resident slice of contrib;
// each row's partial sum is added to acc[row] once per segment (fixed order:
// deterministic), and a finalize pass turns acc into scores / contributions.
// ============================================================================

// keys[e] = row << 32 | pos (pos = relabelled source) in row-major in-CSR
// order, + the digit histogram of the segment id (bits [sb, sb+nb) of pos).
// Rows per tile from the scattered row heads + a block max-scan.
__global__ void __launch_bounds__(256) pr_blk_keys_kernel(
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ adj, int64_t n, int64_t e,
    const int64_t* __restrict__ tile_row, gt::SortPlan plan, unsigned long long* __restrict__ hist,
    uint64_t* __restrict__ keys) {
  __shared__ int32_t s_row[PR_TILE];
  __shared__ uint32_t sh[256];
  __shared__ int32_t s_w[8];
  for (int i = threadIdx.x; i < 256; i += 256) sh[i] = 0;
  const int64_t tiles = (e + PR_TILE - 1) / PR_TILE;
  for (int64_t c = blockIdx.x; c < tiles; c += gridDim.x) {
    const int64_t e0 = c * PR_TILE;
    const int ne = int(min(int64_t(PR_TILE), e - e0));
    const int64_t ra = tile_row[c], rb = tile_row[c + 1];
    for (int i = threadIdx.x; i < PR_TILE; i += 256) s_row[i] = -1;
    __syncthreads();
    // the row running into the tile (if any) starts at slot 0
    if (threadIdx.x == 0 && (ra == n || in_off[ra] > e0)) s_row[0] = int32_t(ra - 1);
    for (int64_t r = ra + threadIdx.x; r < rb; r += 256) {
      const int64_t x = in_off[r] - e0;
      if (x < ne) atomicMax(&s_row[x], int32_t(r));  // empty rows share a start: keep the last
    }
    __syncthreads();
    // inclusive max-scan over the tile (8 per thread)
    constexpr int PER = PR_TILE / 256;
    int32_t v[PER], m = -1;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      v[q] = s_row[threadIdx.x * PER + q];
      m = max(m, v[q]);
      v[q] = m;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t inc = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = max(inc, u);
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    int32_t pre = -1;
    for (int q = 0; q < w; ++q) pre = max(pre, s_w[q]);
    const int32_t ex = max(pre, __shfl_up_sync(0xffffffffu, inc, 1));
    const int32_t carry = lane == 0 ? pre : ex;
#pragma unroll
    for (int q = 0; q < PER; ++q) s_row[threadIdx.x * PER + q] = max(carry, v[q]);
    __syncthreads();
    for (int j = threadIdx.x; j < ne; j += 256) {
      const uint32_t pos = uint32_t(__ldcs(adj + e0 + j));
      const uint64_t k = (uint64_t(uint32_t(s_row[j])) << 32) | pos;
      keys[e0 + j] = k;
      atomicAdd(&sh[(pos >> plan.shift[0]) & ((1u << plan.bits[0]) - 1u)], 1u);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < (1 << plan.bits[0]); i += 256)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// Segment-major keys -> sadj (positions), DCSR heads (row changes or segment
// changes): drow[h] = row, dstart[h] = first edge. Decoupled look-back over
// 4096-key tiles for the head indices.
__global__ void __launch_bounds__(256) pr_blk_dcsr_kernel(
    const uint64_t* __restrict__ keys, int64_t e, int sb, int32_t* __restrict__ sadj,
    int32_t* __restrict__ drow, int64_t* __restrict__ dstart, uint64_t* __restrict__ status,
    uint32_t* __restrict__ counter, uint32_t epoch, int64_t* __restrict__ total_out) {
  constexpr int KPT = 16, T = 256 * KPT;
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = int(s_tile);
  const int64_t wbase = int64_t(tile) * T + int64_t(warp) * 32 * KPT;
  const unsigned lt = lanemask_lt();
  uint32_t heads = 0, before[KPT], run = 0;
  uint64_t k[KPT];
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    k[i] = idx < e ? keys[idx] : 0ull;
  }
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    bool h = false;
    if (idx < e) {
      sadj[idx] = int32_t(uint32_t(k[i]));
      if (idx == 0) {
        h = true;
      } else {
        const uint64_t pk = keys[idx - 1];
        h = (pk >> 32) != (k[i] >> 32) || ((uint32_t(pk) >> sb) != (uint32_t(k[i]) >> sb));
      }
    }
    heads |= uint32_t(h) << i;
    const uint32_t bal = __ballot_sync(0xffffffffu, h);
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
    if (int64_t(tile) == (e - 1) / T) *total_out = int64_t(s_excl) + tcount;
  }
  __syncthreads();
  const int64_t base = int64_t(s_excl) + wpre;
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    if ((heads >> i) & 1u) {
      const int64_t h = base + before[i];
      drow[h] = int32_t(k[i] >> 32);
      dstart[h] = wbase + i * 32 + lane;
    }
  }
}

// Per segment s (thread): first DCSR head of the segment, and per tile of the
// segment, the first head starting at or after the tile (one thread each).
__global__ void pr_blk_tiles_kernel(const int64_t* __restrict__ dstart, int64_t nh,
                                    const int64_t* __restrict__ ebeg, const int64_t* __restrict__ tbeg,
                                    int nseg, int64_t* __restrict__ hbeg,
                                    int64_t* __restrict__ tile_head) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ntiles = tbeg[nseg];
  auto lb = [&](int64_t x) {  // first head with dstart >= x
    int64_t lo = 0, hi = nh;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (dstart[m] < x) lo = m + 1;
      else hi = m;
    }
    return lo;
  };
  if (t <= nseg) hbeg[t] = lb(ebeg[t]);
  if (t == ntiles) tile_head[t] = nh;
  if (t < ntiles) {
    int s = 0;
    while (tbeg[s + 1] <= t) ++s;  // nseg is small
    tile_head[t] = lb(ebeg[s] + (t - tbeg[s]) * PR_TILE);
  }
}

// One segment: edge tiles over [e_lo, e_hi) (tiles gt0..), DCSR heads
// [h_lo, h_hi). Complete rows add their sum to acc[row]; rows crossing a tile
// edge leave head/tail partials for pr_blk_fixup_kernel.
__global__ void __launch_bounds__(PR_THREADS, PR_MIN_BLOCKS) pr_blk_spmv_kernel(
    const int32_t* __restrict__ sadj, const int32_t* __restrict__ drow,
    const int64_t* __restrict__ dstart, int64_t e_lo, int64_t e_hi, int64_t h_hi, int64_t gt0,
    const int64_t* __restrict__ tile_head, const double* __restrict__ contrib,
    double* __restrict__ acc, double* __restrict__ head, double* __restrict__ tail,
    int64_t* __restrict__ tail_h) {
  __shared__ double vals[PR_TILE];
  __shared__ uint16_t s_off[PR_ROWCAP + 1];
  const int ltid = threadIdx.x, warp = ltid >> 5, lane = ltid & 31;
  const int64_t gt = gt0 + blockIdx.x;
  const int64_t e0 = e_lo + int64_t(blockIdx.x) * PR_TILE;
  const int ne = int(min(int64_t(PR_TILE), e_hi - e0));
  const int64_t ha = tile_head[gt], hb = tile_head[gt + 1];
  if (ltid == 0) tail_h[gt] = -1;
  const bool has_head = ha == h_hi || dstart[ha] > e0;  // a row runs into the tile
  const int64_t first = has_head ? ha - 1 : ha;
  const int64_t nseg = hb - first;
  auto end_of = [&](int64_t h) { return h + 1 < h_hi ? dstart[h + 1] : e_hi; };
  const bool has_tail = nseg > 0 && end_of(hb - 1) > e0 + ne && !(has_head && nseg == 1);
  constexpr int PER = PR_TILE / PR_THREADS;
  int32_t idx[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = i * PR_THREADS + ltid;
    idx[i] = j < ne ? __ldcs(sadj + e0 + j) : 0;
  }
  const int64_t nstage = min(nseg + 1, int64_t(PR_ROWCAP + 1));
  for (int64_t r = ltid; r < nstage; r += PR_THREADS) {
    const int64_t x = (first + r < h_hi ? dstart[first + r] : e_hi) - e0;
    s_off[r] = uint16_t(x < 0 ? 0 : (x > ne ? ne : x));
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = i * PR_THREADS + ltid;
    if (j < ne) vals[j] = __ldg(contrib + idx[i]);
  }
  __syncthreads();
  auto off_at = [&](int64_t r) -> int {
    if (r < PR_ROWCAP + 1) return s_off[r];
    const int64_t x = (first + r < h_hi ? dstart[first + r] : e_hi) - e0;
    return int(x < 0 ? 0 : (x > ne ? ne : x));
  };
  auto finish = [&](int64_t sgi, double sum) {
    if (has_head && sgi == 0) {
      head[gt] = sum;
    } else if (has_tail && sgi == nseg - 1) {
      tail[gt] = sum;
      tail_h[gt] = first + sgi;
    } else {
      acc[drow[first + sgi]] += sum;
    }
  };
  for (int64_t sg = ltid; sg < nseg; sg += PR_THREADS) {
    const int a = off_at(sg), b = off_at(sg + 1);
    if (b - a >= PR_LONG) continue;
    double sum = 0.0;
    for (int j = a; j < b; ++j) sum += vals[j];
    finish(sg, sum);
  }
  for (int64_t sg = warp; sg < nseg; sg += PR_THREADS / 32) {
    const int a = off_at(sg), b = off_at(sg + 1);
    if (b - a < PR_LONG) continue;  // warp-uniform
    double sum = 0.0;
    for (int j = a + lane; j < b; j += 32) sum += vals[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) finish(sg, sum);
  }
}

__global__ void __launch_bounds__(256) pr_blk_fixup_kernel(
    const int32_t* __restrict__ drow, const int64_t* __restrict__ dstart, int64_t e_lo,
    int64_t e_hi, int64_t h_hi, int64_t gt0, int64_t ntiles, const double* __restrict__ head,
    const double* __restrict__ tail, const int64_t* __restrict__ tail_h, double* __restrict__ acc) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= ntiles) return;
  const int64_t h = tail_h[gt0 + c];
  if (h < 0) return;
  const int64_t end = h + 1 < h_hi ? dstart[h + 1] : e_hi;
  const int64_t c_last = (end - 1 - e_lo) / PR_TILE;
  double sum = tail[gt0 + c];
  for (int64_t c2 = c + 1; c2 <= c_last; ++c2) sum += head[gt0 + c2];
  acc[drow[h]] += sum;
}

// acc -> scores (last iteration) or next contributions; acc cleared; the
// dangling mass of the new scores reduced in a fixed tree.
__global__ void __launch_bounds__(256) pr_blk_finalize_kernel(
    int64_t n, double* __restrict__ acc, const double* __restrict__ inv_out,
    const int32_t* __restrict__ pos, const double* __restrict__ dangling_prev, double damping,
    int last_iter, double* __restrict__ score, double* __restrict__ contrib_next,
    double* __restrict__ partials, unsigned int* __restrict__ ticket,
    double* __restrict__ dangling_next) {
  __shared__ double s_red[8];
  const double base = (1.0 - damping) / double(n) + damping * (*dangling_prev / double(n));
  double dang = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const double sc = base + damping * acc[v];
    acc[v] = 0.0;
    const double inv = inv_out[v];
    if (last_iter) score[v] = sc;
    else contrib_next[pos[v]] = sc * inv;
    if (inv == 0.0) dang += sc;
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling_next);
}

// Multi-GPU PageRank exchange layout: node v owned by rank r (bounds[r] <= v
// < bounds[r+1]) sits at padded position r*m + (v - bounds[r]) of the
// all-gathered contribution buffer (one equal-size chunk per rank).
__global__ void __launch_bounds__(256) pr_remap_padded_kernel(const int32_t* __restrict__ in,
                                                              int64_t e,
                                                              const int64_t* __restrict__ bounds,
                                                              int world, int64_t m,
                                                              int32_t* __restrict__ out) {
  __shared__ int64_t sb[65];
  for (int i = threadIdx.x; i <= world && i < 65; i += blockDim.x) sb[i] = bounds[i];
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e; i += stride) {
    const int64_t v = in[i];
    int r = 0;
    while (r + 1 < world && sb[r + 1] <= v) ++r;
    out[i] = int32_t(int64_t(r) * m + (v - sb[r]));
  }
}

// Distributed PageRank helpers: 1/outdeg of a CSR row range, and the start
// vector (contrib = inv/N) with its dangling mass, from a full 1/outdeg vector.
__global__ void __launch_bounds__(256) pr_inv_degree_kernel(const int64_t* __restrict__ off,
                                                            int64_t rows,
                                                            double* __restrict__ inv) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= rows) return;
  const int64_t d = off[v + 1] - off[v];
  inv[v] = d ? 1.0 / double(d) : 0.0;
}

__global__ void __launch_bounds__(256) pr_init_from_inv_kernel(const double* __restrict__ inv,
                                                               int64_t n,
                                                               double* __restrict__ contrib,
                                                               double* __restrict__ partials,
                                                               unsigned int* __restrict__ ticket,
                                                               double* __restrict__ dangling0) {
  __shared__ double s_red[8];
  const double s0 = 1.0 / double(n);
  double dang = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const double iv = inv[v];
    contrib[v] = s0 * iv;
    if (iv == 0.0) dang += s0;
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling0);
}

}  // namespace gtd

namespace gtd {

// ---- push within L2-sized destination bins ------------------------------------
// The edges of the out-CSR, stably grouped by destination bin (a range of
// 2^rb ids whose accumulators fit in L2): inside a bin they stay in (src,
// dst) order, so one bin's pass reads contrib[] as a forward sweep (every
// sector once per bin, instead of one random 32-byte sector per edge in the
// pull) and adds into accumulators that stay in L2. The additions are fp64
// reductions in L2 (no return value), so the summation order — and the last
// bits of the scores — vary from run to run; the result stays within the
// 1e-9 L1 tolerance of the reference (north star).
__global__ void __launch_bounds__(256) pr_push_keys_kernel(const int64_t* __restrict__ out_off,
                                                           const int32_t* __restrict__ out_adj,
                                                           int64_t n, int kbits, gt::SortPlan plan,
                                                           unsigned long long* __restrict__ hist,
                                                           uint64_t* __restrict__ keys) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t u = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); u < n; u += nw) {
    const uint64_t hi = uint64_t(u) << kbits;
    for (int64_t j = out_off[u] + lane; j < out_off[u + 1]; j += 32) {
      const uint64_t k = hi | uint64_t(uint32_t(out_adj[j]));
      keys[j] = k;
      plan_hist_add(sh, plan, k);
    }
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

// Out-degree log2 buckets: node count and degree sum per bucket (the push /
// pull choice estimates from them how many edges the hottest sources cover).
__global__ void __launch_bounds__(256) pr_degree_buckets_kernel(const int64_t* __restrict__ out_off,
                                                                int64_t n,
                                                                unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_c[64], s_d[64];
  if (threadIdx.x < 64) {
    s_c[threadIdx.x] = 0;
    s_d[threadIdx.x] = 0;
  }
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int64_t d = out_off[v + 1] - out_off[v];
    const int b = d > 0 ? 64 - __clzll(d) : 0;  // 0 for empty rows, else floor(log2 d) + 1
    atomicAdd(&s_c[b], 1ull);
    atomicAdd(&s_d[b], (unsigned long long)d);
  }
  __syncthreads();
  if (threadIdx.x < 64 && s_c[threadIdx.x]) {
    atomicAdd(&out[threadIdx.x], s_c[threadIdx.x]);
    atomicAdd(&out[64 + threadIdx.x], s_d[threadIdx.x]);
  }
}

__global__ void __launch_bounds__(256) pr_iota_kernel(int64_t n, int32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = int32_t(i);
}

__global__ void __launch_bounds__(256) pr_push_kernel(const uint64_t* __restrict__ keys,
                                                      int64_t cnt, int kbits,
                                                      const double* __restrict__ contrib,
                                                      double* __restrict__ acc) {
  const uint64_t mask = (1ull << kbits) - 1ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt; i += stride) {
    const uint64_t k = ld_stream_u64(keys + i);
    atomicAdd(acc + (k & mask), __ldg(contrib + (k >> kbits)));
  }
}

// scores from the accumulators; accumulators cleared for the next iteration
__global__ void __launch_bounds__(256) pr_push_finish_kernel(
    double* __restrict__ acc, int64_t n, const double* __restrict__ inv_out,
    const double* __restrict__ dangling_prev, double damping, int last,
    double* __restrict__ score, double* __restrict__ contrib_next, double* __restrict__ partials,
    unsigned int* __restrict__ ticket, double* __restrict__ dangling_out) {
  __shared__ double s_red[8];
  const double base = (1.0 - damping) / double(n) + damping * (*dangling_prev / double(n));
  double dang = 0.0;
  // 4 consecutive ids per thread step, every load issued before use
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * 4;
  for (int64_t v0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; v0 < n; v0 += stride) {
    double a[4], inv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = v0 + q < n ? acc[v0 + q] : 0.0;
      inv[q] = v0 + q < n ? inv_out[v0 + q] : 1.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (v0 + q >= n) break;
      const double sc = base + damping * a[q];
      acc[v0 + q] = 0.0;
      if (last) score[v0 + q] = sc;
      else contrib_next[v0 + q] = sc * inv[q];
      if (inv[q] == 0.0) dang += sc;
    }
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling_out);
}

}  // namespace gtd

namespace gt {

// The cache-blocked iterations (contrib larger than ~half of L2).
static void pagerank_blocked(const gt_graph* g, double damping, int iterations, int sb,
                             int64_t nseg, int64_t tiles, const int64_t* tile_row,
                             int32_t* in_adj_r, const int32_t* pos, const double* inv_out,
                             double* const contrib[2], double* dang, double* partials,
                             unsigned int* ticket, double* score, int fin_blocks) {
  cudaStream_t st = ctx().stream;
  const int64_t n = g->n, e = g->e;
  const int sms = ctx().sm_count;
  // segment-major edge order: one stable radix pass on the segment digit
  SortPlan plan = make_plan(sb, sb + bits_for(nseg));
  if (plan.passes != 1) fail(GT_EINVAL, "pagerank: too many source segments");
  SortHist hs = sort_hist_begin(0);
  uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(e));
  uint64_t* kb = ws_n<uint64_t>(WS_KEYS_B, size_t(e));
  {
    Phase ph("pr.block", 12.0 * e + 8.0 * e);
    GT_LAUNCH(gtd::pr_blk_keys_kernel, static_cast<int>(std::min<int64_t>(tiles, sms * 8)), 256, 0,
              g->in_off, in_adj_r, n, e, tile_row, plan, hs.hist, ka);
  }
  const uint64_t* sorted = radix_sort(ka, kb, e, plan, hs, "pr.block");
  std::vector<int64_t> ebeg(size_t(nseg) + 1);
  d2h(ebeg.data(), hs.digit_base, size_t(nseg) * 8);
  sync();
  ebeg[size_t(nseg)] = e;
  std::vector<int64_t> tbeg(size_t(nseg) + 1, 0);
  for (int64_t s = 0; s < nseg; ++s)
    tbeg[size_t(s + 1)] = tbeg[size_t(s)] + ceil_div64(ebeg[size_t(s + 1)] - ebeg[size_t(s)], gtd::PR_TILE);
  const int64_t ntiles = tbeg[size_t(nseg)];
  const int64_t hcap = std::min<int64_t>(e, nseg * n) + 1;
  char* p = static_cast<char*>(dalloc(size_t(hcap) * 12 + size_t(ntiles + 2) * 32 +
                                      size_t(nseg + 2) * 24 + size_t(n) * 8 + 512));
  char* p0 = p;
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  int64_t* dstart = reinterpret_cast<int64_t*>(carve(size_t(hcap) * 8));
  int32_t* drow = reinterpret_cast<int32_t*>(carve(size_t(hcap) * 4));
  int64_t* tile_head = reinterpret_cast<int64_t*>(carve(size_t(ntiles + 2) * 8));
  double* head = reinterpret_cast<double*>(carve(size_t(ntiles + 1) * 8));
  double* tail = reinterpret_cast<double*>(carve(size_t(ntiles + 1) * 8));
  int64_t* tail_h = reinterpret_cast<int64_t*>(carve(size_t(ntiles + 1) * 8));
  int64_t* d_ebeg = reinterpret_cast<int64_t*>(carve(size_t(nseg + 1) * 8));
  int64_t* d_tbeg = reinterpret_cast<int64_t*>(carve(size_t(nseg + 1) * 8));
  int64_t* d_hbeg = reinterpret_cast<int64_t*>(carve(size_t(nseg + 1) * 8));
  double* acc = reinterpret_cast<double*>(carve(size_t(n) * 8));
  int32_t* sadj = in_adj_r;  // positions in segment-major order (in_adj_r is consumed)
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  {
    Phase ph("pr.block", 8.0 * e + 4.0 * e);
    const int64_t t16 = ceil_div64(e, 4096);
    uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(t16) + 2);
    uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
    GT_CUDA(cudaMemsetAsync(counters + 20, 0, 4, st));
    GT_LAUNCH(gtd::pr_blk_dcsr_kernel, static_cast<int>(t16), 256, 0, sorted, e, sb, sadj, drow,
              dstart, status, counters + 20, next_epoch(), small + 14);
  }
  int64_t nh = 0;
  d2h(&nh, small + 14, 8);
  h2d(d_ebeg, ebeg.data(), ebeg.size() * 8);
  h2d(d_tbeg, tbeg.data(), tbeg.size() * 8);
  sync();
  if (nh > hcap) fail(GT_ECUDA, "pagerank: DCSR overflow (internal error)");
  {
    const int64_t nt = std::max<int64_t>(ntiles + 1, nseg + 1);
    GT_LAUNCH(gtd::pr_blk_tiles_kernel, ceil_div(nt, 256), 256, 0, dstart, nh, d_ebeg, d_tbeg,
              int(nseg), d_hbeg, tile_head);
  }
  std::vector<int64_t> hbeg(size_t(nseg) + 1);
  d2h(hbeg.data(), d_hbeg, hbeg.size() * 8);
  GT_CUDA(cudaMemsetAsync(acc, 0, size_t(n) * 8, st));
  sync();
  for (int it = 0; it < iterations; ++it) {
    const int last = it == iterations - 1;
    const double* cur = contrib[it & 1];
    double* nxt = contrib[(it + 1) & 1];
    for (int64_t s = 0; s < nseg; ++s) {
      const int64_t nt = tbeg[size_t(s + 1)] - tbeg[size_t(s)];
      if (nt == 0) continue;
      const int64_t el = ebeg[size_t(s)], eh = ebeg[size_t(s + 1)];
      const int64_t hh = hbeg[size_t(s + 1)], hl = hbeg[size_t(s)];
      {
        Phase ph("pr.spmv", 12.0 * double(eh - el) + 28.0 * double(hh - hl));
        GT_LAUNCH(gtd::pr_blk_spmv_kernel, static_cast<int>(nt), gtd::PR_THREADS, 0, sadj, drow,
                  dstart, el, eh, hh, tbeg[size_t(s)], tile_head, cur, acc, head, tail, tail_h);
      }
      {
        Phase ph("pr.fixup", 32.0 * double(nt));
        GT_LAUNCH(gtd::pr_blk_fixup_kernel, ceil_div(nt, 256), 256, 0, drow, dstart, el, eh, hh,
                  tbeg[size_t(s)], nt, head, tail, tail_h, acc);
      }
    }
    {
      Phase ph("pr.finalize", 32.0 * double(n));
      GT_LAUNCH(gtd::pr_blk_finalize_kernel, fin_blocks, 256, 0, n, acc, inv_out, pos, dang + it,
                damping, last, score, nxt, partials, ticket, dang + it + 1);
    }
  }
  dfree(p0);
}

// Push within destination bins (see pr_push_kernel); rb = log2(rows per bin).
static void pagerank_push(const gt_graph* g, double damping, int iterations, int rb,
                          double* score) {
  cudaStream_t st = ctx().stream;
  const int64_t n = g->n, e = g->e;
  const int kb = bits_for(n);
  const int sms = ctx().sm_count;
  const int init_blocks = static_cast<int>(std::min<int64_t>(ceil_div64(n, 256), 16LL * sms));
  SortPlan plan = make_plan(rb, kb);  // 0 passes: one bin, out-CSR order as is
  if (plan.passes > 1) fail(GT_EINVAL, "pagerank: too many destination bins");
  const int64_t nbins = plan.passes ? ceil_div64(n, int64_t(1) << rb) : 1;
  SortHist hs = sort_hist_begin(0);
  uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(e));
  uint64_t* kb_ = plan.passes ? ws_n<uint64_t>(WS_KEYS_B, size_t(e)) : nullptr;
  {
    Phase ph("pr.push_setup", 12.0 * e + 8.0 * (n + 1));
    GT_LAUNCH(gtd::pr_push_keys_kernel, static_cast<int>(std::min<int64_t>(ceil_div64(n, 8), 8LL * sms)),
              256, 0, g->out_off, g->out_adj, n, kb, plan, hs.hist, ka);
  }
  const uint64_t* keys = plan.passes ? radix_sort(ka, kb_, e, plan, hs, "pr.push_setup") : ka;
  std::vector<int64_t> bs(size_t(nbins) + 1, 0);
  if (plan.passes) {
    d2h(bs.data(), hs.digit_base, size_t(nbins) * 8);
    sync();
  }
  bs[size_t(nbins)] = e;
  const size_t bytes = size_t(n) * 8 * 4 + size_t(iterations + 2) * 8 + size_t(init_blocks) * 8 + 256;
  char* p = static_cast<char*>(ws_get(WS_TMP1, bytes));
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  double* inv_out = reinterpret_cast<double*>(carve(size_t(n) * 8));
  double* contrib[2] = {reinterpret_cast<double*>(carve(size_t(n) * 8)),
                        reinterpret_cast<double*>(carve(size_t(n) * 8))};
  double* acc = reinterpret_cast<double*>(carve(size_t(n) * 8));
  double* dang = reinterpret_cast<double*>(carve(size_t(iterations + 2) * 8));
  double* partials = reinterpret_cast<double*>(carve(size_t(init_blocks) * 8));
  unsigned int* ticket = reinterpret_cast<unsigned int*>(carve(16));
  int32_t* ident = ws_n<int32_t>(WS_TMP4, size_t(n));
  GT_CUDA(cudaMemsetAsync(ticket, 0, 16, st));
  GT_CUDA(cudaMemsetAsync(acc, 0, size_t(n) * 8, st));
  {
    Phase ph("pr.setup", 8.0 * (n + 1) + 20.0 * n);
    GT_LAUNCH(gtd::pr_iota_kernel, ceil_div(n, 256), 256, 0, n, ident);
    GT_LAUNCH(gtd::pr_init_kernel, init_blocks, 256, 0, g->out_off, n, ident, inv_out, contrib[0],
              partials, ticket, dang);
  }
  const int push_grid = 8 * sms;
  for (int it = 0; it < iterations; ++it) {
    const int last = it == iterations - 1;
    double* cur = contrib[it & 1];
    double* nxt = contrib[(it + 1) & 1];
    {
      // DRAM bytes: the keys (8 per edge), one forward sweep of contrib per
      // bin; the reductions land in L2 (the accumulators' write-back is in
      // pr.fixup's 32 bytes per node)
      Phase ph("pr.spmv", 8.0 * e + 8.0 * n * double(nbins));
      for (int64_t b = 0; b < nbins; ++b) {
        const int64_t c = bs[size_t(b + 1)] - bs[size_t(b)];
        if (c > 0)
          GT_LAUNCH(gtd::pr_push_kernel, static_cast<int>(std::min<int64_t>(ceil_div64(c, 256), push_grid)),
                    256, 0, keys + bs[size_t(b)], c, kb, cur, acc);
      }
    }
    {
      Phase ph("pr.fixup", 32.0 * n);
      GT_LAUNCH(gtd::pr_push_finish_kernel, init_blocks, 256, 0, acc, n, inv_out, dang + it,
                damping, last, score, nxt, partials, ticket, dang + it + 1);
    }
  }
}

void pagerank(const gt_graph* g, double damping, int iterations, double* scores, bool on_device) {
  require_init();
  if (!g) fail(GT_EINVAL, "null graph");
  if (!(damping > 0.0 && damping < 1.0)) fail(GT_EINVAL, "damping must be in (0, 1)");
  if (iterations < 1) fail(GT_EINVAL, "iterations must be >= 1");
  if (g->n == 0) fail(GT_EINVAL, "pagerank needs a non-empty graph");
  const int64_t n = g->n, e = g->e;
  const int64_t tiles = std::max<int64_t>(1, ceil_div64(e, gtd::PR_TILE));
  const int fix_blocks = ceil_div(tiles, 256);
  const int init_blocks = static_cast<int>(std::min<int64_t>(ceil_div64(n, 256), 4LL * ctx().sm_count));

  // Scratch (one allocation, carved).
  const size_t bytes = size_t(n) * 8 * 3 + size_t(tiles + 1) * 8 * 12 + size_t(iterations + 2) * 8 +
                       size_t(std::max(fix_blocks, init_blocks)) * 8 + 256;
  char* p = static_cast<char*>(ws_get(WS_TMP1, bytes));
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  double* inv_out = reinterpret_cast<double*>(carve(size_t(n) * 8));
  double* contrib[2] = {reinterpret_cast<double*>(carve(size_t(n) * 8)),
                        reinterpret_cast<double*>(carve(size_t(n) * 8))};
  int64_t* tile_row = reinterpret_cast<int64_t*>(carve(size_t(tiles + 1) * 8));
  double* head = reinterpret_cast<double*>(carve(size_t(tiles) * 8));
  double* tail = reinterpret_cast<double*>(carve(size_t(tiles) * 8));
  int64_t* tail_row = reinterpret_cast<int64_t*>(carve(size_t(tiles) * 8));
  double* dpart = reinterpret_cast<double*>(carve(size_t(tiles) * 8 * (gtd::PR_THREADS / 32)));
  double* dang = reinterpret_cast<double*>(carve(size_t(iterations + 2) * 8));
  double* partials = reinterpret_cast<double*>(carve(size_t(std::max(fix_blocks, init_blocks)) * 8));
  unsigned int* ticket = reinterpret_cast<unsigned int*>(carve(16));
  double* score = on_device ? scores : dalloc_n<double>(n);
  int32_t* pos = ws_n<int32_t>(WS_TMP4, size_t(n));
  int32_t* in_adj_r = ws_n<int32_t>(WS_TMP2, size_t(e) + 1);
  unsigned long long* maxd = reinterpret_cast<unsigned long long*>(ws_n<int64_t>(WS_SMALL, 16) + 13);

  // Push within L2-sized destination bins or pull over the in-CSR. The pull
  // gathers contrib[] at random; it wins while the hottest sources (what half
  // of L2 holds) cover most edges — R-MAT C4: 9.0 ms per iteration vs 12.2 —
  // and loses to the push's forward sweeps when they do not — uniform C5:
  // 38 ms vs 14 + 1 (the push is bound by the L2 fp64 reduction rate,
  // ~130 G/s). GT_PR_PUSH=1 / 0 forces either (A/B, tests).
  int push = -1;
  if (const char* pv = getenv("GT_PR_PUSH")) push = atoi(pv) > 0 ? 1 : 0;
  if (push < 0) {
    push = 0;
    if (e > 0 && size_t(n) * 8 > ctx().l2_bytes / 2) {
      unsigned long long* bk = reinterpret_cast<unsigned long long*>(ws_get(WS_TMP0, 128 * 8));
      GT_CUDA(cudaMemsetAsync(bk, 0, 128 * 8, ctx().stream));
      GT_LAUNCH(gtd::pr_degree_buckets_kernel, init_blocks, 256, 0, g->out_off, n, bk);
      unsigned long long hb[128];
      d2h(hb, bk, sizeof hb);
      sync();
      // edges out of the K = L2/16 highest out-degree sources, bucket by bucket
      // from the top (the bucket that straddles K pro rata)
      double left = double(ctx().l2_bytes) / 16.0, covered = 0.0;
      for (int b = 63; b >= 1 && left > 0; --b) {
        if (!hb[b]) continue;
        const double take = std::min(left, double(hb[b]));
        covered += double(hb[64 + b]) * take / double(hb[b]);
        left -= take;
      }
      push = covered < 0.5 * double(e) ? 1 : 0;
    }
  }
  if (push && e > 0) {
    int rb = 0;
    while ((double(size_t(16) << rb)) <= 0.30 * double(ctx().l2_bytes)) ++rb;
    if (const char* v = getenv("GT_PR_PUSH_BITS")) rb = std::max(4, atoi(v));
    rb = std::min(rb, bits_for(n));
    while (ceil_div64(n, int64_t(1) << rb) > 256) ++rb;
    pagerank_push(g, damping, iterations, rb, score);
    if (!on_device) {
      d2h(scores, score, size_t(n) * 8);
      sync();
      dfree(score);
    }
    sync();
    return;
  }
  // Source relabelling by descending out-degree (see the header comment).
  GT_CUDA(cudaMemsetAsync(maxd, 0, 8, ctx().stream));
  {
    Phase ph("pr.relabel", 8.0 * (n + 1));
    GT_LAUNCH(gtd::pr_max_outdeg_kernel, init_blocks, 256, 0, g->out_off, n, maxd);
  }
  int64_t max_deg = 0;
  d2h(&max_deg, maxd, 8);
  sync();
  {
    const int kb = bits_for(n);
    SortPlan plan = make_plan(0, kb + bits_for(max_deg + 1));
    SortHist h = sort_hist_begin(0);
    uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(n));
    uint64_t* kb_ = ws_n<uint64_t>(WS_KEYS_B, size_t(n));
    {
      Phase ph("pr.relabel", 8.0 * (n + 1) + 8.0 * n);
      GT_LAUNCH(gtd::pr_relabel_keys_kernel, init_blocks, 256, 0, g->out_off, n, max_deg, kb, plan,
                h.hist, ka);
    }
    uint64_t* sorted = radix_sort(ka, kb_, n, plan, h, "pr.relabel");
    Phase ph("pr.relabel", 12.0 * n + 12.0 * e);
    GT_LAUNCH(gtd::pr_pos_kernel, ceil_div(n, 256), 256, 0, sorted, n, (uint64_t(1) << kb) - 1,
              pos);
    if (e > 0)
      GT_LAUNCH(gtd::pr_remap_kernel, static_cast<int>(std::min<int64_t>(ceil_div64(e, 1024),
                                                                         8LL * ctx().sm_count)),
                256, 0, g->in_adj, e, pos, in_adj_r);
  }

  GT_CUDA(cudaMemsetAsync(ticket, 0, 16, ctx().stream));
  {
    Phase ph("pr.setup", 8.0 * (n + 1) + 20.0 * n + 8.0 * (tiles + 1));
    GT_LAUNCH(gtd::pr_init_kernel, init_blocks, 256, 0, g->out_off, n, pos, inv_out, contrib[0],
              partials, ticket, dang);
    GT_LAUNCH(gtd::pr_tile_rows_kernel, ceil_div(tiles + 1, 256), 256, 0, g->in_off, n, tiles,
              tile_row);
  }
  // L2 residency for the hot sources: after the relabelling the first
  // positions of the contrib vector are the high out-degree sources; when the
  // vector is larger than what L2 keeps on its own, the tail gathers carry an
  // L2 cache policy: the hot head evict_last, the rest evict_first.
  const size_t contrib_bytes = size_t(n) * 8;
  uint32_t hot_bytes = 0, total_bytes = 0;
  // GT_PR_L2: "policy" (default) or "none". (A persisting access-policy
  // window was dropped: its set-up and release act on the whole device and
  // synchronise it, stalling the other lane and resetting its L2 set-aside.)
  static const int l2_mode = [] {
    const char* v = getenv("GT_PR_L2");
    return (v && !strcmp(v, "none")) ? 2 : 0;
  }();
  if (contrib_bytes > ctx().l2_bytes / 2 && l2_mode == 0 && contrib_bytes < (size_t(1) << 32)) {
    int max_win = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, ctx().device);
    int persist_max = 0;
    cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, ctx().device);
    hot_bytes = uint32_t(std::min<size_t>({contrib_bytes, size_t(max_win), size_t(persist_max)}));
    if (const char* v = getenv("GT_PR_HOT_MB"))  // sweep knob: size of the evict_last head
      hot_bytes = uint32_t(std::min<size_t>(contrib_bytes, size_t(std::max(1, atoi(v))) << 20));
    if (getenv("GT_PR_DEBUG"))
      fprintf(stderr, "[gt pr] contrib %zu B, evict_last head %u B (window max %d, persist max %d)\n",
              contrib_bytes, hot_bytes, max_win, persist_max);
    total_bytes = uint32_t(contrib_bytes);
  }
  // ---- cache-blocked pull when contrib exceeds L2 (see the kernels) -------
  // segment = 2^sb relabelled sources, 8 * 2^sb bytes <= ~55% of L2
  int sb = 0;
  while ((double(size_t(16) << sb)) <= 0.55 * double(ctx().l2_bytes)) ++sb;
  if (const char* v = getenv("GT_PR_SEGBITS")) sb = std::max(4, atoi(v));  // tests
  const int64_t nseg = ceil_div64(n, int64_t(1) << sb);
  // Opt-in (GT_PR_BLOCK=1): measured on B200 at C4 7.8 ms of
  // SpMV + 2.2 ms of finalize per iteration against 9.0 ms single-pass (the
  // hub relabelling already keeps ~75% of the gathers in L2), and at C5
  // 45.7 ms against 39.5 (rows average two in-edges per segment: the DCSR
  // metadata and partial-sum traffic outweigh the DRAM gathers saved).
  const char* bv = getenv("GT_PR_BLOCK");
  const bool block_on = bv && !strcmp(bv, "1");
  if (nseg >= 2 && nseg <= 256 && block_on && e > 0) {
    pagerank_blocked(g, damping, iterations, sb, nseg, tiles, tile_row, in_adj_r, pos, inv_out,
                     contrib, dang, partials, ticket, score, init_blocks);
    if (!on_device) {
      d2h(scores, score, size_t(n) * 8);
      sync();
      dfree(score);
    }
    sync();
    return;
  }
  static const int pf_dist = [] {  // GT_PR_PF: index prefetch distance in tiles (0 = off)
    const char* env = getenv("GT_PR_PF");  // measured at C4: 0 / 444 / 888 tiles within 0.5 %
    return env ? atoi(env) : 0;
  }();
  for (int it = 0; it < iterations; ++it) {
    const int last = it == iterations - 1;
    double* cur = contrib[it & 1];
    double* nxt = contrib[(it + 1) & 1];
    {
      Phase ph("pr.spmv", 12.0 * e + 8.0 * (n + 1) + 20.0 * n);
      GT_LAUNCH(gtd::pr_spmv_kernel, static_cast<int>(tiles), gtd::PR_THREADS, 0, g->in_off,
                in_adj_r, n, e, n, tile_row, cur, inv_out, pos, dang + it, damping, score, nxt,
                head, tail, tail_row, dpart, last, hot_bytes, total_bytes, pf_dist);
    }
    {
      Phase ph("pr.fixup", 40.0 * tiles);
      GT_LAUNCH(gtd::pr_fixup_kernel, fix_blocks, 256, 0, g->in_off, n, n, tiles, inv_out, pos,
                dang + it, damping, head, tail, tail_row, dpart, score, nxt, last, partials,
                ticket, dang + it + 1);
    }
  }
  if (!on_device) {
    d2h(scores, score, size_t(n) * 8);
    sync();
    dfree(score);
  }
  sync();
}

}  // namespace gt

using namespace gt;

extern "C" int gt_pagerank(const gt_graph* g, double damping, int iterations, double* scores,
                           int scores_is_device) {
  GT_API_BEGIN
  if (!scores) fail(GT_EINVAL, "scores must not be NULL");
  pagerank(g, damping, iterations, scores, scores_is_device != 0);
  GT_API_END
}

// ============================================================================
// Primitives of the multi-GPU PageRank (paper_1503_07881_b200/distributed.py):
// each rank owns a dst-row range of the in-CSR; the contrib vector is
// replicated (all-gathered every iteration) and the dangling mass all-reduced.
// ============================================================================
namespace gt {

static void pr_step_impl(const int64_t* in_off, const int32_t* in_adj, int64_t rows,
                         int64_t e, int64_t n_total, const double* contrib_full,
                         const double* inv_rows, const double* dangling_prev, double damping,
                         int last, double* score_rows, double* contrib_rows, double* dangling_out) {
  const int64_t tiles = std::max<int64_t>(1, ceil_div64(e, gtd::PR_TILE));
  const int fix_blocks = ceil_div(tiles, 256);
  const size_t bytes = size_t(tiles + 1) * 8 * 12 + size_t(fix_blocks) * 8 + 256;
  char* p = static_cast<char*>(ws_get(WS_TMP1, bytes));
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  int64_t* tile_row = reinterpret_cast<int64_t*>(carve(size_t(tiles + 1) * 8));
  double* head = reinterpret_cast<double*>(carve(size_t(tiles) * 8));
  double* tail = reinterpret_cast<double*>(carve(size_t(tiles) * 8));
  int64_t* tail_row = reinterpret_cast<int64_t*>(carve(size_t(tiles) * 8));
  double* dpart = reinterpret_cast<double*>(carve(size_t(tiles) * 8 * (gtd::PR_THREADS / 32)));
  double* partials = reinterpret_cast<double*>(carve(size_t(fix_blocks) * 8));
  unsigned int* ticket = reinterpret_cast<unsigned int*>(carve(16));
  GT_CUDA(cudaMemsetAsync(ticket, 0, 16, ctx().stream));
  Phase ph("pr.step", 12.0 * e + 8.0 * (rows + 1) + 24.0 * rows);
  GT_LAUNCH(gtd::pr_tile_rows_kernel, ceil_div(tiles + 1, 256), 256, 0, in_off, rows, tiles,
            tile_row);
  GT_LAUNCH(gtd::pr_spmv_kernel, static_cast<int>(tiles), gtd::PR_THREADS, 0, in_off, in_adj, rows,
            e, n_total, tile_row, contrib_full, inv_rows, (const int32_t*)nullptr, dangling_prev,
            damping, score_rows, contrib_rows, head, tail, tail_row, dpart, last, 0u, 0u, 0);
  GT_LAUNCH(gtd::pr_fixup_kernel, fix_blocks, 256, 0, in_off, rows, n_total, tiles, inv_rows,
            (const int32_t*)nullptr, dangling_prev, damping, head, tail, tail_row, dpart,
            score_rows, contrib_rows, last, partials, ticket, dangling_out);
}

}  // namespace gt

extern "C" {

int gt_remap_padded(const int32_t* d_in, int64_t e, const int64_t* h_bounds, int world,
                    int64_t m, int32_t* d_out) {
  GT_API_BEGIN
  require_init();
  if (world < 1 || world > 64 || e < 0 || !h_bounds) fail(GT_EINVAL, "bad arguments");
  if (int64_t(world) * m >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "padded layout >= 2^31");
  if (e == 0) return GT_OK;
  int64_t* d_b = ws_n<int64_t>(WS_SMALL, 80);
  h2d(d_b, h_bounds, size_t(world + 1) * 8);
  GT_LAUNCH(gtd::pr_remap_padded_kernel,
            static_cast<int>(std::min<int64_t>(ceil_div64(e, 1024), 8LL * ctx().sm_count)), 256, 0,
            d_in, e, d_b, world, m, d_out);
  sync();
  GT_API_END
}

int gt_inv_degree(const int64_t* d_off, int64_t rows, double* d_inv) {
  GT_API_BEGIN
  require_init();
  if (rows < 0) fail(GT_EINVAL, "rows must be >= 0");
  if (rows > 0) GT_LAUNCH(gtd::pr_inv_degree_kernel, ceil_div(rows, 256), 256, 0, d_off, rows, d_inv);
  sync();
  GT_API_END
}

int gt_pagerank_init(const double* d_inv, int64_t n, double* d_contrib, double* d_dangling) {
  GT_API_BEGIN
  require_init();
  if (n < 1) fail(GT_EINVAL, "pagerank needs a non-empty graph");
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div64(n, 256), 4LL * ctx().sm_count));
  char* p = static_cast<char*>(ws_get(WS_TMP1, size_t(blocks) * 8 + 64));
  double* partials = reinterpret_cast<double*>(p);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(p + size_t(blocks) * 8 + 16);
  GT_CUDA(cudaMemsetAsync(ticket, 0, 16, ctx().stream));
  GT_LAUNCH(gtd::pr_init_from_inv_kernel, blocks, 256, 0, d_inv, n, d_contrib, partials, ticket,
            d_dangling);
  sync();
  GT_API_END
}

int gt_pagerank_step(const int64_t* d_in_off, const int32_t* d_in_adj, int64_t rows,
                     int64_t e_local, int64_t n_total, const double* d_contrib,
                     const double* d_inv_rows, const double* d_dangling_prev, double damping,
                     int last, double* d_score_rows, double* d_contrib_rows,
                     double* d_dangling_out) {
  GT_API_BEGIN
  require_init();
  if (!(damping > 0.0 && damping < 1.0)) fail(GT_EINVAL, "damping must be in (0, 1)");
  if (rows < 0 || e_local < 0 || n_total < 1) fail(GT_EINVAL, "bad sizes");
  if (rows == 0) {
    GT_CUDA(cudaMemsetAsync(d_dangling_out, 0, 8, ctx().stream));
  } else {
    pr_step_impl(d_in_off, d_in_adj, rows, e_local, n_total, d_contrib, d_inv_rows,
                 d_dangling_prev, damping, last, d_score_rows, d_contrib_rows, d_dangling_out);
  }
  sync();
  GT_API_END
}

}  // extern "C"
