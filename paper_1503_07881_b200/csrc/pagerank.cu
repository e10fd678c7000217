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

namespace gtd {

// Gathers: the head of contrib (the PR_HOT highest out-degree sources after
// the relabelling) through the L1-allocating non-coherent path, the tail with
// L1::no_allocate. Measured (scripts/sweep_const.sh): spmv C2 7.75 -> 7.48 ms,
// C4 203 -> 172 ms against __ldg for all; the split point itself did not
// matter (0 .. 2^20 within noise), while a plain no_allocate load for every
// gather compiled to a slower schedule (C2 10.7 ms).
constexpr int PR_HOT = 1 << 15;
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

constexpr int PR_THREADS = 256;
constexpr int PR_TILE = 2048;
constexpr int PR_MIN_BLOCKS = 6;  // resident CTAs per SM the register budget is sized for

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
    int last_iter, uint32_t hot_bytes, uint32_t total_bytes) {
  __shared__ double vals[PR_TILE];
  __shared__ PrRows sr;
  const double base =
      (1.0 - damping) / double(n_total) + damping * (*dangling_prev / double(n_total));
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

namespace gt {

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
    total_bytes = uint32_t(contrib_bytes);
  }
  for (int it = 0; it < iterations; ++it) {
    const int last = it == iterations - 1;
    double* cur = contrib[it & 1];
    double* nxt = contrib[(it + 1) & 1];
    {
      Phase ph("pr.spmv", 12.0 * e + 8.0 * (n + 1) + 20.0 * n);
      GT_LAUNCH(gtd::pr_spmv_kernel, static_cast<int>(tiles), gtd::PR_THREADS, 0, g->in_off,
                in_adj_r, n, e, n, tile_row, cur, inv_out, pos, dang + it, damping, score, nxt,
                head, tail, tail_row, dpart, last, hot_bytes, total_bytes);
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
            damping, score_rows, contrib_rows, head, tail, tail_row, dpart, last, 0u, 0u);
  GT_LAUNCH(gtd::pr_fixup_kernel, fix_blocks, 256, 0, in_off, rows, n_total, tiles, inv_rows,
            (const int32_t*)nullptr, dangling_prev, damping, head, tail, tail_row, dpart,
            score_rows, contrib_rows, last, partials, ticket, dangling_out);
}

}  // namespace gt

extern "C" {

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
