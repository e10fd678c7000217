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
// HBM traffic per iteration (algorithmic): 4E (in_adj) + 8E (contrib gathers)
// + 8(N+1) (in_off) + 8N (inv_out) + 8N (contrib write) [+ 8N score, last
// iteration only].
#include "graph.cuh"
#include "radix_sort.cuh"

#include <algorithm>

namespace gtd {

constexpr int PR_THREADS = 256;
constexpr int PR_TILE = 2048;

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
    contrib[v] = s0 * inv;
    if (deg == 0) dang += s0;
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling0);
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

template <int G>
__device__ __forceinline__ void pr_rows(const double* vals, const int64_t* __restrict__ in_off,
                                        int64_t e0, int64_t e1, int64_t ra, int64_t rb,
                                        bool has_head, int64_t c, double base, double damping,
                                        const double* __restrict__ inv_out,
                                        double* __restrict__ score, double* __restrict__ contrib_next,
                                        double* __restrict__ head, double* __restrict__ tail,
                                        int64_t* __restrict__ tail_row, bool last_iter,
                                        double& dang) {
  constexpr int GPW = 32 / G;  // groups per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int64_t nseg = (rb - ra) + (has_head ? 1 : 0);
  const int64_t first_row = has_head ? ra - 1 : ra;
  for (int64_t s0 = int64_t(warp) * GPW; s0 < nseg; s0 += int64_t(PR_THREADS / 32) * GPW) {
    const int64_t s = s0 + grp;
    const bool active = s < nseg;
    const int64_t row = first_row + s;
    int64_t a = 0, b = 0;
    if (active) {
      a = max(in_off[row], e0) - e0;
      b = min(in_off[row + 1], e1) - e0;
    }
    double sum = 0.0;
    for (int64_t j = a + gl; j < b; j += G) sum += vals[j];
    __syncwarp();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (active && gl == 0) {
      if (has_head && s == 0) {
        head[c] = sum;
      } else if (in_off[row + 1] > e1) {
        tail[c] = sum;
        tail_row[c] = row;
      } else {
        const double sc = base + damping * sum;
        const double inv = inv_out[row];
        if (!last_iter) contrib_next[row] = sc * inv;
        else score[row] = sc;
        if (inv == 0.0) dang += sc;
      }
    }
  }
}

__global__ void __launch_bounds__(PR_THREADS) pr_spmv_kernel(
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_adj, int64_t n, int64_t e,
    const int64_t* __restrict__ tile_row, const double* __restrict__ contrib,
    const double* __restrict__ inv_out, const double* __restrict__ dangling_prev, double damping,
    double* __restrict__ score, double* __restrict__ contrib_next, double* __restrict__ head,
    double* __restrict__ tail, int64_t* __restrict__ tail_row, double* __restrict__ dpart,
    int last_iter) {
  __shared__ double vals[PR_TILE];
  __shared__ double s_red[8];
  const int64_t c = blockIdx.x;
  const int64_t e0 = c * PR_TILE;
  const int64_t e1 = min(e, e0 + PR_TILE);
  const int ne = e1 > e0 ? int(e1 - e0) : 0;
  const int64_t ra = tile_row[c], rb = tile_row[c + 1];
  const double base = (1.0 - damping) / double(n) + damping * (*dangling_prev / double(n));
  if (threadIdx.x == 0) tail_row[c] = -1;

  // Gather phase: PR_TILE/256 independent loads per thread in flight.
  constexpr int PER = PR_TILE / PR_THREADS;
  int32_t idx[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = i * PR_THREADS + threadIdx.x;
    idx[i] = j < ne ? __ldcs(in_adj + e0 + j) : 0;
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = i * PR_THREADS + threadIdx.x;
    if (j < ne) vals[j] = __ldg(contrib + idx[i]);
  }
  __syncthreads();

  const bool has_head = ne > 0 && (ra == n || in_off[ra] > e0);
  const int64_t nseg = (rb - ra) + (has_head ? 1 : 0);
  const int64_t avg = nseg > 0 ? int64_t(ne) / nseg : 32;
  const bool last = last_iter != 0;
  double dang = 0.0;
  if (avg >= 24)
    pr_rows<32>(vals, in_off, e0, e1, ra, rb, has_head, c, base, damping, inv_out, score,
                contrib_next, head, tail, tail_row, last, dang);
  else if (avg >= 12)
    pr_rows<16>(vals, in_off, e0, e1, ra, rb, has_head, c, base, damping, inv_out, score,
                contrib_next, head, tail, tail_row, last, dang);
  else if (avg >= 6)
    pr_rows<8>(vals, in_off, e0, e1, ra, rb, has_head, c, base, damping, inv_out, score,
               contrib_next, head, tail, tail_row, last, dang);
  else if (avg >= 3)
    pr_rows<4>(vals, in_off, e0, e1, ra, rb, has_head, c, base, damping, inv_out, score,
               contrib_next, head, tail, tail_row, last, dang);
  else
    pr_rows<2>(vals, in_off, e0, e1, ra, rb, has_head, c, base, damping, inv_out, score,
               contrib_next, head, tail, tail_row, last, dang);
  dang = block_sum_256(dang, s_red);
  if (threadIdx.x == 0) dpart[c] = dang;
}

__global__ void __launch_bounds__(256) pr_fixup_kernel(
    const int64_t* __restrict__ in_off, int64_t n, int64_t tiles,
    const double* __restrict__ inv_out, const double* __restrict__ dangling_prev, double damping,
    const double* __restrict__ head, const double* __restrict__ tail,
    const int64_t* __restrict__ tail_row, const double* __restrict__ dpart,
    double* __restrict__ score, double* __restrict__ contrib_next, int last_iter,
    double* __restrict__ partials, unsigned int* __restrict__ ticket,
    double* __restrict__ dangling_next) {
  __shared__ double s_red[8];
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const double base = (1.0 - damping) / double(n) + damping * (*dangling_prev / double(n));
  double dang = 0.0;
  if (c < tiles) {
    dang = dpart[c];
    const int64_t v = tail_row[c];
    if (v >= 0) {
      const int64_t c_last = (in_off[v + 1] - 1) / PR_TILE;
      double sum = tail[c];
      for (int64_t c2 = c + 1; c2 <= c_last; ++c2) sum += head[c2];
      const double sc = base + damping * sum;
      const double inv = inv_out[v];
      if (last_iter) score[v] = sc;
      else contrib_next[v] = sc * inv;
      if (inv == 0.0) dang += sc;
    }
  }
  dang = block_sum_256(dang, s_red);
  grid_reduce_last(dang, partials, ticket, dangling_next);
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
  const size_t bytes = size_t(n) * 8 * 3 + size_t(tiles + 1) * 8 * 5 + size_t(iterations + 2) * 8 +
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
  double* dpart = reinterpret_cast<double*>(carve(size_t(tiles) * 8));
  double* dang = reinterpret_cast<double*>(carve(size_t(iterations + 2) * 8));
  double* partials = reinterpret_cast<double*>(carve(size_t(std::max(fix_blocks, init_blocks)) * 8));
  unsigned int* ticket = reinterpret_cast<unsigned int*>(carve(16));
  double* score = on_device ? scores : dalloc_n<double>(n);

  GT_CUDA(cudaMemsetAsync(ticket, 0, 16, ctx().stream));
  {
    Phase ph("pr.setup", 8.0 * (n + 1) + 16.0 * n + 8.0 * (tiles + 1));
    GT_LAUNCH(gtd::pr_init_kernel, init_blocks, 256, 0, g->out_off, n, inv_out, contrib[0],
              partials, ticket, dang);
    GT_LAUNCH(gtd::pr_tile_rows_kernel, ceil_div(tiles + 1, 256), 256, 0, g->in_off, n, tiles,
              tile_row);
  }
  for (int it = 0; it < iterations; ++it) {
    const int last = it == iterations - 1;
    double* cur = contrib[it & 1];
    double* nxt = contrib[(it + 1) & 1];
    {
      Phase ph("pr.spmv", 12.0 * e + 8.0 * (n + 1) + 16.0 * n + (last ? 0.0 : 0.0));
      GT_LAUNCH(gtd::pr_spmv_kernel, static_cast<int>(tiles), gtd::PR_THREADS, 0, g->in_off,
                g->in_adj, n, e, tile_row, cur, inv_out, dang + it, damping, score, nxt, head,
                tail, tail_row, dpart, last);
    }
    {
      Phase ph("pr.fixup", 40.0 * tiles);
      GT_LAUNCH(gtd::pr_fixup_kernel, fix_blocks, 256, 0, g->in_off, n, tiles, inv_out, dang + it,
                damping, head, tail, tail_row, dpart, score, nxt, last, partials, ticket,
                dang + it + 1);
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
