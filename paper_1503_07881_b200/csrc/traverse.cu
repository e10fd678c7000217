// traverse.cu — CSR consumers beyond the path on the
// device CSR a gt_graph already holds:
//
//   gt_bfs                 hop distances from one source along out-edges
//                          (algorithms.sssp, algorithms.py:125-141)
//   gt_connected_components weakly connected components, labels dense in the
//                          order of each component's smallest id
//                          (algorithms.connected_components, :232-248)
//   gt_kcore               maximal subgraph whose nodes keep >= k distinct
//                          undirected neighbours, as a new graph
//                          (algorithms.k_core, :206-229; graphs.py:169-183)
//
// BFS is level-synchronous and direction-optimising: a small frontier expands
// top-down (warp per frontier node, CAS-claimed children appended with one
// warp-aggregated atomic), a large one bottom-up over the in-CSR (every
// unvisited node looks for a parent on the current level and stops at the
// first). Distances are unique, so the result does not depend on scheduling.
// Components: lock-free union-find that always hooks the larger root under
// the smaller (parent[x] <= x), so every root is its component's minimum
// dense index = minimum id; labels = rank of the root among the roots.
// k-core: the undirected degrees of triangles.cu, then frontier peeling with
// atomic decrements (a node dies exactly once, when its degree crosses k-1);
// the surviving directed edges are rebuilt into a CSR by gt_build_csr's
// pipeline (the induced subgraph keeps every original edge between survivors).
#include "graph.cuh"
#include "scan.cuh"

#include <algorithm>
#include <vector>

namespace gt {
gt_graph* build_csr(const int64_t* src, const int64_t* dst, int64_t rows, const int64_t* extra,
                    int64_t n_extra, bool on_device);
}

namespace gtd {

constexpr unsigned FULL = 0xffffffffu;

// Appends v of every flagged lane to queue[*count ...] with one atomic per warp
// (all 32 lanes must call it).
__device__ __forceinline__ void warp_append(bool flag, int32_t v, int32_t* __restrict__ queue,
                                            unsigned int* __restrict__ count) {
  const unsigned b = __ballot_sync(FULL, flag);
  if (!b) return;
  unsigned base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(count, unsigned(__popc(b)));
  base = __shfl_sync(FULL, base, 0);
  if (flag) queue[base + __popc(b & lanemask_lt())] = v;
}

// ---- BFS ---------------------------------------------------------------------

__global__ void __launch_bounds__(256) bfs_init_kernel(int32_t* __restrict__ dist, int64_t n,
                                                       int64_t src, int32_t* __restrict__ frontier) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dist[i] = i == src ? 0 : -1;
  if (i == 0) frontier[0] = int32_t(src);
}

// Warp per frontier node: children not yet visited are claimed with a CAS
// (exactly one claimer appends each).
__global__ void __launch_bounds__(256) bfs_top_down_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
    const int32_t* __restrict__ frontier, int64_t nf, int32_t* __restrict__ dist, int32_t next_level,
    int32_t* __restrict__ next, unsigned int* __restrict__ next_count) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t f = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < nf; f += nwarps) {
    const int32_t u = frontier[f];
    const int64_t a = off[u], b = off[u + 1];
    for (int64_t k0 = a; k0 < b; k0 += 32) {
      const int64_t k = k0 + lane;
      bool claimed = false;
      int32_t v = 0;
      if (k < b) {
        v = adj[k];
        if (__ldcg(dist + v) < 0) claimed = atomicCAS(dist + v, -1, next_level) == -1;
      }
      warp_append(claimed, v, next, next_count);
    }
  }
}

// Thread per node: an unvisited node whose in-neighbour sits on `level` joins
// level + 1 (first parent found ends the scan).
__global__ void __launch_bounds__(256) bfs_bottom_up_kernel(
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_adj, int64_t n,
    int32_t* __restrict__ dist, int32_t level, int32_t* __restrict__ next,
    unsigned int* __restrict__ next_count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    bool found = false;
    if (v < n && dist[v] < 0) {
      const int64_t b = in_off[v + 1];
      for (int64_t k = in_off[v]; k < b; ++k) {
        if (__ldcg(dist + in_adj[k]) == level) {
          found = true;
          break;
        }
      }
      if (found) dist[v] = level + 1;
    }
    warp_append(found, int32_t(v), next, next_count);
  }
}

// ---- weakly connected components ---------------------------------------------

__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t x) {
  // path halving; parent[x] <= x always, so every write moves x closer to the root
  int32_t p = __ldcg(parent + x);
  while (p != x) {
    const int32_t gp = __ldcg(parent + p);
    if (gp != p) parent[x] = gp;
    x = p;
    p = gp;
  }
  return x;
}

__global__ void __launch_bounds__(256) uf_init_kernel(int32_t* __restrict__ parent, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) parent[i] = int32_t(i);
}

// union(a, b): the larger root hooked under the smaller with a CAS (retried
// from the new parent when it loses).
__device__ __forceinline__ void uf_union(int32_t* parent, int32_t a, int32_t b) {
  int32_t x = uf_find(parent, a), y = uf_find(parent, b);
  while (x != y) {
    if (x < y) {
      const int32_t t = x;
      x = y;
      y = t;
    }
    const int32_t old = atomicCAS(parent + x, x, y);  // hook root x (> y) under y
    if (old == x) return;
    x = uf_find(parent, old);
    y = uf_find(parent, y);
  }
}

// Afforest, round r: every node links with its r-th out-neighbour (a sparse
// sample of the edges that already joins nearly all of a giant component).
__global__ void __launch_bounds__(256) uf_sample_kernel(const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ adj, int64_t n,
                                                        int r, int32_t* parent) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += stride) {
    const int64_t a = off[u];
    if (a + r < off[u + 1]) uf_union(parent, int32_t(u), adj[a + r]);
  }
}

// Afforest, final pass: warp per node u outside the dominant component c —
// every remaining out-edge (from position `skip`) and every in-edge of u is
// linked. Edges with both ends in c are already joined and never touched.
__global__ void __launch_bounds__(256) uf_finish_kernel(
    const int64_t* __restrict__ out_off, const int32_t* __restrict__ out_adj,
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_adj, int64_t n, int skip,
    int32_t c, int32_t* parent) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t u = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
    if (uf_find(parent, int32_t(u)) == c) continue;  // warp-uniform
    const int64_t oa = out_off[u] + skip, ob = out_off[u + 1];
    for (int64_t k = oa + lane; k < ob; k += 32) uf_union(parent, int32_t(u), out_adj[k]);
    const int64_t ia = in_off[u], ib = in_off[u + 1];
    for (int64_t k = ia + lane; k < ib; k += 32) uf_union(parent, int32_t(u), in_adj[k]);
  }
}

// Root of sample i (i-th of `ns` nodes spread over [0, n)), for the host to
// pick the dominant component.
__global__ void uf_sample_roots_kernel(int32_t* parent, int64_t n, int ns,
                                       int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ns) out[i] = uf_find(parent, int32_t((uint64_t(i) * 0x9E3779B97F4A7C15ull >> 11) % uint64_t(n)));
}

// Warp per row u, lanes over out(u): union(u, v), the larger root hooked under
// the smaller with a CAS (retried from the new parent when it loses).
__global__ void __launch_bounds__(256) uf_hook_kernel(const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ adj, int64_t n,
                                                      int32_t* parent) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t u = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
    const int64_t a = off[u], b = off[u + 1];
    for (int64_t k = a + lane; k < b; k += 32) {
      int32_t x = uf_find(parent, int32_t(u)), y = uf_find(parent, adj[k]);
      while (x != y) {
        if (x < y) {
          const int32_t t = x;
          x = y;
          y = t;
        }
        const int32_t old = atomicCAS(parent + x, x, y);  // hook root x (> y) under y
        if (old == x) break;
        x = uf_find(parent, old);
        y = uf_find(parent, y);
      }
    }
  }
}

// parent[i] <- root(i); flag[i] = 1 for roots (as int64 for the scan).
__global__ void __launch_bounds__(256) uf_flatten_kernel(int32_t* parent, int64_t n,
                                                         int64_t* __restrict__ flag) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t x = int32_t(i), p = __ldcg(parent + x);
  while (p != x) {
    x = p;
    p = __ldcg(parent + x);
  }
  flag[i] = x == int32_t(i) ? 1 : 0;
  parent[i] = x;
}

__global__ void __launch_bounds__(256) uf_label_kernel(const int32_t* __restrict__ root, int64_t n,
                                                       const int64_t* __restrict__ root_rank,
                                                       int64_t* __restrict__ labels) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) labels[i] = root_rank[root[i]];
}

// ---- k-core ------------------------------------------------------------------

__global__ void __launch_bounds__(256) kcore_seed_kernel(const int32_t* __restrict__ deg, int64_t n,
                                                         int32_t k, uint8_t* __restrict__ alive,
                                                         int32_t* __restrict__ frontier,
                                                         unsigned int* __restrict__ count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool dead = i < n && deg[i] < k;
    if (i < n) alive[i] = dead ? 0 : 1;
    warp_append(dead, int32_t(i), frontier, count);
  }
}

// Warp per removed node: every distinct undirected neighbour still alive loses
// one degree; the one whose degree crosses from k to k-1 dies (exactly once)
// and joins the next frontier.
__global__ void __launch_bounds__(256) kcore_peel_kernel(
    const int64_t* __restrict__ cat, const int64_t* __restrict__ out_off,
    const int32_t* __restrict__ out_adj, const int64_t* __restrict__ in_off,
    const int32_t* __restrict__ in_adj, const uint32_t* __restrict__ keep_bits,
    const int32_t* __restrict__ frontier, int64_t nf, int32_t k, int32_t* deg, uint8_t* alive,
    int32_t* __restrict__ next, unsigned int* __restrict__ next_count) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t f = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < nf; f += nwarps) {
    const int32_t u = frontier[f];
    const int64_t c = cat[u], total = cat[u + 1] - c;
    const int64_t oo = out_off[u], no = out_off[u + 1] - oo, io = in_off[u];
    for (int64_t s0 = 0; s0 < total; s0 += 32) {
      const int64_t s = s0 + lane;
      bool died = false;
      int32_t m = 0;
      if (s < total && ((__ldg(keep_bits + ((c + s) >> 5)) >> ((c + s) & 31)) & 1u)) {
        m = s < no ? out_adj[oo + s] : in_adj[io + (s - no)];
        if (*reinterpret_cast<volatile uint8_t*>(alive + m)) {
          const int32_t old = atomicSub(deg + m, 1);
          if (old == k) {
            alive[m] = 0;
            died = true;
          }
        }
      }
      warp_append(died, m, next, next_count);
    }
  }
}

// Edges (u, v) with both ends alive, as dense indices, appended in any order
// (the CSR build sorts; dense order = id order, so the built graph only needs
// its node list mapped back through ids). Blocks walk chunks of KC_ROWS rows twice: count the chunk's
// kept edges (warp per row), reserve them with ONE global atomic per chunk,
// then write them through a shared-memory cursor. (A global atomic per warp
// step serialised ~45 M atomics on one address: 101 ms at C4.)
constexpr int KC_ROWS = 256;

__global__ void __launch_bounds__(256) kcore_edges_kernel(
    const int64_t* __restrict__ ids, const int64_t* __restrict__ off,
    const int32_t* __restrict__ adj, int64_t n, const uint8_t* __restrict__ alive,
    int64_t* __restrict__ src, int64_t* __restrict__ dst, unsigned long long* __restrict__ count) {
  __shared__ unsigned long long s_cnt, s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t r0 = int64_t(blockIdx.x) * KC_ROWS; r0 < n; r0 += int64_t(gridDim.x) * KC_ROWS) {
    const int64_t r1 = min(n, r0 + KC_ROWS);
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    unsigned long long mine = 0;
    for (int64_t u = r0 + warp; u < r1; u += 8) {
      if (!alive[u]) continue;  // warp-uniform
      for (int64_t k = off[u] + lane, b = off[u + 1]; k < b; k += 32) mine += alive[adj[k]] ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(FULL, mine, o);
    if (lane == 0 && mine) atomicAdd(&s_cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0) {
      s_base = s_cnt ? atomicAdd(count, s_cnt) : 0ull;
      s_cnt = 0;
    }
    __syncthreads();
    for (int64_t u = r0 + warp; u < r1; u += 8) {
      if (!alive[u]) continue;
      const int64_t a = off[u], b = off[u + 1];
      for (int64_t k0 = a; k0 < b; k0 += 32) {
        const int64_t k = k0 + lane;
        int32_t v = 0;
        const bool keep = k < b && alive[v = adj[k]];
        const unsigned bal = __ballot_sync(FULL, keep);
        if (!bal) continue;
        unsigned long long pos = 0;
        if (lane == 0) pos = atomicAdd(&s_cnt, (unsigned long long)__popc(bal));
        pos = s_base + __shfl_sync(FULL, pos, 0);
        if (keep) {
          const unsigned long long p = pos + __popc(bal & lanemask_lt());
          src[p] = u;  // dense indices: the rebuild maps its node list back to ids
          dst[p] = v;
        }
      }
    }
    __syncthreads();
  }
}

// node list of the rebuilt core: dense indices of the old graph -> ids
__global__ void __launch_bounds__(256) kcore_ids_kernel(const int64_t* __restrict__ old_ids,
                                                        int64_t n, int64_t* __restrict__ ids) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = old_ids[ids[i]];
}

}  // namespace gtd

namespace gt {

static int grid_for(int64_t n, int per_thread) {  // blocks of 256 threads, capped
  return static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div64(n, 256 * int64_t(per_thread)), int64_t(ctx().sm_count) * 16)));
}

static int warps_grid(int64_t items) {
  return static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div64(items, 8), int64_t(ctx().sm_count) * 16)));
}

// frontier size (share of n) above which a level runs bottom-up
constexpr int64_t BFS_UP_DIV = 2048;

static void bfs(const gt_graph* g, int64_t source, int32_t* out, bool out_device) {
  require_init();
  const int64_t n = g->n;
  if (source < 0 || source >= n) fail(GT_EINVAL, "bfs: source index out of range");
  cudaStream_t s = ctx().stream;
  int32_t* dist = out_device ? out : dalloc_n<int32_t>(size_t(n));
  int32_t* q0 = ws_n<int32_t>(WS_TMP0, size_t(n));
  int32_t* q1 = ws_n<int32_t>(WS_TMP1, size_t(n));
  unsigned int* counter = ws_n<unsigned int>(WS_COUNTERS, 64) + 40;
  {
    Phase ph("bfs", 4.0 * n);
    GT_LAUNCH(gtd::bfs_init_kernel, ceil_div(n, 256), 256, 0, dist, n, source, q0);
  }
  int64_t nf = 1, visited = 1;
  int32_t level = 0;
  // direction switch (Beamer et al.): bottom-up while the frontier is a large
  // share of the graph, top-down otherwise
  while (nf > 0) {
    GT_CUDA(cudaMemsetAsync(counter, 0, 4, s));
    const bool bottom_up = nf > n / BFS_UP_DIV && n - visited > 0;
    {
      Phase ph(bottom_up ? "bfs.bottom_up" : "bfs.top_down", 0.0);
      if (bottom_up)
        GT_LAUNCH(gtd::bfs_bottom_up_kernel, grid_for(n, 8), 256, 0, g->in_off, g->in_adj, n, dist,
                  level, q1, counter);
      else
        GT_LAUNCH(gtd::bfs_top_down_kernel, warps_grid(nf), 256, 0, g->out_off, g->out_adj, q0, nf,
                  dist, level + 1, q1, counter);
    }
    unsigned int h = 0;
    d2h(&h, counter, 4);
    sync();
    nf = h;
    visited += nf;
    std::swap(q0, q1);
    ++level;
  }
  if (!out_device) {
    d2h(out, dist, size_t(n) * 4);
    sync();
    dfree(dist);
  }
}

static int64_t components(const gt_graph* g, int64_t* out, bool out_device) {
  require_init();
  const int64_t n = g->n;
  int32_t* parent = ws_n<int32_t>(WS_TMP0, size_t(n));
  int64_t* rank = ws_n<int64_t>(WS_TMP1, size_t(n) + 1);
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  int64_t* labels = out_device ? out : dalloc_n<int64_t>(size_t(n));
  // Afforest (Sutton et al.): link a two-neighbour sample, find the dominant
  // root from a sample of nodes, then link every other edge only for nodes
  // outside it (out- and in-edges, so no edge with an end outside is missed)
  constexpr int SAMPLE_ROUNDS = 2, SAMPLE_NODES = 1024;
  int32_t* sroots = reinterpret_cast<int32_t*>(small + 8);  // 64 B, then host mode
  int32_t* sbuf = ws_n<int32_t>(WS_TMP2, SAMPLE_NODES);
  {
    Phase ph("cc.union_find", 8.0 * n + 4.0 * g->e + 8.0 * (n + 1));
    GT_LAUNCH(gtd::uf_init_kernel, ceil_div(n, 256), 256, 0, parent, n);
    for (int r = 0; r < SAMPLE_ROUNDS && g->e; ++r)
      GT_LAUNCH(gtd::uf_sample_kernel, grid_for(n, 4), 256, 0, g->out_off, g->out_adj, n, r,
                parent);
  }
  int32_t c = -1;
  if (g->e) {
    GT_LAUNCH(gtd::uf_sample_roots_kernel, ceil_div(SAMPLE_NODES, 256), 256, 0, parent, n,
              SAMPLE_NODES, sbuf);
    std::vector<int32_t> h(SAMPLE_NODES);
    d2h(h.data(), sbuf, h.size() * 4);
    sync();
    std::sort(h.begin(), h.end());
    int best = 0;
    for (int i = 0, j; i < SAMPLE_NODES; i = j) {
      for (j = i; j < SAMPLE_NODES && h[j] == h[i]; ++j) {}
      if (j - i > best) { best = j - i; c = h[i]; }
    }
    Phase ph("cc.union_find", 0.0);
    GT_LAUNCH(gtd::uf_finish_kernel, warps_grid(n), 256, 0, g->out_off, g->out_adj, g->in_off,
              g->in_adj, n, SAMPLE_ROUNDS, c, parent);
  }
  (void)sroots;
  {
    Phase ph("cc.label", 4.0 * n + 8.0 * n * 3);
    GT_LAUNCH(gtd::uf_flatten_kernel, ceil_div(n, 256), 256, 0, parent, n, rank);
    exclusive_scan_i64(rank, n, small + 7);
    GT_LAUNCH(gtd::uf_label_kernel, ceil_div(n, 256), 256, 0, parent, n, rank, labels);
  }
  int64_t n_comp = 0;
  d2h(&n_comp, small + 7, 8);
  if (!out_device) d2h(out, labels, size_t(n) * 8);
  sync();
  if (!out_device) dfree(labels);
  return n_comp;
}

static gt_graph* kcore(const gt_graph* g, int32_t k) {
  require_init();
  if (k < 1) fail(GT_EINVAL, "k must be >= 1");
  const int64_t n = g->n;
  if (n == 0) return build_csr(nullptr, nullptr, 0, nullptr, 0, true);
  cudaStream_t s = ctx().stream;
  int64_t* cat = dalloc_n<int64_t>(size_t(n) + 1);
  int32_t* deg = dalloc_n<int32_t>(size_t(n));
  uint8_t* alive = dalloc_n<uint8_t>(size_t(n));
  int32_t* q0 = dalloc_n<int32_t>(size_t(n));
  int32_t* q1 = dalloc_n<int32_t>(size_t(n));
  unsigned int* counter = ws_n<unsigned int>(WS_COUNTERS, 64) + 40;
  int64_t* src = nullptr;
  int64_t* dst = nullptr;
  gt_graph* core = nullptr;
  try {
    const uint32_t* keep_bits = undirected_degrees(g, cat, deg, "kcore.degree");
    GT_CUDA(cudaMemsetAsync(counter, 0, 4, s));
    {
      Phase ph("kcore.peel", 0.0);
      GT_LAUNCH(gtd::kcore_seed_kernel, grid_for(n, 8), 256, 0, deg, n, k, alive, q0, counter);
    }
    unsigned int h = 0;
    d2h(&h, counter, 4);
    sync();
    int64_t nf = h;
    while (nf > 0) {
      GT_CUDA(cudaMemsetAsync(counter, 0, 4, s));
      {
        Phase ph("kcore.peel", 0.0);
        GT_LAUNCH(gtd::kcore_peel_kernel, warps_grid(nf), 256, 0, cat, g->out_off, g->out_adj,
                  g->in_off, g->in_adj, keep_bits, q0, nf, k, deg, alive, q1, counter);
      }
      d2h(&h, counter, 4);
      sync();
      nf = h;
      std::swap(q0, q1);
    }
    // induced subgraph: every original edge between survivors
    src = dalloc_n<int64_t>(size_t(std::max<int64_t>(g->e, 1)));
    dst = dalloc_n<int64_t>(size_t(std::max<int64_t>(g->e, 1)));
    unsigned long long* ecount = reinterpret_cast<unsigned long long*>(counter + 2);
    GT_CUDA(cudaMemsetAsync(ecount, 0, 8, s));
    {
      Phase ph("kcore.edges", 16.0 * g->e + 8.0 * n);
      GT_LAUNCH(gtd::kcore_edges_kernel,
                static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div64(n, gtd::KC_ROWS),
                                                                          8LL * ctx().sm_count))),
                256, 0, g->ids, g->out_off, g->out_adj, n, alive, src, dst, ecount);
    }
    unsigned long long rows = 0;
    d2h(&rows, ecount, 8);
    sync();
    core = build_csr(src, dst, int64_t(rows), nullptr, 0, true);
    if (core->n > 0)
      GT_LAUNCH(gtd::kcore_ids_kernel, ceil_div(core->n, 256), 256, 0, g->ids, core->n, core->ids);
  } catch (...) {
    dfree(cat); dfree(deg); dfree(alive); dfree(q0); dfree(q1);
    if (src) dfree(src);
    if (dst) dfree(dst);
    throw;
  }
  dfree(cat); dfree(deg); dfree(alive); dfree(q0); dfree(q1); dfree(src); dfree(dst);
  return core;
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_bfs(const gt_graph* g, int64_t source_index, int32_t* dist, int dist_is_device) {
  GT_API_BEGIN
  if (!g) fail(GT_EINVAL, "null graph");
  if (!dist) fail(GT_EINVAL, "dist must not be NULL");
  bfs(g, source_index, dist, dist_is_device != 0);
  GT_API_END
}

int gt_connected_components(const gt_graph* g, int64_t* labels, int labels_is_device,
                            int64_t* n_components) {
  GT_API_BEGIN
  if (!g) fail(GT_EINVAL, "null graph");
  if (g->n && !labels) fail(GT_EINVAL, "labels must not be NULL");
  const int64_t c = g->n ? components(g, labels, labels_is_device != 0) : 0;
  if (n_components) *n_components = c;
  GT_API_END
}

int gt_kcore(const gt_graph* g, int k, gt_graph** out) {
  GT_API_BEGIN
  if (!g || !out) fail(GT_EINVAL, "null graph or output");
  *out = nullptr;
  *out = kcore(g, int32_t(k));
  GT_API_END
}

}  // extern "C"
