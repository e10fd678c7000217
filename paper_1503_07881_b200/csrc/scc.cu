// scc.cu — strongly connected components on the device CSR
// (algorithms.scc, algorithms.py:144-203).
//
// The reference runs an iterative Tarjan over ascending ids and relabels the
// components densely by first occurrence over ascending ids, i.e. in the
// order of each component's smallest id. That labelling depends only on the
// partition, so any exact SCC algorithm reproduces it; here:
//
//   1. trim       nodes with no live in- or no live out-neighbour (self-loops
//                 ignored) are singleton components; repeated a few rounds.
//   2. pivot FB   the live node of largest total degree; its forward set
//                 (BFS over the out-CSR) ∩ its backward set (BFS over the
//                 in-CSR) is its component — on power-law graphs the giant
//                 one — found in O(diameter) frontier levels.
//   3. colouring  every live node takes the minimum live index that reaches
//                 it (worklist propagation with atomicMin); a node whose
//                 colour is its own index is a root, and the nodes of its
//                 colour that reach it (backward worklist inside the colour)
//                 form its component. Every round completes at least the
//                 component of the smallest live node; rounds repeat until no
//                 node is live.
// Each component is represented by its smallest dense index (the root in
// step 3; a reduction in steps 1-2), so labels = rank of the representative
// among the representatives — ascending smallest id, as the reference.
#include "graph.cuh"
#include "scan.cuh"

#include <algorithm>

namespace gtd {

constexpr unsigned SCC_FULL = 0xffffffffu;

// v of every flagged lane appended to queue[*count...], one atomic per warp
// (all 32 lanes call it).
__device__ __forceinline__ void scc_append(bool flag, int32_t v, int32_t* __restrict__ queue,
                                           unsigned int* __restrict__ count) {
  const unsigned b = __ballot_sync(SCC_FULL, flag);
  if (!b) return;
  unsigned base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(count, unsigned(__popc(b)));
  base = __shfl_sync(SCC_FULL, base, 0);
  if (flag) queue[base + __popc(b & lanemask_lt())] = v;
}

__device__ __forceinline__ int32_t scc_of(const int32_t* scc, int32_t v) {
  return __ldcg(scc + v);
}

__global__ void __launch_bounds__(256) scc_init_kernel(int32_t* __restrict__ scc,
                                                       uint32_t* __restrict__ vis, int64_t n) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < n) {
    scc[v] = -1;
    vis[v] = 0;
  }
}

// Singleton components: live nodes without a live out- or in-neighbour.
__global__ void __launch_bounds__(256) scc_trim_kernel(
    const int64_t* __restrict__ out_off, const int32_t* __restrict__ out_adj,
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_adj, int64_t n,
    int32_t* __restrict__ scc, unsigned int* __restrict__ changed) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (scc_of(scc, int32_t(v)) >= 0) continue;
    bool live_out = false, live_in = false;
    for (int64_t e = out_off[v], b = out_off[v + 1]; e < b && !live_out; ++e) {
      const int32_t w = out_adj[e];
      live_out = w != v && scc_of(scc, w) < 0;
    }
    if (live_out)
      for (int64_t e = in_off[v], b = in_off[v + 1]; e < b && !live_in; ++e) {
        const int32_t u = in_adj[e];
        live_in = u != v && scc_of(scc, u) < 0;
      }
    if (!live_out || !live_in) {
      scc[v] = int32_t(v);
      atomicAdd(changed, 1u);
    }
  }
}

// Pivot: live node of largest out+in degree (ties: smallest index).
__global__ void __launch_bounds__(256) scc_pivot_kernel(const int64_t* __restrict__ out_off,
                                                        const int64_t* __restrict__ in_off,
                                                        int64_t n, const int32_t* __restrict__ scc,
                                                        unsigned long long* __restrict__ best) {
  unsigned long long k = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (scc[v] >= 0) continue;
    const uint64_t d = uint64_t(out_off[v + 1] - out_off[v] + in_off[v + 1] - in_off[v]);
    const unsigned long long key =
        (min(d, uint64_t(0x7fffffff)) << 32) | uint64_t(0xffffffffu - uint32_t(v));
    k = max(k, key);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) k = max(k, __shfl_xor_sync(SCC_FULL, k, o));
  if ((threadIdx.x & 31) == 0 && k) atomicMax(best, k);
}

__global__ void scc_seed_kernel(const unsigned long long* __restrict__ best,
                                uint32_t* __restrict__ vis, int32_t* __restrict__ qf,
                                int32_t* __restrict__ qb) {
  const int32_t p = int32_t(0xffffffffu - uint32_t(*best & 0xffffffffull));
  vis[p] = 3u;
  qf[0] = p;
  qb[0] = p;
}

// One frontier level of a reachability search restricted to live nodes:
// warp per frontier node, lanes over its adjacency; newly reached nodes get
// `bit` in vis and join the next frontier.
__global__ void __launch_bounds__(256) scc_reach_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
    const int32_t* __restrict__ q, int64_t nq, const int32_t* __restrict__ scc,
    uint32_t* __restrict__ vis, uint32_t bit, int32_t* __restrict__ next,
    unsigned int* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < nq; i += warps) {
    const int32_t v = q[i];
    const int64_t a = off[v], b = off[v + 1];
    for (int64_t base = a; base < b; base += 32) {
      const int64_t e = base + lane;
      bool app = false;
      int32_t w = 0;
      if (e < b) {
        w = adj[e];
        if (scc[w] < 0 && !(__ldcg(vis + w) & bit)) app = !(atomicOr(vis + w, bit) & bit);
      }
      scc_append(app, w, next, count);
    }
  }
}

// Top-down level for a handful of frontier nodes (the pivot's first level: one
// hub with up to ~10^6 edges): every warp of the grid takes a slice of each
// node's adjacency instead of one warp walking it alone.
__global__ void __launch_bounds__(256) scc_reach_wide_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
    const int32_t* __restrict__ q, int64_t nq, const int32_t* __restrict__ scc,
    uint32_t* __restrict__ vis, uint32_t bit, int32_t* __restrict__ next,
    unsigned int* __restrict__ count) {
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t i = 0; i < nq; ++i) {
    const int32_t v = q[i];
    const int64_t a = off[v], b = off[v + 1];
    for (int64_t base = a + gw * 32; base < b; base += nw * 32) {
      const int64_t e = base + lane;
      bool app = false;
      int32_t w = 0;
      if (e < b) {
        w = adj[e];
        if (scc[w] < 0 && !(__ldcg(vis + w) & bit)) app = !(atomicOr(vis + w, bit) & bit);
      }
      scc_append(app, w, next, count);
    }
  }
}

// Bottom-up level of the same search (direction optimisation, Beamer et al.):
// every live node not yet reached looks for a reached live neighbour along
// the reverse adjacency and stops at the first. Reachability needs no levels,
// so a node may also be reached through one marked earlier in this sweep.
__global__ void __launch_bounds__(256) scc_reach_up_kernel(
    const int64_t* __restrict__ roff, const int32_t* __restrict__ radj, int64_t n,
    const int32_t* __restrict__ scc, uint32_t* __restrict__ vis, uint32_t bit,
    int32_t* __restrict__ next, unsigned int* __restrict__ count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    bool hit = false;
    if (v < n && scc[v] < 0 && !(__ldcg(vis + v) & bit)) {
      for (int64_t e = roff[v], b = roff[v + 1]; e < b; ++e) {
        const int32_t u = radj[e];
        if (scc[u] < 0 && (__ldcg(vis + u) & bit)) {
          hit = true;
          break;
        }
      }
      if (hit) atomicOr(vis + v, bit);
    }
    scc_append(hit, int32_t(v), next, count);
  }
}

// Forward ∩ backward of the pivot: smallest member, then assignment.
__global__ void __launch_bounds__(256) scc_fb_min_kernel(int64_t n, const int32_t* __restrict__ scc,
                                                         const uint32_t* __restrict__ vis,
                                                         int* __restrict__ rep) {
  int m = 0x7fffffff;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    if (scc[v] < 0 && vis[v] == 3u) m = min(m, int(v));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(SCC_FULL, m, o));
  if ((threadIdx.x & 31) == 0 && m != 0x7fffffff) atomicMin(rep, m);
}

__global__ void __launch_bounds__(256) scc_fb_assign_kernel(int64_t n, int32_t* __restrict__ scc,
                                                            uint32_t* __restrict__ vis,
                                                            const int* __restrict__ rep) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int r = *rep;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (scc[v] < 0 && vis[v] == 3u) scc[v] = r;
    vis[v] = 0;
  }
}

// Live nodes into a list; colour = own index.
__global__ void __launch_bounds__(256) scc_live_kernel(int64_t n, const int32_t* __restrict__ scc,
                                                       int32_t* __restrict__ color,
                                                       int32_t* __restrict__ live,
                                                       unsigned int* __restrict__ count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const bool l = v < n && scc[v] < 0;
    if (l) color[v] = int32_t(v);
    scc_append(l, int32_t(v), live, count);
  }
}

// Colour propagation along out-edges among live nodes (minimum wins); a node
// whose colour dropped joins the next worklist once per sweep (stamp).
__global__ void __launch_bounds__(256) scc_color_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
    const int32_t* __restrict__ q, int64_t nq, const int32_t* __restrict__ scc,
    int32_t* __restrict__ color, int32_t* __restrict__ stamp, int32_t sweep,
    int32_t* __restrict__ next, unsigned int* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < nq; i += warps) {
    const int32_t v = q[i];
    const int32_t c = __ldcg(color + v);
    const int64_t a = off[v], b = off[v + 1];
    for (int64_t base = a; base < b; base += 32) {
      const int64_t e = base + lane;
      bool app = false;
      int32_t w = 0;
      if (e < b) {
        w = adj[e];
        if (scc[w] < 0 && __ldcg(color + w) > c && atomicMin(color + w, c) > c)
          app = atomicExch(stamp + w, sweep) != sweep;
      }
      scc_append(app, w, next, count);
    }
  }
}

// Roots (colour == own index) start the backward search of their colour.
__global__ void __launch_bounds__(256) scc_roots_kernel(const int32_t* __restrict__ live,
                                                        int64_t nl,
                                                        const int32_t* __restrict__ color,
                                                        uint32_t* __restrict__ vis,
                                                        int32_t* __restrict__ next,
                                                        unsigned int* __restrict__ count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nl; base += stride) {
    const int64_t i = base + threadIdx.x;
    int32_t v = 0;
    bool r = false;
    if (i < nl) {
      v = live[i];
      r = color[v] == v;
      if (r) vis[v] = 1u;
    }
    scc_append(r, v, next, count);
  }
}

// Backward search inside a colour: in-neighbours of the same colour that are
// not yet marked.
__global__ void __launch_bounds__(256) scc_back_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
    const int32_t* __restrict__ q, int64_t nq, const int32_t* __restrict__ scc,
    const int32_t* __restrict__ color, uint32_t* __restrict__ vis, int32_t* __restrict__ next,
    unsigned int* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < nq; i += warps) {
    const int32_t v = q[i];
    const int32_t c = color[v];
    const int64_t a = off[v], b = off[v + 1];
    for (int64_t base = a; base < b; base += 32) {
      const int64_t e = base + lane;
      bool app = false;
      int32_t u = 0;
      if (e < b) {
        u = adj[e];
        if (scc[u] < 0 && color[u] == c && !__ldcg(vis + u)) app = atomicExch(vis + u, 1u) == 0u;
      }
      scc_append(app, u, next, count);
    }
  }
}

// Marked live nodes take their colour (= their component's smallest index);
// the rest stay live for the next round.
__global__ void __launch_bounds__(256) scc_assign_kernel(const int32_t* __restrict__ live,
                                                         int64_t nl, int32_t* __restrict__ scc,
                                                         const int32_t* __restrict__ color,
                                                         uint32_t* __restrict__ vis,
                                                         unsigned int* __restrict__ remaining) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  const int32_t v = live[i];
  if (vis[v]) {
    scc[v] = color[v];
    vis[v] = 0u;
  } else {
    atomicAdd(remaining, 1u);
  }
}

__global__ void __launch_bounds__(256) scc_flag_kernel(const int32_t* __restrict__ scc, int64_t n,
                                                       int64_t* __restrict__ flag) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < n) flag[v] = scc[v] == int32_t(v) ? 1 : 0;
}

__global__ void __launch_bounds__(256) scc_label_kernel(const int32_t* __restrict__ scc, int64_t n,
                                                        const int64_t* __restrict__ rank,
                                                        int64_t* __restrict__ labels) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < n) labels[v] = rank[scc[v]];
}

}  // namespace gtd

namespace gt {

// bottom-up once the frontier exceeds n / SCC_UP_DIV nodes: on power-law
// graphs the frontier after the pivot's first level already holds most of the
// edges (C2: 8 top-down levels 17.1 ms vs bottom-up sweeps ~0.05 ms each)
constexpr int64_t SCC_UP_DIV = 2048;

static int scc_grid(int64_t items, int per_block) {
  return static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div64(items, per_block), int64_t(ctx().sm_count) * 16)));
}

static unsigned read_counter(const unsigned int* d) {
  unsigned h = 0;
  d2h(&h, d, 4);
  sync();
  return h;
}

static int64_t scc(const gt_graph* g, int64_t* out, bool out_device) {
  require_init();
  const int64_t n = g->n;
  if (n >= (int64_t(1) << 31) - 1) fail(GT_ECAPACITY, "scc: too many nodes");
  cudaStream_t s = ctx().stream;
  int32_t* sc = ws_n<int32_t>(WS_TMP0, size_t(n));
  uint32_t* vis = ws_n<uint32_t>(WS_TMP1, size_t(n));
  int32_t* color = ws_n<int32_t>(WS_TMP2, size_t(n));
  int32_t* q0 = ws_n<int32_t>(WS_TMP3, size_t(n) * 2 + 2);
  int32_t* q1 = q0 + n + 1;
  int32_t* stamp = ws_n<int32_t>(WS_TMP4, size_t(n));
  int32_t* live = reinterpret_cast<int32_t*>(ws_n<uint64_t>(WS_KEYS_A, size_t(n)));
  int64_t* rank = reinterpret_cast<int64_t*>(ws_n<uint64_t>(WS_KEYS_B, size_t(n) + 1));
  unsigned int* cnt = ws_n<unsigned int>(WS_COUNTERS, 64) + 44;
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  unsigned long long* best = reinterpret_cast<unsigned long long*>(small + 11);
  int* rep = reinterpret_cast<int*>(small + 12);
  const int gn = scc_grid(n, 256);
  {
    Phase ph("scc.init", 8.0 * n);
    GT_LAUNCH(gtd::scc_init_kernel, ceil_div(n, 256), 256, 0, sc, vis, n);
    GT_CUDA(cudaMemsetAsync(stamp, 0xff, size_t(n) * 4, s));
  }
  auto trim = [&](int rounds) {
    for (int r = 0; r < rounds; ++r) {
      GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
      {
        Phase ph("scc.trim", 8.0 * n + 16.0 * (n + 1));
        GT_LAUNCH(gtd::scc_trim_kernel, gn, 256, 0, g->out_off, g->out_adj, g->in_off, g->in_adj,
                  n, sc, cnt);
      }
      if (read_counter(cnt) == 0) break;
    }
  };
  // frontier search from q0[0] over (off, adj) marking `bit`; large
  // frontiers switch to bottom-up sweeps over the reverse adjacency
  auto reach = [&](const int64_t* off, const int32_t* adj, const int64_t* roff,
                   const int32_t* radj, uint32_t bit, int32_t* qa, int32_t* qb) {
    int64_t nq = 1;
    while (nq > 0) {
      GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
      {
        const bool up = nq > n / SCC_UP_DIV;
        Phase ph(up ? "scc.reach_up" : "scc.reach_down", 0.0);
        if (up)
          GT_LAUNCH(gtd::scc_reach_up_kernel, gn, 256, 0, roff, radj, n, sc, vis, bit, qb, cnt);
        else if (nq <= 32)
          GT_LAUNCH(gtd::scc_reach_wide_kernel, 4 * ctx().sm_count, 256, 0, off, adj, qa, nq, sc,
                    vis, bit, qb, cnt);
        else
          GT_LAUNCH(gtd::scc_reach_kernel, scc_grid(nq, 8), 256, 0, off, adj, qa, nq, sc, vis,
                    bit, qb, cnt);
      }
      nq = read_counter(cnt);
      std::swap(qa, qb);
    }
  };

  trim(4);
  // pivot forward-backward for the (usually giant) component of the hub
  GT_CUDA(cudaMemsetAsync(best, 0, 8, s));
  {
    Phase ph("scc.pivot", 16.0 * (n + 1) * 2 + 4.0 * n);
    GT_LAUNCH(gtd::scc_pivot_kernel, gn, 256, 0, g->out_off, g->in_off, n, sc, best);
  }
  unsigned long long hb = 0;
  d2h(&hb, best, 8);
  sync();
  if (hb) {
    int32_t* qf = q0;
    int32_t* qb = q1;
    GT_LAUNCH(gtd::scc_seed_kernel, 1, 1, 0, best, vis, qf, live);
    reach(g->out_off, g->out_adj, g->in_off, g->in_adj, 1u, qf, qb);
    GT_CUDA(cudaMemcpyAsync(q0, live, 4, cudaMemcpyDeviceToDevice, s));
    reach(g->in_off, g->in_adj, g->out_off, g->out_adj, 2u, q0, q1);
    const int big = 0x7fffffff;
    GT_CUDA(cudaMemcpyAsync(rep, &big, 4, cudaMemcpyHostToDevice, s));
    Phase ph("scc.pivot", 12.0 * n);
    GT_LAUNCH(gtd::scc_fb_min_kernel, gn, 256, 0, n, sc, vis, rep);
    GT_LAUNCH(gtd::scc_fb_assign_kernel, gn, 256, 0, n, sc, vis, rep);
  }
  trim(2);

  // colouring rounds until no node is live
  int32_t sweep = 0;
  while (true) {
    GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
    {
      Phase ph("scc.color", 8.0 * n);
      GT_LAUNCH(gtd::scc_live_kernel, gn, 256, 0, n, sc, color, live, cnt);
    }
    const int64_t nl = read_counter(cnt);
    if (nl == 0) break;
    GT_CUDA(cudaMemcpyAsync(q0, live, size_t(nl) * 4, cudaMemcpyDeviceToDevice, s));
    int64_t nq = nl;
    int32_t* qa = q0;
    int32_t* qb = q1;
    while (nq > 0) {
      GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
      {
        Phase ph("scc.color", 0.0);
        GT_LAUNCH(gtd::scc_color_kernel, scc_grid(nq, 8), 256, 0, g->out_off, g->out_adj, qa, nq,
                  sc, color, stamp, ++sweep, qb, cnt);
      }
      nq = read_counter(cnt);
      std::swap(qa, qb);
    }
    GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
    {
      Phase ph("scc.back", 0.0);
      GT_LAUNCH(gtd::scc_roots_kernel, scc_grid(nl, 256), 256, 0, live, nl, color, vis, q0, cnt);
    }
    nq = read_counter(cnt);
    qa = q0;
    qb = q1;
    while (nq > 0) {
      GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
      {
        Phase ph("scc.back", 0.0);
        GT_LAUNCH(gtd::scc_back_kernel, scc_grid(nq, 8), 256, 0, g->in_off, g->in_adj, qa, nq, sc,
                  color, vis, qb, cnt);
      }
      nq = read_counter(cnt);
      std::swap(qa, qb);
    }
    GT_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
    {
      Phase ph("scc.assign", 12.0 * nl);
      GT_LAUNCH(gtd::scc_assign_kernel, ceil_div(nl, 256), 256, 0, live, nl, sc, color, vis, cnt);
    }
    if (read_counter(cnt) == 0) break;
    trim(1);
  }

  int64_t* labels = out_device ? out : dalloc_n<int64_t>(size_t(n));
  {
    Phase ph("scc.label", 4.0 * n + 8.0 * n * 3);
    GT_LAUNCH(gtd::scc_flag_kernel, ceil_div(n, 256), 256, 0, sc, n, rank);
    exclusive_scan_i64(rank, n, small + 13);
    GT_LAUNCH(gtd::scc_label_kernel, ceil_div(n, 256), 256, 0, sc, n, rank, labels);
  }
  int64_t n_comp = 0;
  d2h(&n_comp, small + 13, 8);
  if (!out_device) d2h(out, labels, size_t(n) * 8);
  sync();
  if (!out_device) dfree(labels);
  return n_comp;
}

}  // namespace gt

using namespace gt;

extern "C" int gt_scc(const gt_graph* g, int64_t* labels, int labels_is_device,
                      int64_t* n_components) {
  GT_API_BEGIN
  if (!g) fail(GT_EINVAL, "null graph");
  int64_t c = 0;
  if (g->n > 0) {
    if (!labels) fail(GT_EINVAL, "labels must not be NULL");
    c = scc(g, labels, labels_is_device != 0);
  }
  if (n_components) *n_components = c;
  GT_API_END
}
