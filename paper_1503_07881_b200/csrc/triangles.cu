// triangles.cu — exact triangle count of the symmetrised graph.
//
// Reference (algorithms.py:90-119): undirected neighbourhoods = union of in-
// and out-neighbours minus self (graphs.py:163-167); rank nodes by
// (undirected degree, id) (algorithms.py:103-106); keep only higher-ranked
// neighbours (algorithms.py:108); total = sum over oriented arcs (u,v) of
// |N+(u) ∩ N+(v)| (algorithms.py:110-116).
//
// Device pipeline (everything after step 2 lives in RANK space: node r is the
// r-th smallest (degree, id), so N+(r) ⊂ (r, n) and hubs sit at the top):
//   1 cand_degree_kernel edge-parallel over the 2E "candidate slots" out(i) ++
//                        in(i): a slot is an undirected neighbour unless it is
//                        a self-loop or an in-slot whose source is also in the
//                        sorted out-row (binary search) -> undirected degree
//   2 rank               radix sort of (degree, id) keys -> rank[id]
//   3 fill_rows          warp per row: the higher-ranked candidates as rank
//                        values, compacted into a degree-sized slice and
//                        sorted in place (shuffle / shared-memory bitonic)
//   4 place_rows         rows moved to their rank-space slot (offsets = scans
//                        of d+ and deg - d+ in rank order) -> oriented CSR N+;
//                        every arc (u,v) filed under N-(v) as the suffix of
//                        N+(u) after v: (first index, remaining length)
//   5 count              task = (v, chunk of N-(v)), one warp each. The N+(v)
//                        membership structure is a per-warp shared-memory
//                        BITMAP over (v, n) when n-1-v <= 2^16 (the top ranks,
//                        where R-MAT puts nearly all the work: 94% at C3),
//                        else a per-warp hash table (or per CTA for large
//                        d+(v)). For every arc (u,v) the warp probes the
//                        suffix of N+(u) after v — exactly the w > v
//                        candidates — with coalesced reads; each triangle
//                        u<v<w is counted once, at its middle vertex v.
// Work = sum over u of d+(u)(d+(u)-1)/2 probes. All arithmetic is integer:
// exact and independent of scheduling.
#include "graph.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "segment.cuh"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace gtd {

constexpr int TC_CAND_TILE = 2048;             // slots per CTA in cand_kernel
constexpr int TC_ROWS_CAP = TC_CAND_TILE + 2;  // staged row offsets per tile
constexpr int TC_SLOTS = 2048;                 // hash slots per warp (8 KB)
constexpr int TC_WARP_MAX = TC_SLOTS / 4;      // largest d+(v) of a warp hash task
#ifndef GT_TC_CHUNK
#define GT_TC_CHUNK 256
#endif
constexpr int TC_CHUNK = GT_TC_CHUNK;          // arcs per warp task
#ifndef GT_TC_CHUNK_CTA
#define GT_TC_CHUNK_CTA 16384
#endif
constexpr int TC_CHUNK_CTA = GT_TC_CHUNK_CTA;  // arcs per CTA task (v order, C4: 1024 -> 16384 = 219 -> 183 ms)
constexpr int TC_BM_BITS = TC_SLOTS * 32;      // per-warp bitmap window (same 8 KB region)
constexpr int TC_SPLIT_TOP = TC_BM_BITS / 2;   // split tables: bitmap of the top 2^15 ranks ...
constexpr int TC_SPLIT_SLOTS = TC_SLOTS / 2;   // ... + hash of the rest (4 KB each)
constexpr int TC_SPLIT_MAX = TC_SPLIT_SLOTS / 4;  // largest d+(v) of a split task
constexpr int32_t TC_EMPTY = -1;
// (register-budget knobs for sweeps: -DGT_PLACE_MINB=k / -DGT_FILL_MINB=k)
#ifdef GT_PLACE_MINB
#define GT_LB_PLACE __launch_bounds__(256, GT_PLACE_MINB)
#else
#define GT_LB_PLACE __launch_bounds__(256)
#endif
#ifdef GT_FILL_MINB
#define GT_LB_FILL __launch_bounds__(256, GT_FILL_MINB)
#else
#define GT_LB_FILL __launch_bounds__(256)
#endif

__global__ void __launch_bounds__(256) cat_off_kernel(const int64_t* __restrict__ out_off,
                                                      const int64_t* __restrict__ in_off,
                                                      int64_t n, int64_t* __restrict__ cat) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i <= n) cat[i] = out_off[i] + in_off[i];
}

// Largest r in [lo, hi] with off[r] <= e (the row holding slot e).
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ off, int64_t lo, int64_t hi,
                                          int64_t e) {
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ bool bsearch_in(const int32_t* __restrict__ list, int64_t len,
                                           int32_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (list[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && list[lo] == x;
}

// tile_row[t] = row holding slot t*TC_CAND_TILE (one binary search per tile,
// all tiles in parallel, so the candidate kernels start without a serial
// search chain in their prologue); tile_row[tiles] = n - 1.
__global__ void __launch_bounds__(256) cand_tile_rows_kernel(const int64_t* __restrict__ cat,
                                                             int64_t n, int64_t slots,
                                                             int64_t tiles,
                                                             int64_t* __restrict__ tile_row) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > tiles) return;
  const int64_t e = t < tiles ? t * TC_CAND_TILE : slots - 1;
  tile_row[t] = row_of(cat, 0, n - 1, e);
}

// Edge-parallel pass over the concatenated candidate slots of all rows:
// deg[row] += candidate slots (the undirected degree, graphs.py:163-167), and
// one keep bit per slot (keep_bits, 2E bits) for the row-parallel fill.
// Per 2048-slot tile, in shared memory: the tile's row offsets (relative to
// the tile, int32), the slot -> row map (row heads scattered, then a block
// max-scan: no per-slot search), and the tile's neighbour ids, so the
// reciprocity test of an in-slot (is its source also in the sorted out-row?)
// is a shared-memory binary search whenever that out-row lies in the tile.
// Tiles with more than TC_ROWS_CAP - 2 rows (only possible with isolated
// nodes) map slots by a global binary search instead.
__global__ void __launch_bounds__(256) cand_degree_kernel(
    const int64_t* __restrict__ cat, const int64_t* __restrict__ tile_row,
    const int64_t* __restrict__ out_off, const int32_t* __restrict__ out_adj,
    const int32_t* __restrict__ in_adj, int64_t n, int64_t slots, int32_t* __restrict__ deg,
    uint32_t* __restrict__ keep_bits) {
  constexpr int T = TC_CAND_TILE, PER = T / 256;
  __shared__ int32_t s_c[TC_ROWS_CAP];  // cat[r0 + i] - e0
  __shared__ int32_t s_o[TC_ROWS_CAP];  // out_off[r0 + i] - out_off[r0]
  __shared__ __align__(16) int32_t s_row[T];  // slot -> row - r0
  __shared__ int32_t s_j[T];
  __shared__ int32_t s_wmax[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t e0 = int64_t(blockIdx.x) * T;
  const int64_t r0 = tile_row[blockIdx.x], r1 = tile_row[blockIdx.x + 1];
  const int64_t oo0 = out_off[r0];
  const int64_t nr = r1 - r0 + 2;  // rows r0..r1 plus the end offset of r1
  const bool staged = nr <= TC_ROWS_CAP;
  const int tn = int(slots - e0 < T ? slots - e0 : int64_t(T));
  if (staged) {
    for (int i = tid; i < int(nr); i += 256) {
      s_c[i] = int32_t(cat[r0 + i] - e0);
      s_o[i] = int32_t(out_off[r0 + i] - oo0);
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) s_row[q * 256 + tid] = 0;
    __syncthreads();
    // heads of the non-empty rows that start inside the tile (distinct slots)
    for (int i = tid + 1; i < int(nr) - 1; i += 256) {
      const int32_t c = s_c[i];
      if (c < T && s_c[i + 1] > c) s_row[c] = i;
    }
    __syncthreads();
    // inclusive max-scan: thread t owns slots [8t, 8t+8)
    int4 a = reinterpret_cast<int4*>(s_row)[2 * tid];
    int4 b = reinterpret_cast<int4*>(s_row)[2 * tid + 1];
    a.y = max(a.y, a.x); a.z = max(a.z, a.y); a.w = max(a.w, a.z);
    b.x = max(b.x, a.w); b.y = max(b.y, b.x); b.z = max(b.z, b.y); b.w = max(b.w, b.z);
    int run = b.w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, run, o);
      if (lane >= o) run = max(run, y);
    }
    if (lane == 31) s_wmax[warp] = run;
    int excl = __shfl_up_sync(0xffffffffu, run, 1);
    if (lane == 0) excl = 0;
    __syncthreads();
    for (int w = 0; w < warp; ++w) excl = max(excl, s_wmax[w]);
    a.x = max(a.x, excl); a.y = max(a.y, excl); a.z = max(a.z, excl); a.w = max(a.w, excl);
    b.x = max(b.x, excl); b.y = max(b.y, excl); b.z = max(b.z, excl); b.w = max(b.w, excl);
    reinterpret_cast<int4*>(s_row)[2 * tid] = a;
    reinterpret_cast<int4*>(s_row)[2 * tid + 1] = b;
  } else {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = q * 256 + tid;
      if (t < tn) s_row[t] = int32_t(row_of(cat, r0, r1, e0 + t) - r0);
    }
  }
  __syncthreads();
  // The rest of the tile, generic over the index type: 32-bit tile-relative
  // offsets when the rows are staged (every tile but those of isolated-node
  // runs; ncu: the kernel is issue-bound and most of its integer work was
  // 64-bit offset arithmetic), 64-bit offsets read from global memory otherwise.
  // c_at(ri): row start (tile-relative slot); o_at(ri): out-row extent.
  auto tile_body = [&](auto zero, auto c_at, auto o_at) {
    using I = decltype(zero);
    // ---- neighbour ids of the tile (all loads issued before any is consumed) ----
    int32_t j[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = q * 256 + tid;
      j[q] = 0;
      if (t < tn) {
        const int ri = s_row[t];
        const I c = c_at(ri), oa = o_at(ri), no = o_at(ri + 1) - oa;
        const I k = I(t) - c;
        j[q] = k < no ? out_adj[oo0 + oa + k] : in_adj[(e0 - oo0) + (c - oa) + (k - no)];
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) s_j[q * 256 + tid] = j[q];
    __syncthreads();

    // drop self-loops and in-slots whose source is also an out-neighbour
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = q * 256 + tid;
      const bool valid = t < tn;
      bool cand = false;
      int ri = -1;
      if (valid) {
        ri = s_row[t];
        cand = int64_t(j[q]) != r0 + ri;
        const I c = c_at(ri), oa = o_at(ri), no = o_at(ri + 1) - oa;
        if (cand && I(t) - c >= no) {
          if (c >= 0) {  // the whole out-row [c, c+no) precedes t inside the tile
            int lo = int(c), hi = int(c + no);
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (s_j[mid] < j[q]) lo = mid + 1;
              else hi = mid;
            }
            cand = !(lo < int(c + no) && s_j[lo] == j[q]);
          } else {
            cand = !bsearch_in(out_adj + oo0 + oa, no, j[q]);
          }
        }
      }
      // per-row counts: the 32 slots of a warp step are consecutive, so each
      // row is a run of lanes; the first lane of a run adds the run's count
      const unsigned active = __ballot_sync(0xffffffffu, valid);
      const unsigned kb = __ballot_sync(0xffffffffu, cand);
      if (lane == 0 && active) keep_bits[(e0 + q * 256 + warp * 32) >> 5] = kb;
      const int prev = __shfl_up_sync(0xffffffffu, ri, 1);
      const bool head = valid && (lane == 0 || prev != ri);
      const unsigned heads = __ballot_sync(0xffffffffu, head);
      if (head) {
        const unsigned after = heads & ~((2u << lane) - 1u);  // later heads
        const unsigned runm = (after ? (after & (0u - after)) - 1u : 0xffffffffu) & ~((1u << lane) - 1u);
        const int cnt = __popc(kb & runm);
        if (cnt) atomicAdd(&deg[r0 + ri], cnt);
      }
    }
  };
  if (staged)
    tile_body(int32_t(0), [&](int ri) -> int32_t { return s_c[ri]; },
              [&](int ri) -> int32_t { return s_o[ri]; });
  else
    tile_body(int64_t(0), [&](int ri) -> int64_t { return cat[r0 + ri] - e0; },
              [&](int ri) -> int64_t { return out_off[r0 + ri] - oo0; });
}

// ---- rank (algorithms.py:103-106: lexsort by (degree, id)) ------------------

__global__ void __launch_bounds__(256) rank_keys_kernel(const int32_t* __restrict__ deg, int64_t n,
                                                        int kbits, SortPlan plan,
                                                        unsigned long long* __restrict__ hist,
                                                        uint64_t* __restrict__ keys) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = (uint64_t(uint32_t(deg[i])) << kbits) | uint64_t(i);
    keys[i] = k;
    plan_hist_add(sh, plan, k);
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

__global__ void __launch_bounds__(256) rank_scatter_kernel(const uint64_t* __restrict__ sorted,
                                                           int64_t n, uint64_t lowmask,
                                                           int32_t* __restrict__ rank,
                                                           int32_t* __restrict__ order) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t id = int32_t(sorted[r] & lowmask);
  rank[id] = int32_t(r);
  order[r] = id;
}

__global__ void __launch_bounds__(256) max_i32_kernel(const int32_t* __restrict__ x, int64_t n,
                                                      int* __restrict__ out) {
  int mx = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    mx = max(mx, x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// ---- rank-space oriented CSR without a global sort ---------------------------
// fill_rows: warp per id-row i: the candidates of i (out(i) ++ in(i), self and
// in-slots already in the sorted out-row dropped) of higher rank, as rank
// values, compacted into the row's slice of `buf` (capacity deg(i), offsets
// = scan of the undirected degrees) and sorted there (shuffle bitonic up to
// 32, per-warp shared-memory bitonic up to TC_SORT_WARP); d+(i) recorded.
// Rows with more than TC_FILL_BIG candidates go to fill_rows_big (CTA per
// row); rows with more than TC_SORT_WARP survivors to sort_rows_big.
constexpr int TC_FILL_BIG = 4096;
constexpr int TC_SORT_WARP = 512;
constexpr int TC_SORT_CTA = 16384;

__device__ __forceinline__ uint64_t warp_bitonic32_u64(uint64_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = ((lower == up) == (y < x)) ? y : x;
    }
  }
  return x;
}

__device__ __forceinline__ int32_t warp_bitonic32(int32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = (lower == up) ? min(x, y) : max(x, y);
    }
  }
  return x;
}

// Bitonic sort of s[0, p) (p a power of two) by the threads [0, nthreads) of
// the caller group; `sync` is the group barrier.
template <typename Sync>
__device__ __forceinline__ void bitonic_smem(int32_t* s, int p, int t0, int nthreads, Sync sync) {
  for (int k = 2; k <= p; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int lj = __ffs(j) - 1;  // j is a power of two: no integer division
      for (int t = t0; t < p / 2; t += nthreads) {
        const int e = ((t >> lj) << (lj + 1)) + (t & (j - 1));
        const int f = e + j;
        const bool up = (e & k) == 0;
        const int32_t a = s[e], b = s[f];
        if ((a > b) == up) {
          s[e] = b;
          s[f] = a;
        }
      }
      sync();
    }
  }
}

// Stable LSD radix sort (8-bit digits over the low `kbits` bits) of row[0,
// cnt) by one warp, cnt <= TC_SORT_WARP: the row is read from global memory
// once, the passes ping-pong between two per-warp shared buffers, and the
// sorted row is written back once. Per pass a shared histogram, its scan,
// and a rank/scatter in index order (__match_any_sync peers).
__device__ __forceinline__ void warp_radix_sort(int32_t* row, int cnt, int32_t* sa, int32_t* sb,
                                                uint32_t* hist, int kbits) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  for (int k = lane; k < cnt; k += 32) sa[k] = row[k];
  int32_t* src = sa;
  int32_t* dst = sb;
  for (int shift = 0; shift < kbits; shift += 8) {
#pragma unroll
    for (int b = lane; b < 256; b += 32) hist[b] = 0u;
    __syncwarp();
    for (int k = lane; k < cnt; k += 32) atomicAdd(&hist[(uint32_t(src[k]) >> shift) & 255u], 1u);
    __syncwarp();
    uint32_t h[8], tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      h[q] = hist[lane * 8 + q];
      tot += h[q];
    }
    uint32_t run = warp_incl_scan(tot) - tot;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      hist[lane * 8 + q] = run;
      run += h[q];
    }
    __syncwarp();
    for (int k0 = 0; k0 < cnt; k0 += 32) {
      const int k = k0 + lane;
      const bool valid = k < cnt;
      const int32_t x = valid ? src[k] : 0;
      const uint32_t d = valid ? (uint32_t(x) >> shift) & 255u : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const int leader = 31 - __clz(peers);
      uint32_t before = 0;
      if (valid && lane == leader) before = atomicAdd(&hist[d], __popc(peers));
      before = __shfl_sync(0xffffffffu, before, leader);
      if (valid) dst[before + __popc(peers & lt)] = x;
    }
    __syncwarp();
    int32_t* t = src;
    src = dst;
    dst = t;
  }
  for (int k = lane; k < cnt; k += 32) row[k] = src[k];
  __syncwarp();
}

__global__ void __launch_bounds__(256) i32_to_u64_kernel(const int32_t* __restrict__ in, int64_t n,
                                                         uint64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = uint64_t(uint32_t(in[i]));
}

__global__ void __launch_bounds__(256) u64_to_i32_kernel(const uint64_t* __restrict__ in, int64_t n,
                                                         int32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = int32_t(in[i]);
}

__global__ void __launch_bounds__(256) deg64_kernel(const int32_t* __restrict__ deg, int64_t n,
                                                    int64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = deg[i];
}

__device__ __forceinline__ bool slot_kept(const uint32_t* __restrict__ bits, int64_t slot) {
  return (__ldg(bits + (slot >> 5)) >> (slot & 31)) & 1u;
}

__device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
  return static_cast<int64_t>(__shfl_sync(0xffffffffu, static_cast<long long>(v), src));
}

// Warp per batch of 32 consecutive id-rows: the rows' offsets, rank and slot
// base are loaded once, coalesced (lane l holding row base+l), and broadcast
// by shuffle (measured faster than interleaving the rows across warps).
// Rows with at most 32 candidates are packed several to a warp step (below);
// longer rows take the warp one at a time.
__global__ void GT_LB_FILL fill_rows_kernel(
    const int64_t* __restrict__ cat, const int64_t* __restrict__ out_off,
    const int32_t* __restrict__ out_adj, const int64_t* __restrict__ in_off,
    const int32_t* __restrict__ in_adj, int64_t n, const int32_t* __restrict__ rank,
    const uint32_t* __restrict__ keep_bits, const int64_t* __restrict__ und_off,
    int32_t* __restrict__ buf, int32_t* __restrict__ dplus, int32_t* __restrict__ big_fill,
    int32_t* __restrict__ big_sort, unsigned int* __restrict__ nbig, int kbits) {
  __shared__ int32_t s_sort[8][TC_SORT_WARP];
  __shared__ int32_t s_tmp[8][TC_SORT_WARP];
  __shared__ uint32_t s_hist[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int64_t nbatch = (n + 31) >> 5;
  const int64_t nwarps = int64_t(gridDim.x) * 8;
  for (int64_t bt = int64_t(blockIdx.x) * 8 + warp; bt < nbatch; bt += nwarps) {
    const int64_t base = bt << 5;
    const int64_t me = base + lane;
    int64_t m_oo = 0, m_io = 0, m_c = 0, m_uo = 0;
    int32_t m_no = 0, m_tot = -1, m_r = 0;
    if (me < n) {
      m_oo = out_off[me];
      m_io = in_off[me];
      const int64_t no = out_off[me + 1] - m_oo, ni = in_off[me + 1] - m_io;
      m_c = cat[me];
      m_uo = und_off[me];
      m_r = rank[me];
      m_no = int32_t(no);
      m_tot = no + ni > TC_FILL_BIG ? -1 : int32_t(no + ni);
      if (no + ni > TC_FILL_BIG) {  // hub row: fill_big_kernel, d+ is its cursor
        dplus[me] = 0;
        big_fill[atomicAdd(&nbig[0], 1u)] = int32_t(me);
      }
    }
    // rows with 1..32 candidates, packed: the next rows (in lane order) whose
    // candidates fit in 32 lanes share one step — element -> row by a shuffle
    // binary search over the packed prefix, survivors sorted by (row, rank)
    // in one 64-bit shuffle bitonic, each landing at its index in its row
    if (me < n && m_tot == 0) dplus[me] = 0;
    unsigned todo = __ballot_sync(0xffffffffu, m_tot > 0 && m_tot <= 32);
    while (todo) {
      const bool in = (todo >> lane) & 1u;
      int inc = in ? m_tot : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int ex = inc - (in ? m_tot : 0);
      const bool take = in && inc <= 32;
      todo &= ~__ballot_sync(0xffffffffu, take);
      const int G = __reduce_max_sync(0xffffffffu, take ? unsigned(inc) : 0u);
      int k = 0;  // the last lane whose packed prefix is <= lane: this element's row
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (__shfl_sync(0xffffffffu, ex, k + st) <= lane) k += st;
      const int t = lane - __shfl_sync(0xffffffffu, ex, k);
      const int64_t c = shfl64(m_c, k), oo = shfl64(m_oo, k), io = shfl64(m_io, k);
      const int32_t no = __shfl_sync(0xffffffffu, m_no, k);
      const int32_t ri = __shfl_sync(0xffffffffu, m_r, k);
      bool keep = lane < G && slot_kept(keep_bits, c + t);
      int32_t val = keep ? (t < no ? out_adj[oo + t] : in_adj[io + (t - no)]) : 0;
      if (keep) {
        val = rank[val];
        keep = val > ri;
      }
      const unsigned sb = __ballot_sync(0xffffffffu, keep);
      if (take) {
        const unsigned rm = (m_tot == 32 ? 0xffffffffu : ((1u << m_tot) - 1u)) << ex;
        dplus[me] = __popc(sb & rm);
      }
      if (sb == 0) continue;
      uint64_t key = keep ? (uint64_t(k) << 32) | uint32_t(val) : ~0ull;
      key = warp_bitonic32_u64(key);
      const bool has = key != ~0ull;
      const int k2 = has ? int(key >> 32) : 0;
      const unsigned peers = __match_any_sync(0xffffffffu, uint32_t(key >> 32));
      const int64_t uo = shfl64(m_uo, k2);
      if (has) buf[uo + __popc(peers & lt)] = int32_t(uint32_t(key));
    }
    const int rows = n - base < 32 ? int(n - base) : 32;
    for (int k = 0; k < rows; ++k) {
      const int32_t total = __shfl_sync(0xffffffffu, m_tot, k);
      if (total <= 32) continue;  // packed above, or chunked by the big-row kernels
      const int64_t i = base + k;
      const int64_t oo = shfl64(m_oo, k), io = shfl64(m_io, k), c = shfl64(m_c, k);
      const int32_t no = __shfl_sync(0xffffffffu, m_no, k);
      const int32_t ri = __shfl_sync(0xffffffffu, m_r, k);
      int32_t* row = buf + shfl64(m_uo, k);
      int cnt = 0;
      for (int64_t k0 = 0; k0 < total; k0 += 128) {  // 4 x 32 candidates in flight
        int32_t val[4];
        bool keep[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t q = k0 + 32 * u + lane;
          keep[u] = q < total && slot_kept(keep_bits, c + q);
          val[u] = keep[u] ? (q < no ? out_adj[oo + q] : in_adj[io + (q - no)]) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (keep[u]) {
            val[u] = rank[val[u]];
            keep[u] = val[u] > ri;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned b = __ballot_sync(0xffffffffu, keep[u]);
          if (keep[u]) row[cnt + __popc(b & lt)] = val[u];
          cnt += __popc(b);
        }
      }
      if (lane == 0) dplus[i] = cnt;
      __syncwarp();
      if (cnt <= 32) {
        int32_t x = lane < cnt ? row[lane] : INT_MAX;
        x = warp_bitonic32(x);
        if (lane < cnt) row[lane] = x;
      } else if (cnt <= TC_SORT_WARP) {
        warp_radix_sort(row, cnt, s_sort[warp], s_tmp[warp], s_hist[warp], kbits);
      } else if (lane == 0) {
        big_sort[atomicAdd(&nbig[1], 1u)] = int32_t(i);
      }
      __syncwarp();
    }
  }
}

// Rows with more than TC_FILL_BIG candidates (hubs), in chunks of
// TC_BIG_CHUNK candidates, one pass: a CTA takes a chunk, compacts its
// survivors and claims their place in the row with one atomicAdd on the row's
// d+ (zeroed by fill_rows; the row is sorted afterwards, so the order in which
// chunks land does not matter). Chunks are numbered by a scan of the rows'
// chunk counts; CTAs stride over them, so the host needs no chunk list.
constexpr int TC_BIG_CHUNK = 2048;

__global__ void __launch_bounds__(256) big_chunk_count_kernel(const int32_t* __restrict__ rows,
                                                              int nr,
                                                              const int64_t* __restrict__ cat,
                                                              int64_t* __restrict__ chunks) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const int64_t i = rows[r];
  chunks[r] = (cat[i + 1] - cat[i] + TC_BIG_CHUNK - 1) / TC_BIG_CHUNK;
}

__global__ void __launch_bounds__(256) fill_big_kernel(
    const int32_t* __restrict__ rows, int nr, const int64_t* __restrict__ coff,
    const int64_t* __restrict__ cat, const int64_t* __restrict__ out_off,
    const int32_t* __restrict__ out_adj, const int64_t* __restrict__ in_off,
    const int32_t* __restrict__ in_adj, const int32_t* __restrict__ rank,
    const uint32_t* __restrict__ keep_bits, const int64_t* __restrict__ und_off,
    int32_t* __restrict__ buf, int32_t* __restrict__ dplus) {
  constexpr int PER = TC_BIG_CHUNK / 256;
  __shared__ uint32_t s_scan[8];
  __shared__ int32_t s_base;
  const int64_t nchunks = coff[nr];
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    int lo = 0, hi = nr - 1;  // the row holding chunk ch: last r with coff[r] <= ch
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (coff[mid] <= ch) lo = mid;
      else hi = mid - 1;
    }
    const int64_t i = rows[lo];
    const int64_t oo = out_off[i], no = out_off[i + 1] - oo, io = in_off[i];
    const int64_t c = cat[i], total = cat[i + 1] - c;
    const int32_t ri = rank[i];
    const int64_t k0 = (ch - coff[lo]) * TC_BIG_CHUNK;
    int32_t val[PER];
    bool keep[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t k = k0 + q * 256 + threadIdx.x;
      keep[q] = k < total && slot_kept(keep_bits, c + k);
      val[q] = keep[q] ? (k < no ? out_adj[oo + k] : in_adj[io + (k - no)]) : 0;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if (keep[q]) {
        val[q] = rank[val[q]];
        keep[q] = val[q] > ri;
      }
      mine += keep[q] ? 1u : 0u;
    }
    uint32_t tot;
    const uint32_t pre = block_excl_scan_256<uint32_t>(mine, s_scan, tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(&dplus[i], int32_t(tot)) : 0;
    __syncthreads();
    int32_t* out = buf + und_off[i] + s_base + pre;
    __syncthreads();  // s_base is rewritten by the next chunk
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (keep[q]) *out++ = val[q];
  }
}

// Appends rows[0, n) to list[0, n) (the hub rows join the rows to sort).
__global__ void copy_rows_kernel(const int32_t* __restrict__ rows, int n, int32_t* __restrict__ list) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) list[r] = rows[r];
}

// out[r] = a[rows[r]] (+ a[rows[r] + 1] into out[nr + r] when `both`).
__global__ void gather_rows_kernel(const int32_t* __restrict__ rows, int nr,
                                   const int64_t* __restrict__ a64, const int32_t* __restrict__ a32,
                                   int both, int64_t* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const int64_t i = rows[r];
  out[r] = a64 ? a64[i] : int64_t(a32[i]);
  if (both) out[nr + r] = a64[i + 1];
}

// Listed rows (d+ > TC_SORT_WARP, and the hub rows) up to TC_SORT_MID: warp
// per row (4 per CTA), the same shared-memory radix sort with larger per-warp
// buffers (dynamic smem); longer rows only raise *max_big.
constexpr int TC_SORT_MID = 2048;
__global__ void __launch_bounds__(128) sort_rows_mid_kernel(const int32_t* __restrict__ rows, int nr,
                                                            const int64_t* __restrict__ und_off,
                                                            const int32_t* __restrict__ dplus,
                                                            int32_t* __restrict__ buf, int kbits,
                                                            unsigned int* __restrict__ max_big) {
  extern __shared__ int32_t s_dyn[];
  const int warp = threadIdx.x >> 5;
  int32_t* sa = s_dyn + warp * (2 * TC_SORT_MID + 256);
  int32_t* sb = sa + TC_SORT_MID;
  uint32_t* hist = reinterpret_cast<uint32_t*>(sb + TC_SORT_MID);
  for (int r = blockIdx.x * 4 + warp; r < nr; r += gridDim.x * 4) {
    const int64_t i = rows[r];
    const int cnt = dplus[i];
    if (cnt > TC_SORT_MID) {  // left to the CTA sorts
      if ((threadIdx.x & 31) == 0) atomicMax(max_big, unsigned(cnt));
      continue;
    }
    if (cnt > 1) warp_radix_sort(buf + und_off[i], cnt, sa, sb, hist, kbits);
  }
}

// CTA bitonic sort of the rows with TC_SORT_MID < d+ <= TC_SORT_CTA (dynamic smem).
__global__ void __launch_bounds__(256) sort_rows_big_kernel(const int32_t* __restrict__ rows,
                                                            const int64_t* __restrict__ und_off,
                                                            const int32_t* __restrict__ dplus,
                                                            int32_t* __restrict__ buf) {
  extern __shared__ int32_t s_dyn[];
  const int64_t i = rows[blockIdx.x];
  const int cnt = dplus[i];
  if (cnt > TC_SORT_CTA) return;  // host falls back to a radix sort
  int32_t* row = buf + und_off[i];
  int p = 64;
  while (p < cnt) p <<= 1;
  for (int t = threadIdx.x; t < p; t += 256) s_dyn[t] = t < cnt ? row[t] : INT_MAX;
  __syncthreads();
  bitonic_smem(s_dyn, p, int(threadIdx.x), 256, [] { __syncthreads(); });
  for (int t = threadIdx.x; t < cnt; t += 256) row[t] = s_dyn[t];
}

// Rank-order counts: dp[rank i] = d+(i), dm[rank i] = deg(i) - d+(i).
__global__ void __launch_bounds__(256) rank_counts_kernel(const int32_t* __restrict__ rank,
                                                          const int32_t* __restrict__ deg,
                                                          const int32_t* __restrict__ dplus,
                                                          int64_t n, int64_t* __restrict__ dp,
                                                          int64_t* __restrict__ dm) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t r = rank[i];
  dp[r] = dplus[i];
  dm[r] = deg[i] - dplus[i];
}

// Warp per rank-row (ascending, so N-(v) lists come out nearly sorted by u,
// which keeps the count's suffix reads local): the sorted row moves to its
// rank-space slot of adj_p, and every arc (u,v) at position a is filed under
// N-(v) as (a+1, remaining length of N+(u)); the exact order inside an N-(v)
// list is scheduling dependent, the count is not.
__global__ void __launch_bounds__(256) place_rows_kernel(
    const int32_t* __restrict__ order, const int64_t* __restrict__ und_off,
    const int32_t* __restrict__ dplus, const int32_t* __restrict__ buf, int64_t n,
    const int64_t* __restrict__ off_p, const int64_t* __restrict__ off_m,
    int32_t* __restrict__ adj_p, unsigned int* __restrict__ cur, int2* __restrict__ nm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * 8;
  for (int64_t r = int64_t(blockIdx.x) * 8 + warp; r < n; r += nwarps) {
    const int64_t i = order[r];
    const int cnt = dplus[i];
    if (cnt == 0) continue;
    const int32_t* row = buf + und_off[i];
    const int64_t a0 = off_p[r];
    for (int t = lane; t < cnt; t += 32) {
      const int32_t v = row[t];
      const int64_t a = a0 + t;
      adj_p[a] = v;
      const unsigned slot = atomicAdd(&cur[v], 1u);
      nm[off_m[v] + slot] = make_int2(int(a + 1), cnt - t - 1);
    }
  }
}

// Arc-parallel version of place_rows_kernel: 2048-arc tiles of the
// rank-space CSR, the tile's rows staged in shared memory (start, buffer
// base) with the slot -> row map built like cand_degree_kernel's. Each thread
// handles 8 arcs and has all 8 N-(v) slot claims (returning atomics) in
// flight at once, where the warp-per-row kernel waited on one claim per lane
// per row (latency-bound: rows average ~30 arcs).
__global__ void GT_LB_PLACE place_tiles_kernel(
    const int64_t* __restrict__ off_p, const int64_t* __restrict__ tile_row, int64_t m,
    const int32_t* __restrict__ order, const int64_t* __restrict__ und_off,
    const int32_t* __restrict__ buf, unsigned long long* __restrict__ cur64,
    int32_t* __restrict__ adj_p, int2* __restrict__ nm) {
  // cur64[v] starts at off_m[v]: the claim returns the absolute N- slot, so an
  // arc costs two random accesses (the claim, the nm store) instead of three
  // (claim, off_m[v], store)
  constexpr int T = TC_CAND_TILE, PER = T / 256;
  // (per-tile aggregation of the slot claims through a shared hash measured
  // slower at C4: 52.6 vs 45.3 ms — the claims are not serialising on hubs)
  constexpr size_t RAW = size_t(TC_ROWS_CAP) * 12 + size_t(T) * 4;
  __shared__ __align__(16) unsigned char s_raw[RAW];
  int64_t* s_b = reinterpret_cast<int64_t*>(s_raw);                       // und_off[order[r0 + i]]
  int32_t* s_row = reinterpret_cast<int32_t*>(s_raw + TC_ROWS_CAP * 8);   // slot -> row - r0
  int32_t* s_c = s_row + T;                                               // off_p[r0 + i] - e0
  __shared__ int32_t s_wmax[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t e0 = int64_t(blockIdx.x) * T;
  const int64_t r0 = tile_row[blockIdx.x], r1 = tile_row[blockIdx.x + 1];
  const int64_t nr = r1 - r0 + 2;
  const bool staged = nr <= TC_ROWS_CAP;
  const int tn = int(m - e0 < T ? m - e0 : int64_t(T));
  if (staged) {
    for (int i = tid; i < int(nr); i += 256) {
      s_c[i] = int32_t(off_p[r0 + i] - e0);
      if (i < int(nr) - 1) s_b[i] = und_off[order[r0 + i]];
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) s_row[q * 256 + tid] = 0;
    __syncthreads();
    for (int i = tid + 1; i < int(nr) - 1; i += 256) {
      const int32_t c = s_c[i];
      if (c < T && s_c[i + 1] > c) s_row[c] = i;
    }
    __syncthreads();
    int4 a = reinterpret_cast<int4*>(s_row)[2 * tid];
    int4 b = reinterpret_cast<int4*>(s_row)[2 * tid + 1];
    a.y = max(a.y, a.x); a.z = max(a.z, a.y); a.w = max(a.w, a.z);
    b.x = max(b.x, a.w); b.y = max(b.y, b.x); b.z = max(b.z, b.y); b.w = max(b.w, b.z);
    int run = b.w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, run, o);
      if (lane >= o) run = max(run, y);
    }
    if (lane == 31) s_wmax[warp] = run;
    int excl = __shfl_up_sync(0xffffffffu, run, 1);
    if (lane == 0) excl = 0;
    __syncthreads();
    for (int w = 0; w < warp; ++w) excl = max(excl, s_wmax[w]);
    a.x = max(a.x, excl); a.y = max(a.y, excl); a.z = max(a.z, excl); a.w = max(a.w, excl);
    b.x = max(b.x, excl); b.y = max(b.y, excl); b.z = max(b.z, excl); b.w = max(b.w, excl);
    reinterpret_cast<int4*>(s_row)[2 * tid] = a;
    reinterpret_cast<int4*>(s_row)[2 * tid + 1] = b;
  } else {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = q * 256 + tid;
      if (t < tn) s_row[t] = int32_t(row_of(off_p, r0, r1, e0 + t) - r0);
    }
  }
  __syncthreads();
  int32_t v[PER], rem[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = q * 256 + tid;
    v[q] = -1;
    if (t < tn) {
      const int ri = s_row[t];
      const int64_t c = staged ? s_c[ri] : off_p[r0 + ri] - e0;
      const int64_t c1 = staged ? s_c[ri + 1] : off_p[r0 + ri + 1] - e0;
      const int64_t base = staged ? s_b[ri] : und_off[order[r0 + ri]];
      const int64_t k = t - c;
      v[q] = buf[base + k];
      rem[q] = int32_t(c1 - t - 1);
      adj_p[e0 + t] = v[q];
    }
  }
  unsigned long long slot[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) slot[q] = v[q] >= 0 ? atomicAdd(&cur64[v[q]], 1ull) : 0ull;
#pragma unroll
  for (int q = 0; q < PER; ++q)
    if (v[q] >= 0) nm[slot[q]] = make_int2(int(e0 + q * 256 + tid + 1), rem[q]);
}

// ---- work lists --------------------------------------------------------------
// kind 0: warp bitmap tasks (n-1-v <= TC_BM_BITS), 3: warp split tasks
// (d+(v) <= TC_SPLIT_MAX), 1: warp hash tasks, 2: CTA hash tasks. A task is (v, chunk of N-(v)); it needs d+(v), d-(v) >= 1.
__global__ void __launch_bounds__(256) tc_task_count_kernel(const int64_t* __restrict__ off_p,
                                                            const int64_t* __restrict__ off_m,
                                                            int64_t n, int part, int nparts,
                                                            int64_t bm_bits,
                                                            int64_t* __restrict__ c0,
                                                            int64_t* __restrict__ c1,
                                                            int64_t* __restrict__ c2,
                                                            int64_t* __restrict__ c3) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t dp = off_p[v + 1] - off_p[v];
  const int64_t dm = off_m[v + 1] - off_m[v];
  // a part owns whole N-(v) lists (v = part mod nparts): the order inside a
  // list is scheduling dependent, so chunks of one list must stay together
  const bool live = dp >= 1 && dm >= 1 && v % nparts == part;
  const bool bm = n - 1 - v <= bm_bits;
  c0[v] = (live && bm) ? (dm + TC_CHUNK - 1) / TC_CHUNK : 0;
  c1[v] = (live && !bm && dp > TC_SPLIT_MAX && dp <= TC_WARP_MAX)
              ? (dm + TC_CHUNK - 1) / TC_CHUNK : 0;
  c3[v] = (live && !bm && dp <= TC_SPLIT_MAX) ? (dm + TC_CHUNK - 1) / TC_CHUNK : 0;
  c2[v] = (live && !bm && dp > TC_WARP_MAX) ? (dm + TC_CHUNK_CTA - 1) / TC_CHUNK_CTA : 0;
}

// Diagnostics (GT_TC_STATS=1): per task kind, the number of v, sum d+(v)
// (table build work) and the probes (suffix elements) of its N-(v) list.
__global__ void __launch_bounds__(256) tc_stats_kernel(const int64_t* __restrict__ off_p,
                                                       const int64_t* __restrict__ off_m,
                                                       const int2* __restrict__ nm, int64_t n,
                                                       int64_t bm_bits,
                                                       unsigned long long* __restrict__ out) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t dp = off_p[v + 1] - off_p[v];
  const int64_t om = off_m[v], dm = off_m[v + 1] - om;
  if (dp < 1 || dm < 1) return;
  const int kind = n - 1 - v <= bm_bits ? 0 : dp <= TC_SPLIT_MAX ? 3 : dp <= TC_WARP_MAX ? 1 : 2;
  unsigned long long pr = 0;
  for (int64_t j = 0; j < dm; ++j) pr += unsigned(nm[om + j].y);
  if (kind == 2) {  // CTA tasks by distance from the top: <= 2^17, 2^18, 2^19, 2^20
    const int64_t dist = n - 1 - v;
    for (int b = 0; b < 4; ++b)
      if (dist <= (int64_t(1) << (17 + b))) atomicAdd(&out[16 + b], pr);
  }
  atomicAdd(&out[kind * 4 + 0], 1ull);
  atomicAdd(&out[kind * 4 + 1], (unsigned long long)dp);
  atomicAdd(&out[kind * 4 + 2], pr);
  atomicAdd(&out[kind * 4 + 3], (unsigned long long)dm);
}

// Bitmap tasks reordered by the adj_p position of their first arc (the rank
// of its u), so that the warps running at the same time walk N+(u) suffixes
// of nearby u: the suffix data of the tasks in flight stays in L2. In v order
// (tasks of one v adjacent, so a warp reuses its table) every task walks ~256
// scattered N+(u) lists and ncu at C4 showed 656 GB of DRAM reads at a 26%
// L2 hit rate in the count kernel; in u order the table is rebuilt per task
// (clearing <= 8 KB and setting d+(v) bits), small against ~10^5 probes.
__global__ void __launch_bounds__(256) tc_task_keys_kernel(const int2* __restrict__ tasks,
                                                           int64_t nt, int chunk,
                                                           const int64_t* __restrict__ off_m,
                                                           const int2* __restrict__ nm,
                                                           uint64_t* __restrict__ keys) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const int2 t = tasks[i];
  const int32_t a = nm[off_m[t.x] + int64_t(t.y) * chunk].x;
  keys[i] = (uint64_t(uint32_t(a)) << 32) | uint64_t(i);
}

__global__ void __launch_bounds__(256) tc_task_permute_kernel(const uint64_t* __restrict__ keys,
                                                              int64_t nt,
                                                              const int2* __restrict__ tasks,
                                                              int2* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nt) out[i] = tasks[keys[i] & 0xffffffffull];
}

__global__ void __launch_bounds__(256) tc_task_fill_kernel(const int64_t* __restrict__ toff,
                                                           int64_t n, int2* __restrict__ tasks) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t a = toff[v], b = toff[v + 1];
  for (int64_t i = a; i < b; ++i) tasks[i] = make_int2(int(v), int(i - a));
}

// max d+ (out[0]) and the probe count sum_u d+(u)(d+(u)-1)/2 (out[1]): every
// suffix element the count kernels read, i.e. their algorithmic traffic.
__global__ void __launch_bounds__(256) max_dplus_kernel(const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ adj, int64_t n,
                                                        int64_t win_lo,
                                                        unsigned long long* __restrict__ out,
                                                        unsigned long long* __restrict__ out_bm) {
  unsigned long long mx = 0, pr = 0, pb = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += stride) {
    const int64_t o = off[u];
    const unsigned long long d = (unsigned long long)(off[u + 1] - o);
    mx = max(mx, d);
    pr += d * (d - (d > 0)) / 2;
    // t = elements of N+(u) at or above win_lo (its sorted tail): arcs (u,v)
    // with v there are bitmap-task arcs and probe t(t-1)/2 window elements
    int64_t lo = 0, hi = int64_t(d);
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (adj[o + mid] < win_lo) lo = mid + 1;
      else hi = mid;
    }
    const unsigned long long t = d - (unsigned long long)lo;
    pb += t * (t - (t > 0)) / 2;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    pr += __shfl_xor_sync(0xffffffffu, pr, o);
    pb += __shfl_xor_sync(0xffffffffu, pb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx) atomicMax(&out[0], mx);
    if (pr) atomicAdd(&out[1], pr);
    if (pb) atomicAdd(out_bm, pb);
  }
}

// ---- membership structures of N+(v) ------------------------------------------

__device__ __forceinline__ uint32_t tc_hash(int32_t x, int log_slots) {
  return (uint32_t(x) * 0x9E3779B1u) >> (32 - log_slots);
}

// Probes: kChecked = the walk pads idle lanes with TC_EMPTY and tests for it
// before probing; an unchecked probe names an element (pad) whose lookup is
// always false, so the walk probes every lane without the test.
struct HashProbe {
  static constexpr bool kChecked = true;
  static constexpr int32_t pad = TC_EMPTY;
  int32_t* tab;
  uint32_t mask;
  int log_slots;
  __device__ __forceinline__ void insert(int32_t x) const {
    uint32_t h = tc_hash(x, log_slots);
    while (atomicCAS(&tab[h], TC_EMPTY, x) != TC_EMPTY) h = (h + 1) & mask;
  }
  __device__ __forceinline__ bool operator()(int32_t x) const {
    uint32_t h = tc_hash(x, log_slots);
    while (true) {
      const int32_t y = tab[h];
      if (y == x) return true;
      if (y == TC_EMPTY) return false;
      h = (h + 1) & mask;
    }
  }
};

// Bit w of a bitmap indexed by the element itself: the table of a task holds
// N+(v) at ABSOLUTE window positions (w - window base, the base a multiple of
// 32 folded into sbase), so a probe is shift, address, LDS, shift, mask with
// no per-task subtraction, and `pad` — an element at or below v, never a
// member, its word cleared — lets idle lanes probe without a test (ncu of the
// C4 warp count: 13.6 instructions per element, 9 of them the probe). The
// bitmap is addressed through its 32-bit shared-window address so every
// probe is one LDS (a generic pointer would cost the window translation).
struct BitmapProbe {
  static constexpr bool kChecked = false;
  uint32_t sbase;  // shared-space address of the word of element 0 (may lie below the table)
  int32_t pad;
  __device__ __forceinline__ bool operator()(int32_t w) const {
    const uint32_t i = uint32_t(w);
    uint32_t x;
    uint32_t a;  // word index * 4 + base as one multiply-add (the compiler's shift, mask,
                 // add costs an instruction more: C4 warp count 292 -> 283 ms)
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(i >> 5), "r"(sbase));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a) : "memory");
    return (x >> (i & 31)) & 1u;
  }
};

// Split table for v below the bitmap window: the members of N+(v) among the
// top TC_SPLIT_TOP ranks in a bitmap (where R-MAT sends nearly every probe),
// the others in a small open-addressing hash (load <= 1/4).
struct SplitProbe {
  static constexpr bool kChecked = true;
  static constexpr int32_t pad = TC_EMPTY;
  uint32_t sbm;   // shared address of the bitmap words
  uint32_t stab;  // shared address of the hash slots
  int32_t top;    // n - TC_SPLIT_TOP
  __device__ __forceinline__ bool operator()(int32_t w) const {
    uint32_t x;
    if (w >= top) {
      const uint32_t i = uint32_t(w - top);
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(sbm + ((i >> 5) << 2)) : "memory");
      return (x >> (i & 31)) & 1u;
    }
    constexpr int L = 10;  // log2(TC_SPLIT_SLOTS)
    uint32_t h = tc_hash(w, L);
    while (true) {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(stab + (h << 2)) : "memory");
      if (int32_t(x) == w) return true;
      if (int32_t(x) == TC_EMPTY) return false;
      h = (h + 1) & (TC_SPLIT_SLOTS - 1);
    }
  }
};

__device__ __forceinline__ int tc_log_slots(int64_t d, int cap_log) {
  int l = 5;  // >= 32 slots, >= 4 slots per element (load <= 1/4)
  while (l < cap_log && (int64_t(1) << l) < 4 * d) ++l;
  return l;
}

// One warp probes up to 32 suffixes (lane = arc (u,v): positions [s, s+len)
// of adj, all w > v) against N+(v).
//  * long suffixes (>= TC_LONG) are walked by the whole warp one arc at a
//    time, TC_UNROLL coalesced loads in flight, the next arc prefetched;
//  * the short rest is flattened: position t of the concatenation of the
//    short suffixes belongs to the lane whose suffix starts last at or before
//    t (position -> lane map in shared memory), TC_WIN windows of 32
//    positions resolved per step, so lanes stay busy and reads coalesced.
// The cost is issued instructions per probe, i.e. lane occupancy: a warp walk
// of a suffix shorter than 32*TC_UNROLL idles lanes, the flattened walk pays
// the owner lookup. The three constants were swept on C2
// (scripts/sweep_tc_consts.sh): 16/4/8 -> 64/7/4 took the count 11.3 -> 8.8 ms.
#ifndef GT_TC_WIN
#define GT_TC_WIN 7
#endif
#ifndef GT_TC_LONG
#define GT_TC_LONG 64
#endif
#ifndef GT_TC_UNROLL
#define GT_TC_UNROLL 4
#endif
constexpr int TC_WIN = GT_TC_WIN;
constexpr int TC_LONG = GT_TC_LONG;
constexpr int TC_UNROLL = GT_TC_UNROLL;

// The part of a long suffix past its first 32*TC_UNROLL elements, walked by
// the warp with 16-byte vector loads (4 ranks per load): at C4 most probes
// land here (ncu: the scalar walk's load, bounds test and select cost as many
// instructions as the probe itself). Unaligned head and short rest by single
// loads. Used by the CTA count kernel only (see tc_wedges32).
template <typename Probe, typename T>
__device__ __forceinline__ uint32_t tc_long_tail(const T* __restrict__ p, int len,
                                                 const Probe& probe) {
  constexpr int VE = 16 / int(sizeof(T));
  const int lane = threadIdx.x & 31;
  uint32_t cnt = 0;
  const int mis = int((reinterpret_cast<uintptr_t>(p) & 15u) / sizeof(T));
  const int head = min(len, mis ? VE - mis : 0);
  if (lane < head) cnt += probe(int32_t(__ldg(p + lane))) ? 1u : 0u;
  p += head;
  len -= head;
  const int nv = len / VE;
  const uint4* pv = reinterpret_cast<const uint4*>(p);
  auto probe_vec = [&](const uint4 q) {
    const uint32_t x[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (sizeof(T) == 2) {
        cnt += probe(int32_t(x[h] & 0xffffu)) ? 1u : 0u;
        cnt += probe(int32_t(x[h] >> 16)) ? 1u : 0u;
      } else {
        cnt += probe(int32_t(x[h])) ? 1u : 0u;
      }
    }
  };
  int j = lane;
  for (; j + 32 < nv; j += 64) {  // two loads in flight per lane
    const uint4 a = __ldg(pv + j), b = __ldg(pv + j + 32);
    probe_vec(a);
    probe_vec(b);
  }
  if (j < nv) probe_vec(__ldg(pv + j));
  const int rest = len - nv * VE;
  if (lane < rest) cnt += probe(int32_t(__ldg(p + nv * VE + lane))) ? 1u : 0u;
  return cnt;
}

template <typename Probe, typename T = int32_t, bool VEC = false>
__device__ __forceinline__ uint32_t tc_wedges32(const T* __restrict__ adj, int2 suffix,
                                                const Probe& probe,
                                                uint8_t* s_start /* [32 * TC_WIN] */) {
  const int lane = threadIdx.x & 31;
  uint32_t cnt = 0;
  const int32_t PAD = probe.pad;  // what idle lanes hold (TC_EMPTY for the checked probes)
  auto hit = [&](int32_t w) -> uint32_t {
    if (std::remove_cv_t<std::remove_reference_t<Probe>>::kChecked)
      return (w != TC_EMPTY && probe(w)) ? 1u : 0u;
    return probe(w) ? 1u : 0u;
  };
  // ---- long suffixes: warp per arc; the first 32*TC_UNROLL positions of the
  // NEXT arc are loaded before the current one is probed (software pipeline)
  unsigned longs = __ballot_sync(0xffffffffu, suffix.y >= TC_LONG);
  auto fetch = [&](int i, const T*& b, int& l, int32_t (&w)[TC_UNROLL]) {
    b = adj + __shfl_sync(0xffffffffu, suffix.x, i);
    l = __shfl_sync(0xffffffffu, suffix.y, i);
#pragma unroll
    for (int q = 0; q < TC_UNROLL; ++q) {
      const int k = 32 * q + lane;
      w[q] = k < l ? int32_t(__ldg(b + k)) : PAD;
    }
  };
  if (longs) {
    int32_t wa[TC_UNROLL], wb[TC_UNROLL];
    const T *ba, *bb = adj;
    int la, lb = 0;
    int i = __ffs(longs) - 1;
    longs &= longs - 1;
    fetch(i, ba, la, wa);
    while (i >= 0) {
      const int j = longs ? __ffs(longs) - 1 : -1;
      if (j >= 0) {
        longs &= longs - 1;
        fetch(j, bb, lb, wb);
      }
#pragma unroll
      for (int q = 0; q < TC_UNROLL; ++q) cnt += hit(wa[q]);
      if (VEC) {  // vector walk: C4 CTA count 193 -> 180 ms; slower in the warp kernel
        // (16-bit window ranks: 357 vs 307 ms; split / hash tasks: +20 ms)
        if (la > 32 * TC_UNROLL) cnt += tc_long_tail(ba + 32 * TC_UNROLL, la - 32 * TC_UNROLL, probe);
      } else {
        int k0 = 32 * TC_UNROLL;
        // (whole blocks without the per-element bounds test measured slower twice:
        // 307 -> 394 ms with the checked probes, 292 -> 306 ms with these)
        for (; k0 < la; k0 += 32 * TC_UNROLL) {
          int32_t w[TC_UNROLL];
#pragma unroll
          for (int q = 0; q < TC_UNROLL; ++q) {
            const int k = k0 + 32 * q + lane;
            w[q] = k < la ? int32_t(__ldg(ba + k)) : PAD;
          }
#pragma unroll
          for (int q = 0; q < TC_UNROLL; ++q) cnt += hit(w[q]);
        }
      }
      i = j;
      ba = bb;
      la = lb;
#pragma unroll
      for (int q = 0; q < TC_UNROLL; ++q) wa[q] = wb[q];
    }
  }
  // ---- short suffixes: flattened across the lanes --------------------------
  const int64_t ou = suffix.x;
  const int du = suffix.y < TC_LONG ? suffix.y : 0;
  const int incl = warp_incl_scan(du);
  const int tot = __shfl_sync(0xffffffffu, incl, 31);
  const int excl = incl - du;
  int carry = 0;
  for (int t0 = 0; t0 < tot; t0 += 32 * TC_WIN) {
    // suffixes starting in this step: position -> lane map + per-window masks
    const int rel = excl - t0;
    const bool st = du > 0 && rel >= 0 && rel < 32 * TC_WIN;
    if (st) s_start[rel] = uint8_t(lane);
    unsigned starts[TC_WIN];
#pragma unroll
    for (int q = 0; q < TC_WIN; ++q)
      starts[q] = __reduce_or_sync(0xffffffffu, (st && (rel >> 5) == q) ? 1u << (rel & 31) : 0u);
    __syncwarp();
    int32_t w[TC_WIN];
#pragma unroll
    for (int q = 0; q < TC_WIN; ++q) {
      w[q] = PAD;
      if (t0 + 32 * q >= tot) continue;  // warp-uniform: nothing left
      const unsigned mine = starts[q] & (0xffffffffu >> (31 - lane));
      const int owner = mine ? int(s_start[32 * q + 31 - __clz(mine)]) : carry;
      carry = __shfl_sync(0xffffffffu, owner, 31);
      const int64_t o = __shfl_sync(0xffffffffu, ou, owner);
      const int ex = __shfl_sync(0xffffffffu, excl, owner);
      const int t = t0 + 32 * q + lane;
      if (t < tot) w[q] = int32_t(__ldg(adj + o + (t - ex)));
    }
#pragma unroll
    for (int q = 0; q < TC_WIN; ++q) cnt += hit(w[q]);
    __syncwarp();
  }
  return cnt;
}

// Bitmap tasks only read suffix elements w > v inside the window
// [base16, n) (base16 = n - window), so they read them from adj16, a copy of
// adj_p holding w - base16 in 16 bits: the same load count, half the bytes
// and half the L2 footprint of the suffix data.
__global__ void __launch_bounds__(256) adj16_kernel(const int32_t* __restrict__ adj, int64_t m,
                                                    int32_t base16, uint16_t* __restrict__ adj16) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; a < m; a += stride) {
    const int32_t w = adj[a];
    adj16[a] = w >= base16 ? uint16_t(w - base16) : uint16_t(0);
  }
}

// Warp per task (v, chunk of N-(v)), dynamic task grabbing. Each warp owns
// an 8 KB shared-memory region that holds N+(v) either as a BITMAP of the
// window (v, n) (kind 0: n-1-v <= TC_BM_BITS) or as a hash table (kind 1:
// d+(v) <= TC_WARP_MAX, load <= 1/4). Tasks of the same v are adjacent in
// the list, so a warp that draws the next chunk of its v reuses the table.
// (GT_TC_MINB: min-blocks hint of the two count kernels, for register sweeps)
#ifdef GT_TC_MINB
#define GT_TC_LB __launch_bounds__(256, GT_TC_MINB)
#else
#define GT_TC_LB __launch_bounds__(256)
#endif
__global__ void GT_TC_LB tc_count_warp_kernel(
    const int64_t* __restrict__ off_p, const int32_t* __restrict__ adj_p,
    const int64_t* __restrict__ off_m, const int2* __restrict__ nm,
    const int2* __restrict__ tasks, int64_t n_bitmap_tasks, int64_t n_split_end, int64_t n_tasks,
    int64_t n, int split_top, int part, int nparts, unsigned int* __restrict__ next_task,
    unsigned long long* __restrict__ total, const uint16_t* __restrict__ adj16, int32_t base16) {
  extern __shared__ int32_t s_tab[];  // [8][TC_SLOTS]
  __shared__ uint8_t s_start[8][32 * TC_WIN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* tab = s_tab + warp * TC_SLOTS;
  uint32_t* bm = reinterpret_cast<uint32_t*>(tab);
  int cur_v = -1;
  HashProbe hprobe{tab, 31u, 5};
  unsigned long long acc = 0;
  while (true) {
    unsigned int k = 0;
    if (lane == 0) k = atomicAdd(next_task, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    const int64_t it = int64_t(k);
    if (it >= n_tasks) break;
    const int2 task = tasks[it];
    const int v = task.x;
    const bool use_bm = it < n_bitmap_tasks;
    const bool use_split = !use_bm && it < n_split_end;
    if (v != cur_v) {
      const int64_t ov = off_p[v];
      const int dv = int(off_p[v + 1] - ov);
      if (use_split) {
        const int32_t top = int32_t(n - split_top);
        uint32_t* sbm = reinterpret_cast<uint32_t*>(tab);
        int32_t* stab = tab + TC_SPLIT_TOP / 32;
        for (int i = lane; i < TC_SPLIT_TOP / 32; i += 32) sbm[i] = 0u;
        for (int i = lane; i < TC_SPLIT_SLOTS; i += 32) stab[i] = TC_EMPTY;
        __syncwarp();
        const HashProbe low{stab, TC_SPLIT_SLOTS - 1u, 10};
        for (int i = lane; i < dv; i += 32) {
          const int32_t x = adj_p[ov + i];
          if (x >= top) atomicOr(&sbm[uint32_t(x - top) >> 5], 1u << (uint32_t(x - top) & 31));
          else low.insert(x);
        }
      } else if (use_bm) {
        // absolute window positions w - base16 (what adj16 holds): members lie
        // in [v + 1 - base16, n - base16), all >= 1; position 0 is the pad
        const int w0 = (v + 1 - base16) >> 5, w1 = int((n - base16 + 31) >> 5);
        if (lane == 0) bm[0] = 0u;
        for (int i = w0 + lane; i < w1; i += 32) bm[i] = 0u;
        __syncwarp();
        for (int i = lane; i < dv; i += 32) {
          const uint32_t b = uint32_t(adj_p[ov + i] - base16);
          atomicOr(&bm[b >> 5], 1u << (b & 31));
        }
      } else {
        hprobe.log_slots = tc_log_slots(dv, 11);
        hprobe.mask = (1u << hprobe.log_slots) - 1u;
        for (int i = lane; i <= int(hprobe.mask); i += 32) tab[i] = TC_EMPTY;
        __syncwarp();
        for (int i = lane; i < dv; i += 32) hprobe.insert(adj_p[ov + i]);
      }
      __syncwarp();
      cur_v = v;
    }
    const int64_t om = off_m[v];
    const int dm = int(off_m[v + 1] - om);
    const int end = min(dm, (task.y + 1) * TC_CHUNK);
    uint32_t cnt = 0;
    if (use_split) {
      const uint32_t sb = uint32_t(__cvta_generic_to_shared(tab));
      const SplitProbe probe{sb, sb + TC_SPLIT_TOP / 8, int32_t(n - split_top)};
      for (int jb = task.y * TC_CHUNK; jb < end; jb += 32) {
        const int jj = jb + lane;
        const int2 sfx = jj < end ? nm[om + jj] : make_int2(0, 0);
        cnt += tc_wedges32(adj_p, sfx, probe, s_start[warp]);
      }
    } else if (use_bm) {
      const BitmapProbe probe{uint32_t(__cvta_generic_to_shared(bm)), 0};
      for (int jb = task.y * TC_CHUNK; jb < end; jb += 32) {
        const int jj = jb + lane;
        const int2 sfx = jj < end ? nm[om + jj] : make_int2(0, 0);
        cnt += tc_wedges32(adj16, sfx, probe, s_start[warp]);
      }
    } else {
      for (int jb = task.y * TC_CHUNK; jb < end; jb += 32) {
        const int jj = jb + lane;
        const int2 sfx = jj < end ? nm[om + jj] : make_int2(0, 0);
        cnt += tc_wedges32(adj_p, sfx, hprobe, s_start[warp]);
      }
    }
    acc += cnt;
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
}

// Tasks with large d+(v) below the bitmap window, CTA per (v, chunk). When
// the window (v, n) fits the shared table as a bitmap (2^19 ranks), N+(v) is
// a CTA bitmap; otherwise it goes to a hash table as sparse as shared memory
// allows (TC_CTA_SLOTS slots,
// probed with shared-window loads: nearly every miss resolves in one probe),
// or, when 2 d+(v) exceeds that, to a per-CTA global table of gtab_slots.
#ifndef GT_TC_CTA_LOG
#define GT_TC_CTA_LOG 13
#endif
#ifndef GT_TC_CTA_MINB
#define GT_TC_CTA_MINB 4
#endif
// 32 KB tables (bitmap window 2^18 ranks: 89 % of the CTA probes at C4; the
// rest hashed), 4 CTAs per SM at 64 registers: C4 178 -> 161 ms against
// 64 KB tables at 3 CTAs per SM (the kernel is latency-bound on its suffix
// reads, so residency pays more than the wider bitmap window)
constexpr int TC_CTA_SLOTS = 1 << GT_TC_CTA_LOG;
#ifndef GT_TC_CTA_GROUP
#define GT_TC_CTA_GROUP 4
#endif
constexpr int TC_CTA_GROUP = GT_TC_CTA_GROUP;  // arcs a warp draws at a time (<= 32)

struct SmemHashProbe {
  static constexpr bool kChecked = true;
  static constexpr int32_t pad = TC_EMPTY;
  uint32_t stab;  // shared address of the slots
  uint32_t mask;
  int log_slots;
  __device__ __forceinline__ bool operator()(int32_t w) const {
    uint32_t h = tc_hash(w, log_slots);
    while (true) {
      uint32_t x;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(stab + (h << 2)) : "memory");
      if (int32_t(x) == w) return true;
      if (int32_t(x) == TC_EMPTY) return false;
      h = (h + 1) & mask;
    }
  }
};

// with (256) alone ptxas settles on 48 registers and spills; the min-blocks
// hint sizes the register budget to the residency the table allows
__global__ void __launch_bounds__(256, GT_TC_CTA_MINB) tc_count_cta_kernel(
    const int64_t* __restrict__ off_p, const int32_t* __restrict__ adj_p,
    const int64_t* __restrict__ off_m, const int2* __restrict__ nm,
    const int2* __restrict__ tasks, int64_t n_tasks, int smem_log, int32_t* __restrict__ gtab,
    int gtab_log, unsigned long long* __restrict__ total, int64_t n, int64_t bm_bits,
    int32_t win_base) {
  extern __shared__ __align__(16) int32_t s_cta[];
  __shared__ uint8_t s_start[8][32 * TC_WIN];
  __shared__ unsigned long long s_red[8];
  __shared__ int s_next;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* mytab = gtab ? gtab + (int64_t(blockIdx.x) << gtab_log) : nullptr;
  unsigned long long acc = 0;
  // the warps draw groups of TC_CTA_GROUP arcs of the chunk from a shared
  // counter, so the CTA's end-of-task barrier waits for at most one group, not
  // a fixed share (ncu at C4 with 32-arc groups: 31 % of the stall samples at
  // that barrier — a group's work varies with its suffix lengths)
  auto walk = [&](int64_t om, int begin, int end, const auto& probe) {
    uint32_t cnt = 0;
    while (true) {
      int g = 0;
      if (lane == 0) g = atomicAdd(&s_next, 1);
      const int jb = begin + TC_CTA_GROUP * __shfl_sync(0xffffffffu, g, 0);
      if (jb >= end) break;
      const int jj = jb + lane;
      const int2 sfx = (lane < TC_CTA_GROUP && jj < end) ? nm[om + jj] : make_int2(0, 0);
      cnt += tc_wedges32<decltype(probe), int32_t, true>(adj_p, sfx, probe, s_start[warp]);
    }
    acc += cnt;
  };
  for (int64_t it = blockIdx.x; it < n_tasks; it += gridDim.x) {
    const int2 task = tasks[it];
    const int v = task.x;
    const int64_t ov = off_p[v];
    const int dv = int(off_p[v + 1] - ov);
    const int64_t om = off_m[v];
    const int dm = int(off_m[v + 1] - om);
    const int begin = task.y * TC_CHUNK_CTA;
    const int end = min(dm, begin + TC_CHUNK_CTA);
    __syncthreads();  // previous task done with the table and the group counter
    if (threadIdx.x == 0) s_next = 0;
    if (n - 1 - v <= bm_bits) {
      // the whole window (v, n) fits a CTA bitmap (the shared table as bits):
      // one LDS per probe instead of a hash walk (99.6% of these probes at C4)
      // absolute positions w - win_base (win_base a multiple of 32, folded
      // into the probe's base address); win_base itself is the pad: below
      // every member, its word cleared
      uint32_t* bm = reinterpret_cast<uint32_t*>(s_cta);
      const int w0 = (v + 1 - win_base) >> 5, w1 = int((n - win_base + 31) >> 5);
      if (threadIdx.x == 0) bm[0] = 0u;
      for (int i = w0 + threadIdx.x; i < w1; i += 256) bm[i] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < dv; i += 256) {
        const uint32_t b = uint32_t(adj_p[ov + i] - win_base);
        atomicOr(&bm[b >> 5], 1u << (b & 31));
      }
      __syncthreads();
      walk(om, begin, end,
           BitmapProbe{uint32_t(__cvta_generic_to_shared(bm)) - (uint32_t(win_base) >> 5) * 4u,
                       win_base});
      continue;
    }
    const bool in_smem = 2 * int64_t(dv) <= (int64_t(1) << smem_log);
    const int log_slots = in_smem ? smem_log : gtab_log;
    int32_t* tab = in_smem ? s_cta : mytab;
    const int slots = 1 << log_slots;
    for (int i = threadIdx.x; i < slots; i += 256) tab[i] = TC_EMPTY;
    __syncthreads();
    const HashProbe ins{tab, uint32_t(slots - 1), log_slots};
    for (int i = threadIdx.x; i < dv; i += 256) ins.insert(adj_p[ov + i]);
    __syncthreads();
    if (in_smem)
      walk(om, begin, end,
           SmemHashProbe{uint32_t(__cvta_generic_to_shared(tab)), uint32_t(slots - 1), log_slots});
    else
      walk(om, begin, end, ins);
  }
  acc = block_sum_256(acc, s_red);
  if (threadIdx.x == 0 && acc) atomicAdd(total, acc);
}

// ---- sharded orientation (distributed.triangle_count) ------------------------
// A rank holds the undirected rows of an id range [row_lo, row_lo + rows)
// (local offsets, global neighbour ids). Warp per row; outputs compacted in
// row order with ballots after a count pass and a scan.

// 2 x (neighbours other than the row itself): both directions of every edge.
__global__ void __launch_bounds__(256) tc_und_count_kernel(const int64_t* __restrict__ off,
                                                           const int32_t* __restrict__ adj,
                                                           int64_t rows, int64_t row_lo,
                                                           int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); r < rows; r += nw) {
    const int32_t u = int32_t(row_lo + r);
    int c = 0;
    for (int64_t j = off[r] + lane; j < off[r + 1]; j += 32) c += adj[j] != u;
    c = warp_sum(c);
    if (lane == 0) cnt[r] = 2 * int64_t(c);
  }
}

__global__ void __launch_bounds__(256) tc_und_write_kernel(const int64_t* __restrict__ off,
                                                           const int32_t* __restrict__ adj,
                                                           int64_t rows, int64_t row_lo, int kbits,
                                                           const int64_t* __restrict__ pos,
                                                           uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); r < rows; r += nw) {
    const uint64_t u = uint64_t(row_lo + r);
    int64_t o = pos[r];
    for (int64_t j0 = off[r]; j0 < off[r + 1]; j0 += 32) {
      const int64_t j = j0 + lane;
      const uint64_t x = j < off[r + 1] ? uint64_t(uint32_t(adj[j])) : u;
      const bool keep = x != u;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int64_t k = o + 2 * __popc(bal & lt);
        keys[k] = (u << kbits) | x;
        keys[k + 1] = (x << kbits) | u;
      }
      o += 2 * __popc(bal);
    }
  }
}

// Arcs to higher-ranked neighbours: (rank(u) << kbits | rank(v)).
__global__ void __launch_bounds__(256) tc_orient_count_kernel(const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ adj,
                                                              int64_t rows, int64_t row_lo,
                                                              const int32_t* __restrict__ rank,
                                                              int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); r < rows; r += nw) {
    const int32_t ru = rank[row_lo + r];
    int c = 0;
    for (int64_t j = off[r] + lane; j < off[r + 1]; j += 32) c += rank[adj[j]] > ru;
    c = warp_sum(c);
    if (lane == 0) cnt[r] = c;
  }
}

__global__ void __launch_bounds__(256) tc_orient_write_kernel(const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ adj,
                                                              int64_t rows, int64_t row_lo,
                                                              const int32_t* __restrict__ rank,
                                                              int kbits,
                                                              const int64_t* __restrict__ pos,
                                                              uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); r < rows; r += nw) {
    const int32_t ru = rank[row_lo + r];
    int64_t o = pos[r];
    for (int64_t j0 = off[r]; j0 < off[r + 1]; j0 += 32) {
      const int64_t j = j0 + lane;
      const int32_t rv = j < off[r + 1] ? rank[adj[j]] : -1;
      const bool keep = rv > ru;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (keep) keys[o + __popc(bal & lt)] = (uint64_t(uint32_t(ru)) << kbits) | uint64_t(uint32_t(rv));
      o += __popc(bal);
    }
  }
}

__global__ void __launch_bounds__(256) deg64_to_32_kernel(const int64_t* __restrict__ d, int64_t n,
                                                          int32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = int32_t(d[i]);
}

// N-(v) sizes of the middle vertices this part owns (v = part mod nparts).
__global__ void __launch_bounds__(256) tc_owned_indeg_kernel(const int32_t* __restrict__ adj_p,
                                                             int64_t m, int part, int nparts,
                                                             unsigned long long* __restrict__ dm) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; a < m; a += stride) {
    const int32_t v = adj_p[a];
    if (v % nparts == part) atomicAdd(&dm[v], 1ull);
  }
}

// Warp per rank-row u: every arc (u, v) with an owned v filed under N-(v) as
// (a+1, remaining length of N+(u)) — place_rows_kernel without the move.
__global__ void __launch_bounds__(256) tc_file_owned_kernel(const int64_t* __restrict__ off_p,
                                                            const int32_t* __restrict__ adj_p,
                                                            int64_t n, int part, int nparts,
                                                            const int64_t* __restrict__ off_m,
                                                            unsigned int* __restrict__ cur,
                                                            int2* __restrict__ nm) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t u = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); u < n; u += nw) {
    const int64_t a0 = off_p[u];
    const int cnt = int(off_p[u + 1] - a0);
    for (int t = lane; t < cnt; t += 32) {
      const int32_t v = adj_p[a0 + t];
      if (v % nparts != part) continue;
      const unsigned slot = atomicAdd(&cur[v], 1u);
      nm[off_m[v] + slot] = make_int2(int(a0 + t + 1), cnt - t - 1);
    }
  }
}

}  // namespace gtd

namespace gt {

static int grid_cap(int64_t blocks) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, 8LL * ctx().sm_count)));
}

uint32_t* undirected_degrees(const gt_graph* g, int64_t* cat, int32_t* deg, const char* phase) {
  const int64_t n = g->n, slots = 2 * g->e;
  cudaStream_t s = ctx().stream;
  const int64_t tiles = ceil_div64(slots, gtd::TC_CAND_TILE);
  if (tiles >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "undirected degrees: too many slot tiles");
  GT_CUDA(cudaMemsetAsync(deg, 0, size_t(n) * 4, s));
  int64_t* tile_row = ws_n<int64_t>(WS_TMP1, size_t(tiles) + 1);
  uint32_t* keep_bits = ws_n<uint32_t>(WS_RANKMAP, size_t(tiles) * (gtd::TC_CAND_TILE / 32));
  Phase ph(phase, 8.0 * (n + 1) * 3 + 4.0 * slots + 4.0 * n + slots / 8.0);
  GT_LAUNCH(gtd::cat_off_kernel, ceil_div(n + 1, 256), 256, 0, g->out_off, g->in_off, n, cat);
  if (tiles == 0) return keep_bits;
  GT_LAUNCH(gtd::cand_tile_rows_kernel, ceil_div(tiles + 1, 256), 256, 0, cat, n, slots, tiles,
            tile_row);
  GT_LAUNCH(gtd::cand_degree_kernel, static_cast<int>(tiles), 256, 0, cat, tile_row, g->out_off,
            g->out_adj, g->in_adj, n, slots, deg, keep_bits);
  return keep_bits;
}

// Degree-ordered orientation in rank space (device scratch, valid until the
// next library call that uses the workspace).
struct Oriented {
  int64_t n = 0, m = 0;
  int kbits = 1;
  int32_t* deg = nullptr;    // [n] by id
  int32_t* rank = nullptr;   // [n] id -> rank
  int64_t* off_p = nullptr;  // [n+1] by rank
  int32_t* adj_p = nullptr;  // [m] ranks, ascending per row
  int64_t* off_m = nullptr;  // [n+1] by rank
  int2* nm = nullptr;        // [m] N-(v) entries: (first index after v in N+(u), remaining)
};

static Oriented orient(const gt_graph* g) {
  const int64_t n = g->n, e = g->e;
  cudaStream_t s = ctx().stream;
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  const int64_t slots = 2 * e;
  Oriented o;
  o.n = n;
  o.kbits = bits_for(n);
  // scratch (WS_TMP3): cat | und_off | off_p | off_m (n+1 each) | deg | rank | dplus | cur
  const size_t need = size_t(n + 1) * 8 * 4 + size_t(n) * 20 + 4 * 4096 * 2 + 256;
  char* p = static_cast<char*>(ws_get(WS_TMP3, need));
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  int64_t* cat = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  int64_t* und_off = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  o.off_p = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  o.off_m = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  o.deg = reinterpret_cast<int32_t*>(carve(size_t(n) * 4));
  o.rank = reinterpret_cast<int32_t*>(carve(size_t(n) * 4));
  int32_t* dplus = reinterpret_cast<int32_t*>(carve(size_t(n) * 4));
  unsigned int* cur = reinterpret_cast<unsigned int*>(carve(size_t(n) * 4));
  int32_t* order = reinterpret_cast<int32_t*>(carve(size_t(n) * 4));

  // 1. undirected degrees over the concatenated (out ++ in) rows
  GT_CUDA(cudaMemsetAsync(small + 12, 0, 8, s));
  uint32_t* keep_bits = undirected_degrees(g, cat, o.deg, "tc.und_degree");
  {
    Phase ph("tc.und_degree", 0.0);
    GT_LAUNCH(gtd::max_i32_kernel, grid_cap(ceil_div64(n, 256)), 256, 0, o.deg, n,
              reinterpret_cast<int*>(small + 12));
    GT_LAUNCH(gtd::deg64_kernel, ceil_div(n, 256), 256, 0, o.deg, n, und_off);
    exclusive_scan_i64(und_off, n, small + 13);  // = 2m
  }
  int64_t hh[2];
  d2h(hh, small + 12, sizeof hh);
  sync();
  const int max_deg = int(hh[0] & 0xffffffff);
  const int64_t two_m = hh[1];
  // 2. rank = position in (degree, id) order
  {
    uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(n));
    uint64_t* kbuf = ws_n<uint64_t>(WS_KEYS_B, size_t(n));
    SortPlan plan = make_plan(0, o.kbits + bits_for(int64_t(max_deg) + 1));
    SortHist h = sort_hist_begin(0);
    {
      Phase ph("tc.rank", 12.0 * n);
      GT_LAUNCH(gtd::rank_keys_kernel, grid_cap(ceil_div64(n, 1024)), 256, 0, o.deg, n, o.kbits,
                plan, h.hist, ka);
    }
    uint64_t* sorted = radix_sort(ka, kbuf, n, plan, h, "tc.sort");
    Phase ph("tc.rank", 12.0 * n);
    GT_LAUNCH(gtd::rank_scatter_kernel, ceil_div(n, 256), 256, 0, sorted, n,
              (uint64_t(1) << o.kbits) - 1, o.rank, order);
  }
  // 3. higher-ranked neighbours of every id-row, sorted, in a degree-sized slice
  int32_t* buf = ws_n<int32_t>(WS_TMP2, size_t(std::max<int64_t>(two_m, 1)));
  int32_t* lists = reinterpret_cast<int32_t*>(ws_get(WS_TMP4, size_t(n) * 8 + 64));
  int32_t* big_fill = lists;
  int32_t* big_sort = lists + n;
  unsigned int* nbig = reinterpret_cast<unsigned int*>(small + 14);
  GT_CUDA(cudaMemsetAsync(nbig, 0, 16, s));  // [14] list sizes, [15] max d+ past the warp sorts
  {
    Phase ph("tc.orient", 16.0 * (n + 1) * 2 + 4.0 * slots + 8.0 * n + 4.0 * two_m);
    GT_LAUNCH(gtd::fill_rows_kernel, grid_cap(ceil_div64(n, 256)), 256, 0, cat, g->out_off,
              g->out_adj, g->in_off, g->in_adj, n, o.rank, keep_bits, und_off, buf, dplus,
              big_fill, big_sort, nbig, o.kbits);
  }
  unsigned int nb[2];
  d2h(nb, nbig, sizeof nb);
  sync();
  if (nb[0]) {  // hub rows: chunked, one pass, then sorted with the other long rows
    Phase ph("tc.orient_big", 0.0);
    const int nr = int(nb[0]);
    int64_t* coff = ws_n<int64_t>(WS_TMP1, size_t(nr) + 1);  // tile_row is dead by now
    GT_LAUNCH(gtd::big_chunk_count_kernel, ceil_div(nr, 256), 256, 0, big_fill, nr, cat, coff);
    exclusive_scan_i64(coff, nr, coff + nr);
    GT_LAUNCH(gtd::fill_big_kernel, 4 * ctx().sm_count, 256, 0, big_fill, nr, coff, cat,
              g->out_off, g->out_adj, g->in_off, g->in_adj, o.rank, keep_bits, und_off, buf,
              dplus);
    GT_LAUNCH(gtd::copy_rows_kernel, ceil_div(nr, 256), 256, 0, big_fill, nr, big_sort + nb[1]);
    nb[1] += nb[0];
  }
  // long rows (listed in big_sort): warp radix sorts in shared memory; the
  // rare rows beyond TC_SORT_MID are only flagged here (small[15] = their max
  // d+) and sorted after the offsets' sync below, so the common case costs no
  // extra host round trip
  if (nb[1]) {
    Phase ph("tc.orient_sort", 0.0);
    const int nr = int(nb[1]);
    const int smem = 4 * (2 * gtd::TC_SORT_MID + 256) * 4;
    GT_CUDA(cudaFuncSetAttribute(gtd::sort_rows_mid_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    GT_LAUNCH(gtd::sort_rows_mid_kernel, std::min(ceil_div(nr, 4), 3 * ctx().sm_count), 128, smem,
              big_sort, nr, und_off, dplus, buf, o.kbits,
              reinterpret_cast<unsigned int*>(small + 15));
  }
  // 4. rank-space offsets of N+ and N-, then rows placed + N- filed
  {
    Phase ph("tc.oriented_csr", 8.0 * n + 16.0 * (n + 1) * 2);
    GT_LAUNCH(gtd::rank_counts_kernel, ceil_div(n, 256), 256, 0, o.rank, o.deg, dplus, n, o.off_p,
              o.off_m);
    exclusive_scan_i64(o.off_p, n, small + 4);
    exclusive_scan_i64(o.off_m, n, small + 5);
  }
  int64_t hm[12];
  d2h(hm, small + 4, sizeof hm);
  sync();
  o.m = hm[0];
  if (uint32_t(hm[11]) > uint32_t(gtd::TC_SORT_MID)) {
    // rows past the warp sorts: shared-memory bitonic, one launch per padded
    // size so each CTA reserves only what its rows need; longer rows: LSD
    // radix sort of that row alone
    Phase ph("tc.orient_sort", 0.0);
    const int nr = int(nb[1]);
    int64_t* d_cd = reinterpret_cast<int64_t*>(ws_get(WS_TMP0, size_t(nr) * 16 + 64));
    GT_LAUNCH(gtd::gather_rows_kernel, ceil_div(nr, 256), 256, 0, big_sort, nr,
              (const int64_t*)nullptr, dplus, 0, d_cd);
    GT_LAUNCH(gtd::gather_rows_kernel, ceil_div(nr, 256), 256, 0, big_sort, nr, und_off,
              (const int32_t*)nullptr, 0, d_cd + nr);
    std::vector<int64_t> cd(2 * size_t(nr));
    d2h(cd.data(), d_cd, cd.size() * 8);
    std::vector<int32_t> ids(nr);
    d2h(ids.data(), big_sort, size_t(nr) * 4);
    sync();
    std::vector<int32_t> by_size;
    int32_t* d_rows = big_sort;
    for (int p2 = 2 * gtd::TC_SORT_MID; p2 <= gtd::TC_SORT_CTA; p2 <<= 1) {
      by_size.clear();
      for (int r = 0; r < nr; ++r)
        if (cd[r] <= p2 && cd[r] > p2 / 2) by_size.push_back(ids[r]);
      if (by_size.empty()) continue;
      h2d(d_rows, by_size.data(), by_size.size() * 4);
      const int smem = p2 * 4;
      GT_CUDA(cudaFuncSetAttribute(gtd::sort_rows_big_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      GT_LAUNCH(gtd::sort_rows_big_kernel, int(by_size.size()), 256, smem, d_rows, und_off, dplus,
                buf);
      d_rows += by_size.size();
    }
    for (int r = 0; r < nr; ++r) {
      const int64_t c = cd[r], off = cd[nr + r];
      if (c <= gtd::TC_SORT_CTA) continue;
      uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(c));
      uint64_t* kbuf = ws_n<uint64_t>(WS_KEYS_B, size_t(c));
      GT_LAUNCH(gtd::i32_to_u64_kernel, ceil_div(c, 256), 256, 0, buf + off, int64_t(c), ka);
      SortPlan plan = make_plan(0, o.kbits);
      SortHist h = sort_hist_begin(0);
      sort_histogram(ka, c, plan, h);
      uint64_t* srt = radix_sort(ka, kbuf, c, plan, h, "tc.sort");
      GT_LAUNCH(gtd::u64_to_i32_kernel, ceil_div(c, 256), 256, 0, srt, int64_t(c), buf + off);
    }
  }
  o.adj_p = ws_n<int32_t>(WS_TMP0, size_t(o.m) + 1);
  o.nm = reinterpret_cast<int2*>(ws_get(WS_TMP1, size_t(o.m) * 8 + 16));
  {
    Phase ph("tc.oriented_csr", 8.0 * o.m + 4.0 * o.m + 4.0 * o.m + 8.0 * o.m + 8.0 * n);
    if (o.m > 0) {
      const int64_t tiles = ceil_div64(o.m, gtd::TC_CAND_TILE);
      int64_t* tile_row = ws_n<int64_t>(WS_KEYS_A, size_t(tiles) + 1);  // sorts are done
      unsigned long long* cur64 = ws_n<unsigned long long>(WS_KEYS_B, size_t(n));
      GT_CUDA(cudaMemcpyAsync(cur64, o.off_m, size_t(n) * 8, cudaMemcpyDeviceToDevice, s));
      GT_LAUNCH(gtd::cand_tile_rows_kernel, ceil_div(tiles + 1, 256), 256, 0, o.off_p, n, o.m,
                tiles, tile_row);
      GT_LAUNCH(gtd::place_tiles_kernel, static_cast<int>(tiles), 256, 0, o.off_p, tile_row, o.m,
                order, und_off, buf, cur64, o.adj_p, o.nm);
    }
  }
  return o;
}

void triangle_orientation(const gt_graph* g, int32_t* h_deg, int32_t* h_rank, int64_t* h_off_p,
                          int32_t* h_adj_p, int64_t* m_out) {
  require_init();
  if (!g) fail(GT_EINVAL, "null graph");
  *m_out = 0;
  if (g->n == 0) return;
  if (g->e == 0) fail(GT_EINVAL, "graph has no edges");
  Oriented o = orient(g);
  *m_out = o.m;
  if (h_deg) d2h(h_deg, o.deg, size_t(g->n) * 4);
  if (h_rank) d2h(h_rank, o.rank, size_t(g->n) * 4);
  if (h_off_p) d2h(h_off_p, o.off_p, size_t(g->n + 1) * 8);
  if (h_adj_p) d2h(h_adj_p, o.adj_p, size_t(o.m) * 4);
  sync();
}

static int64_t count_oriented(const Oriented& o, int part, int nparts);

int64_t triangles(const gt_graph* g, int part, int nparts) {
  require_init();
  if (nparts < 1 || part < 0 || part >= nparts) fail(GT_EINVAL, "part must be in [0, nparts)");
  if (!g) fail(GT_EINVAL, "null graph");
  const int64_t n = g->n, e = g->e;
  if (n == 0 || e == 0) return 0;
  cudaStream_t s = ctx().stream;
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  const Oriented o = orient(g);
  g->m_und = o.m;
  return count_oriented(o, part, nparts);
}

// The count over an orientation (rank space: N+ rows, N- lists of the middle
// vertices v = part mod nparts).
static int64_t count_oriented(const Oriented& o, int part, int nparts) {
  const int64_t n = o.n, m = o.m;
  cudaStream_t s = ctx().stream;
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  if (m == 0) return 0;
  if (m >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "triangles: >= 2^31 undirected edges");

  int64_t* off_m = o.off_m;
  const int2* nm = o.nm;
  // work-list scratch
  char* p = static_cast<char*>(ws_get(WS_COLS, size_t(n + 1) * 8 * 4 + 96));
  auto carve = [&](size_t b) { char* r = p; p += (b + 15) & ~size_t(15); return r; };
  int64_t* t0 = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  int64_t* t1 = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  int64_t* t2 = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  int64_t* t3 = reinterpret_cast<int64_t*>(carve(size_t(n + 1) * 8));
  // table windows; GT_TC_WINDOW (ranks, power of two >= 64) shrinks them so
  // that small test graphs exercise the split / hash / CTA paths
  int64_t bm_bits = gtd::TC_BM_BITS;
  if (const char* env = getenv("GT_TC_WINDOW")) bm_bits = std::max<int64_t>(64, atoll(env));
  bm_bits = std::min<int64_t>(bm_bits, gtd::TC_BM_BITS);
  const int split_top = int(std::min<int64_t>(bm_bits / 2, gtd::TC_SPLIT_TOP));
  // the window holds bm_cap positions; position 0 (rank n - bm_cap) is kept
  // free as the probe pad, so bitmap tasks are the v with n - 1 - v <= bm_cap - 1
  const int64_t bm_cap = bm_bits;
  bm_bits = bm_cap - 1;
  // 6. work lists
  {
    Phase ph("tc.tasks", 8.0 * (n + 1) * 8);
    GT_CUDA(cudaMemsetAsync(small + 14, 0, 16, s));
    GT_LAUNCH(gtd::tc_task_count_kernel, ceil_div(n, 256), 256, 0, o.off_p, off_m, n, part, nparts,
              bm_bits, t0, t1, t2, t3);
    exclusive_scan_i64(t0, n, small + 8);
    exclusive_scan_i64(t1, n, small + 9);
    exclusive_scan_i64(t2, n, small + 10);
    exclusive_scan_i64(t3, n, small + 11);
    GT_CUDA(cudaMemsetAsync(small + 12, 0, 8, s));
    GT_LAUNCH(gtd::max_dplus_kernel, grid_cap(ceil_div64(n, 256)), 256, 0, o.off_p, o.adj_p, n,
              n - 1 - bm_bits, reinterpret_cast<unsigned long long*>(small + 14),
              reinterpret_cast<unsigned long long*>(small + 12));
    // [14] max d+, [15] probes, [12] probes of the bitmap tasks
  }
  int64_t h[8];
  d2h(h, small + 8, sizeof h);  // bitmap / warp / CTA task counts, ..., max d+, probes
  sync();
  if (const char* st = getenv("GT_TC_STATS"); st && atoi(st)) {
    unsigned long long* d_st = reinterpret_cast<unsigned long long*>(counters + 32);
    d_st = reinterpret_cast<unsigned long long*>(ws_get(WS_TMP4, 32 * 8));
    GT_CUDA(cudaMemsetAsync(d_st, 0, 32 * 8, s));
    GT_LAUNCH(gtd::tc_stats_kernel, ceil_div(n, 256), 256, 0, o.off_p, off_m, nm, n, bm_bits, d_st);
    unsigned long long hs[32];
    d2h(hs, d_st, sizeof hs);
    sync();
    const char* names[4] = {"bitmap", "hash-warp", "cta", "split"};
    for (int k = 0; k < 4; ++k)
      fprintf(stderr, "[gt tc stats] %-9s v=%llu sum_d+=%llu sum_d-=%llu probes=%llu\n", names[k],
              hs[4 * k], hs[4 * k + 1], hs[4 * k + 3], hs[4 * k + 2]);
    fprintf(stderr, "[gt tc stats] cta probes with n-1-v <= 2^17..2^20: %llu %llu %llu %llu\n",
            hs[16], hs[17], hs[18], hs[19]);
    fprintf(stderr, "[gt tc stats] n=%lld m=%lld max_d+=%lld probes=%lld probes_bm=%lld\n", (long long)n,
            (long long)m, (long long)h[6], (long long)h[7], (long long)h[4]);
  }
  const int64_t n_bm = h[0], n_hw = h[1], n_ct = h[2], n_sp = h[3], max_dp = h[6], probes = h[7];
  const int64_t probes_bm = h[4];  // read as 16-bit window ranks (adj16)
  const int64_t n_wt = n_sp + n_hw;  // warp tasks after the bitmap ones: split, then hash
  if (n_bm + n_wt + n_ct >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "triangle work list too long");
  int2* tasks = ws_n<int2>(WS_TMP2, size_t(n_bm + n_wt + n_ct) + 1);  // buf is dead by now
  {
    Phase ph("tc.tasks", 8.0 * (n_bm + n_wt + n_ct));
    if (n_bm) GT_LAUNCH(gtd::tc_task_fill_kernel, ceil_div(n, 256), 256, 0, t0, n, tasks);
    if (n_sp) GT_LAUNCH(gtd::tc_task_fill_kernel, ceil_div(n, 256), 256, 0, t3, n, tasks + n_bm);
    if (n_hw)
      GT_LAUNCH(gtd::tc_task_fill_kernel, ceil_div(n, 256), 256, 0, t1, n, tasks + n_bm + n_sp);
    if (n_ct)
      GT_LAUNCH(gtd::tc_task_fill_kernel, ceil_div(n, 256), 256, 0, t2, n, tasks + n_bm + n_wt);
  }
  static const bool order_by_u = [] {  // GT_TC_ORDER=0: bitmap tasks in v order (A/B)
    const char* env = getenv("GT_TC_ORDER");
    return !(env && atoi(env) == 0);
  }();
  auto order_tasks = [&](int2* tk, int64_t nt, int chunk) {
    Phase ph("tc.tasks", 40.0 * nt);
    uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(nt));
    uint64_t* kb = ws_n<uint64_t>(WS_KEYS_B, size_t(nt));
    GT_LAUNCH(gtd::tc_task_keys_kernel, ceil_div(nt, 256), 256, 0, tk, nt, chunk, off_m, nm, ka);
    SortPlan plan = make_plan(32, 32 + bits_for(m + 1));
    SortHist hs = sort_hist_begin(0);
    sort_histogram(ka, nt, plan, hs);
    uint64_t* srt = radix_sort(ka, kb, nt, plan, hs, "tc.tasks");
    int2* tmp = reinterpret_cast<int2*>(srt == ka ? kb : ka);
    GT_LAUNCH(gtd::tc_task_permute_kernel, ceil_div(nt, 256), 256, 0, srt, nt, tk, tmp);
    GT_CUDA(cudaMemcpyAsync(tk, tmp, size_t(nt) * sizeof(int2), cudaMemcpyDeviceToDevice, s));
  };
  if (order_by_u && n_bm > 1) order_tasks(tasks, n_bm, gtd::TC_CHUNK);
  // (the CTA tasks are left in v order: in u order, with chunks of 2048..16384
  // arcs, they measured 198-207 ms against 193 at C4 — a chunk of a long
  // N-(v) list spans most of the u range, so tasks in flight share little)
  unsigned long long* total = reinterpret_cast<unsigned long long*>(small + 6);
  GT_CUDA(cudaMemsetAsync(total, 0, 8, s));
  if (n_bm + n_wt) {
    // algorithmic bytes: every probed suffix element (2 B for the bitmap
    // tasks, which read adj16, 4 B otherwise), the N- entries (8 B) and the N+
    // lists loaded into tables (4 B); hash tasks counted here too
    Phase ph("tc.count", 0.0);  // issue-bound probes: no HBM bytes claimed
    GT_CUDA(cudaMemsetAsync(counters + 22, 0, 4, s));
    // GT_TC_WARPS (A/B): warps per CTA, each with its own 8 KB table; the
    // grid fills every SM to its occupancy limit
    static const int tc_warps = [] {
      const char* env = getenv("GT_TC_WARPS");
      const int w = env ? atoi(env) : 8;
      return w < 1 ? 1 : (w > 8 ? 8 : w);
    }();
    const int smem = tc_warps * gtd::TC_SLOTS * 4;
    GT_CUDA(cudaFuncSetAttribute(gtd::tc_count_warp_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    GT_CUDA(cudaFuncSetAttribute(gtd::tc_count_warp_kernel,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 0;
    GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gtd::tc_count_warp_kernel,
                                                          32 * tc_warps, smem));
    per_sm = std::max(per_sm, 1);
    // 16-bit copy of the window ranks for the bitmap tasks
    const int32_t base16 = int32_t(n - bm_cap);
    uint16_t* adj16 = reinterpret_cast<uint16_t*>(ws_get(WS_KEYS_A, size_t(m) * 2 + 64));
    if (n_bm) GT_LAUNCH(gtd::adj16_kernel, grid_cap(ceil_div64(m, 256)), 256, 0, o.adj_p, m, base16,
                        adj16);
    GT_LAUNCH(gtd::tc_count_warp_kernel, ctx().sm_count * per_sm, 32 * tc_warps, smem, o.off_p,
              o.adj_p, off_m,
              nm, tasks, n_bm, n_bm + n_sp, n_bm + n_wt, n, split_top, part, nparts, counters + 22,
              total, adj16, base16);
  }
  if (n_ct) {
    Phase ph("tc.count_hash", 0.0);
    // GT_TC_TABLE_SMEM_MAX (bytes) shrinks the shared table (tests drive the
    // global-table path with it)
    size_t cap = size_t(gtd::TC_CTA_SLOTS) * 4;
    if (const char* env = getenv("GT_TC_TABLE_SMEM_MAX")) cap = std::min(cap, size_t(atoll(env)));
    int smem_log = 5;
    while ((size_t(4) << (smem_log + 1)) <= cap) ++smem_log;
    const int smem = 4 << smem_log;
    GT_CUDA(cudaFuncSetAttribute(gtd::tc_count_cta_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // CTA bitmap window = the shared table as bits; a GT_TC_WINDOW test run
    // turns it off unless GT_TC_CTA_WINDOW (ranks) sets it, so that the hash
    // paths stay covered
    int64_t cta_bm_bits = int64_t(smem) * 8;
    if (getenv("GT_TC_WINDOW")) {
      const char* cw = getenv("GT_TC_CTA_WINDOW");
      cta_bm_bits = cw ? std::min<int64_t>(cta_bm_bits, atoll(cw)) : 0;
    }
    int per_sm = 0;
    GT_CUDA(cudaFuncSetAttribute(gtd::tc_count_cta_kernel,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gtd::tc_count_cta_kernel, 256,
                                                          smem));
    const int grid = static_cast<int>(
        std::min<int64_t>(n_ct, int64_t(std::max(per_sm, 1)) * ctx().sm_count));
    int32_t* gtab = nullptr;
    int gtab_log = 0;
    if (2 * max_dp > (int64_t(1) << smem_log)) {
      gtab_log = 5;
      while ((int64_t(1) << gtab_log) < 8 * max_dp) ++gtab_log;
      gtab = ws_n<int32_t>(WS_TMP4, size_t(grid) << gtab_log);
    }
    // window base: a multiple of 32 with every rank of [win_base, n) inside
    // the table; the threshold leaves ranks below v + 1 for the pad
    const int64_t cta_thresh = cta_bm_bits >= 128 ? cta_bm_bits - 64 : -1;
    const int32_t win_base =
        cta_thresh < 0 ? 0 : int32_t(std::max<int64_t>(0, (n - cta_bm_bits + 31) & ~int64_t(31)));
    GT_LAUNCH(gtd::tc_count_cta_kernel, grid, 256, smem, o.off_p, o.adj_p, off_m, nm,
              tasks + n_bm + n_wt, n_ct, smem_log, gtab, gtab_log, total, n, cta_thresh, win_base);
  }
  int64_t result = 0;
  d2h(&result, total, 8);
  sync();
  return result;
}

// Sharded orientation primitives (distributed.triangle_count); see the
// kernels above and include/gtb200.h.
int64_t tc_undirected_keys(const int64_t* off, const int32_t* adj, int64_t rows, int64_t row_lo,
                           int kbits, uint64_t* keys) {
  require_init();
  if (rows <= 0) return 0;
  int64_t* cnt = ws_n<int64_t>(WS_TMP3, size_t(rows) + 1);
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  const int grid = grid_cap(ceil_div64(rows, 8));
  GT_LAUNCH(gtd::tc_und_count_kernel, grid, 256, 0, off, adj, rows, row_lo, cnt);
  exclusive_scan_i64(cnt, rows, small + 2);
  GT_LAUNCH(gtd::tc_und_write_kernel, grid, 256, 0, off, adj, rows, row_lo, kbits, cnt, keys);
  int64_t total = 0;
  d2h(&total, small + 2, 8);
  sync();
  return total;
}

int64_t tc_orient_keys(const int64_t* off, const int32_t* adj, int64_t rows, int64_t row_lo,
                       const int32_t* rank, int kbits, uint64_t* keys) {
  require_init();
  if (rows <= 0) return 0;
  int64_t* cnt = ws_n<int64_t>(WS_TMP3, size_t(rows) + 1);
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  const int grid = grid_cap(ceil_div64(rows, 8));
  GT_LAUNCH(gtd::tc_orient_count_kernel, grid, 256, 0, off, adj, rows, row_lo, rank, cnt);
  exclusive_scan_i64(cnt, rows, small + 2);
  GT_LAUNCH(gtd::tc_orient_write_kernel, grid, 256, 0, off, adj, rows, row_lo, rank, kbits, cnt,
            keys);
  int64_t total = 0;
  d2h(&total, small + 2, 8);
  sync();
  return total;
}

// rank[id] = position of id in (degree, id) order (algorithms.py:103-106).
void tc_degree_rank(const int64_t* deg, int64_t n, int32_t* rank) {
  require_init();
  if (n <= 0) return;
  if (n >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "degree rank: >= 2^31 nodes");
  int32_t* d32 = ws_n<int32_t>(WS_TMP3, size_t(n) * 2);
  int32_t* order = d32 + n;
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  GT_LAUNCH(gtd::deg64_to_32_kernel, ceil_div(n, 256), 256, 0, deg, n, d32);
  GT_CUDA(cudaMemsetAsync(small + 12, 0, 8, ctx().stream));
  GT_LAUNCH(gtd::max_i32_kernel, grid_cap(ceil_div64(n, 256)), 256, 0, d32, n,
            reinterpret_cast<int*>(small + 12));
  int64_t mx = 0;
  d2h(&mx, small + 12, 8);
  sync();
  const int kbits = bits_for(n);
  uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(n));
  uint64_t* kb = ws_n<uint64_t>(WS_KEYS_B, size_t(n));
  SortPlan plan = make_plan(0, kbits + bits_for(int64_t(mx & 0xffffffff) + 1));
  SortHist h = sort_hist_begin(0);
  GT_LAUNCH(gtd::rank_keys_kernel, grid_cap(ceil_div64(n, 1024)), 256, 0, d32, n, kbits, plan,
            h.hist, ka);
  uint64_t* sorted = radix_sort(ka, kb, n, plan, h, "tc.sort");
  GT_LAUNCH(gtd::rank_scatter_kernel, ceil_div(n, 256), 256, 0, sorted, n,
            (uint64_t(1) << kbits) - 1, rank, order);
  sync();
}

// Triangles whose middle vertex v = part (mod nparts), from a rank-space
// orientation given by the caller (replicated N+ rows).
int64_t triangles_oriented(const int64_t* off_p, const int32_t* adj_p, int64_t n, int64_t m,
                           int part, int nparts) {
  require_init();
  if (nparts < 1 || part < 0 || part >= nparts) fail(GT_EINVAL, "part must be in [0, nparts)");
  if (n <= 0 || m <= 0) return 0;
  if (n >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "triangles: >= 2^31 nodes");
  cudaStream_t s = ctx().stream;
  Oriented o;
  o.n = n;
  o.m = m;
  o.kbits = bits_for(n);
  o.off_p = const_cast<int64_t*>(off_p);
  o.adj_p = const_cast<int32_t*>(adj_p);
  char* p = static_cast<char*>(ws_get(WS_TMP3, size_t(n + 1) * 8 + size_t(n) * 4 + 64));
  o.off_m = reinterpret_cast<int64_t*>(p);
  unsigned int* cur = reinterpret_cast<unsigned int*>(p + ((size_t(n + 1) * 8 + 15) & ~size_t(15)));
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  GT_CUDA(cudaMemsetAsync(o.off_m, 0, size_t(n + 1) * 8, s));
  GT_LAUNCH(gtd::tc_owned_indeg_kernel, grid_cap(ceil_div64(m, 256)), 256, 0, adj_p, m, part,
            nparts, reinterpret_cast<unsigned long long*>(o.off_m));
  exclusive_scan_i64(o.off_m, n, small + 3);
  int64_t owned = 0;
  d2h(&owned, small + 3, 8);
  sync();
  o.nm = reinterpret_cast<int2*>(ws_get(WS_TMP1, size_t(std::max<int64_t>(owned, 1)) * 8 + 16));
  GT_CUDA(cudaMemsetAsync(cur, 0, size_t(n) * 4, s));
  GT_LAUNCH(gtd::tc_file_owned_kernel, grid_cap(ceil_div64(n, 8)), 256, 0, off_p, adj_p, n, part,
            nparts, o.off_m, cur, o.nm);
  return count_oriented(o, part, nparts);
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_triangles(const gt_graph* g, int64_t* count) {
  GT_API_BEGIN
  if (!count) fail(GT_EINVAL, "count must not be NULL");
  *count = triangles(g, 0, 1);
  GT_API_END
}

int gt_graph_undirected_edges(const gt_graph* g, int64_t* m) {
  GT_API_BEGIN
  if (!g || !m) fail(GT_EINVAL, "graph and m must not be NULL");
  *m = g->m_und;
  GT_API_END
}

int gt_triangles_part(const gt_graph* g, int part, int nparts, int64_t* count) {
  GT_API_BEGIN
  if (!count) fail(GT_EINVAL, "count must not be NULL");
  *count = triangles(g, part, nparts);
  GT_API_END
}

int gt_tc_undirected_keys(const int64_t* d_off, const int32_t* d_adj, int64_t rows, int64_t row_lo,
                          int kbits, uint64_t* d_keys, int64_t* n_keys) {
  GT_API_BEGIN
  if (!n_keys || (rows > 0 && (!d_off || !d_adj || !d_keys))) fail(GT_EINVAL, "null argument");
  if (kbits < 1 || kbits > 31) fail(GT_EINVAL, "kbits must be in [1, 31]");
  *n_keys = tc_undirected_keys(d_off, d_adj, rows, row_lo, kbits, d_keys);
  GT_API_END
}

int gt_tc_degree_rank(const int64_t* d_deg, int64_t n, int32_t* d_rank) {
  GT_API_BEGIN
  if (n > 0 && (!d_deg || !d_rank)) fail(GT_EINVAL, "null argument");
  tc_degree_rank(d_deg, n, d_rank);
  GT_API_END
}

int gt_tc_orient_keys(const int64_t* d_off, const int32_t* d_adj, int64_t rows, int64_t row_lo,
                      const int32_t* d_rank, int kbits, uint64_t* d_keys, int64_t* m_keys) {
  GT_API_BEGIN
  if (!m_keys || (rows > 0 && (!d_off || !d_adj || !d_rank || !d_keys)))
    fail(GT_EINVAL, "null argument");
  if (kbits < 1 || kbits > 31) fail(GT_EINVAL, "kbits must be in [1, 31]");
  *m_keys = tc_orient_keys(d_off, d_adj, rows, row_lo, d_rank, kbits, d_keys);
  GT_API_END
}

int gt_triangles_oriented_part(const int64_t* d_off_p, const int32_t* d_adj_p, int64_t n,
                               int64_t m, int part, int nparts, int64_t* count) {
  GT_API_BEGIN
  if (!count) fail(GT_EINVAL, "count must not be NULL");
  if (n > 0 && m > 0 && (!d_off_p || !d_adj_p)) fail(GT_EINVAL, "null argument");
  *count = triangles_oriented(d_off_p, d_adj_p, n, m, part, nparts);
  GT_API_END
}

int gt_triangle_orientation(const gt_graph* g, int32_t* h_deg, int32_t* h_rank, int64_t* h_off_p,
                            int32_t* h_adj_p, int64_t* m) {
  GT_API_BEGIN
  if (!m) fail(GT_EINVAL, "m must not be NULL");
  triangle_orientation(g, h_deg, h_rank, h_off_p, h_adj_p, m);
  GT_API_END
}

}  // extern "C"
