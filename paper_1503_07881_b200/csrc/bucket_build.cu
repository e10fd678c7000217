// bucket_build.cu — ToGraph, dense-id path: MSD bucket build of both CSRs.
//
// Reference: table_to_graph (convert.py:128-175) = node set (np.unique,
// convert.py:45-59) + sort of packed (src, dst) keys and drop of adjacent
// duplicates (convert.py:71-89, parallel.py:52-93) + offsets by bincount /
// cumsum (convert.py:154-157) + per-node pools (convert.py:92-125).
//
// Device design. When the ids span a range
// W not much wider than the table (W <= 4R), a key is built from id OFFSETS
// (x - lo), kw = ceil(log2 W) bits per side, so no rank lookup is needed
// before the sort:
//   out key = (src-lo) << kw | (dst-lo),   in key = (dst-lo) << kw | (src-lo)
// and both CSRs are built independently from the raw rows (the set of
// distinct (src, dst) pairs is the set of distinct (dst, src) pairs).
//
//   bk_presence_hist   16 B/row   presence bit per id + level-1 digit counts
//   word_prefix/ids              rank of every present id, sorted ids
//   bk_pack_part       32 B/row   both keys, scattered by level-1 digit
//                                 (non-stable: the leaf sort orders fully)
//   bk_seg_hist/part   8+16 B/key per further level, P key bits in total
//   bk_leaf<MAIN>      8+4 B/key  leaf = consecutive buckets of <= CAP keys:
//                                 LSD radix sort in shared memory, dedupe,
//                                 decoupled look-back for the CSR position,
//                                 adjacency (ranks) + row offsets written
// Buckets holding more than CAP keys (rows of high degree) are split further
// (by row, then by the top bits of the column), sorted + deduplicated in a
// COUNT pass (LSD leaves, or a shared-memory bitmap per column range for the
// largest pieces), placed by the main pass through a placeholder whose count
// is the bucket's deduplicated total, and written by an EMIT pass.
// Every partition level is a non-stable scatter (shared-memory atomics +
// one global cursor per digit per tile): measured at 4.2 TB/s for 8-bit
// digits on B200 (scripts/ubench/ubench_r2.cu), against 2.4 TB/s for the
// stable onesweep pass it replaces.
#include "graph.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace gt {
// build.cu
void launch_word_prefix(uint2* words, int64_t nw, int64_t* total_out);
void launch_ids(const uint2* words, int64_t nw, int64_t lo, int64_t* ids);
void launch_presence(const int64_t* a, const int64_t* b, int64_t n, int64_t lo, uint2* words);
}  // namespace gt

namespace gtd {

constexpr int BK_MAXD = 512;           // digits per partition level (<= 9 bits)
constexpr int LF_THREADS = 1024;       // leaf sort: threads per CTA
constexpr int LF_KPT = 8;              // keys per thread
constexpr int LF_CAP = LF_THREADS * LF_KPT;  // keys per leaf (8192)
constexpr int LF_WARPS = LF_THREADS / 32;
constexpr int LF_SLOTS = 32 * LF_KPT;  // keys per warp (256)

// ---------------------------------------------------------------- leaves --
enum : int32_t { LK_GROUP = 0, LK_PLACEHOLDER = 1, LK_ROWS = 2, LK_HUBKIDS = 3, LK_BITMAP = 4 };

struct BkLeaf {
  int64_t begin;     // first key (index into the 2R-key buffer)
  uint64_t key_lo;   // smallest key of the leaf's key range
  uint64_t key_hi;   // end of the key range (exclusive)
  int32_t count;     // keys in the buffer (<= LF_CAP, except placeholder/bitmap)
  int32_t info;      // bit 0: buffer (0 = A, 1 = B); bit 1: side; bits 2..4: kind
  int32_t huge;      // huge-bucket index (placeholder / huge leaves), else -1
  int32_t hub;       // hub-row index (kinds 3, 4), else -1
  int32_t k0;        // first column child (kinds 3, 4)
  int32_t pad;
};

struct BkArgs {
  const uint64_t* buf[2];    // A, B (keys)
  uint64_t* wbuf[2];         // writable views (COUNT writes deduplicated keys back)
  const uint2* words;        // rank map over id offsets
  int kw;                    // bits per side
  int64_t n_ids;             // W: id offsets are in [0, W)
  int64_t n_nodes;
  int64_t* off[2];           // out_off, in_off  [N+1]
  int32_t* adj[2];           // out_adj, in_adj
  uint32_t* deg;             // [2][N] deduplicated row counts of huge buckets
  unsigned long long* huge_total;  // [n_huge] deduplicated keys per huge bucket
  uint32_t* child_cnt;       // [n_hub][n_kids]
  uint32_t* child_base;      // [n_hub][n_kids]
  int kid_bits;              // column bits per hub child (kw - c)
  int n_kids;                // 2^c
  int32_t* leaf_d;           // [n_leaves] deduplicated keys of each huge leaf
  int64_t* main_d;           // [u0+1 | u1+1] per main leaf: count, then (scanned) position
  uint32_t* tmp[2];          // adjacency at raw positions (rows entries per side)
  int64_t rows;              // R: side 1 keys start at R in the key buffers
};

__device__ __forceinline__ uint32_t bk_rank(const uint2* __restrict__ words, uint64_t off) {
  const uint2 w = words[off >> 5];
  return w.y + __popc(w.x & ((1u << (off & 31)) - 1u));
}
__device__ __forceinline__ bool bk_present(const uint2* __restrict__ words, uint64_t off) {
  return (words[off >> 5].x >> (off & 31)) & 1u;
}

// ------------------------------------------------ presence + level-1 digits --
__global__ void __launch_bounds__(256) bk_presence_hist_kernel(
    const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t n, int64_t lo,
    uint2* __restrict__ words, int s1, int nd1, unsigned long long* __restrict__ hist1) {
  __shared__ uint32_t sh[2 * BK_MAXD];
  for (int i = threadIdx.x; i < 2 * BK_MAXD; i += blockDim.x) sh[i] = 0;
  __syncthreads();
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
      atomicAdd(&sh[(u & 1) * BK_MAXD + uint32_t(off[u] >> s1)], 1u);
    }
  }
  for (; i < n; i += stride) {
    const uint64_t a = uint64_t(ld_stream_s64(src + i)) - uint64_t(lo);
    const uint64_t b = uint64_t(ld_stream_s64(dst + i)) - uint64_t(lo);
    atomicOr(&words[a >> 5].x, 1u << (a & 31));
    atomicOr(&words[b >> 5].x, 1u << (b & 31));
    atomicAdd(&sh[uint32_t(a >> s1)], 1u);
    atomicAdd(&sh[BK_MAXD + uint32_t(b >> s1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nd1; d += blockDim.x) {
    if (sh[d]) atomicAdd(&hist1[d], (unsigned long long)sh[d]);
    if (sh[BK_MAXD + d]) atomicAdd(&hist1[nd1 + d], (unsigned long long)sh[BK_MAXD + d]);
  }
}

// Block exclusive scan (256 threads) of per-thread u32 sums; s_w needs 8 slots.
__device__ __forceinline__ uint32_t bk_scan256(uint32_t v, uint32_t* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  uint32_t pre = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) pre += q < w ? s_w[q] : 0u;
  __syncthreads();
  return pre + inc - v;
}

// In-tile digit starts + one global reservation per digit: s_cnt[d] holds
// the tile's count on entry and its in-tile start on exit; s_g[d] = global
// position of the digit's run minus its in-tile start.
__device__ __forceinline__ void bk_reserve(uint32_t* s_cnt, int64_t* s_g, int nd,
                                           unsigned long long* __restrict__ cursor,
                                           uint32_t* s_w) {
  const int per = (nd + 255) >> 8;  // 1 or 2
  uint32_t c0 = 0, c1 = 0;
  const int d0 = threadIdx.x * per;
  if (d0 < nd) c0 = s_cnt[d0];
  if (per == 2 && d0 + 1 < nd) c1 = s_cnt[d0 + 1];
  const uint32_t ex = bk_scan256(c0 + c1, s_w);
  if (d0 < nd) {
    int64_t g = 0;
    if (c0) g = int64_t(atomicAdd(&cursor[d0], (unsigned long long)c0));
    s_g[d0] = g - int64_t(ex);
    s_cnt[d0] = ex;
  }
  if (per == 2 && d0 + 1 < nd) {
    int64_t g = 0;
    if (c1) g = int64_t(atomicAdd(&cursor[d0 + 1], (unsigned long long)c1));
    s_g[d0 + 1] = g - int64_t(ex + c0);
    s_cnt[d0 + 1] = ex + c0;
  }
}

// ------------------------------------------------ pack + level-1 partition --
// Both keys of every row, scattered by the level-1 digit (top bits of the
// row offset) into the side's region of `out` ([0,n) out-keys, [n,2n)
// in-keys); cursor[side*nd1 + d] holds absolute positions.
template <int KPT>
__global__ void __launch_bounds__(256) bk_pack_part_kernel(
    const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t n, int64_t lo,
    int kw, int s1, int nd1, unsigned long long* __restrict__ cursor, uint64_t* __restrict__ out) {
  constexpr int T = 256 * KPT;
  extern __shared__ __align__(16) unsigned char bk_dsm[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(bk_dsm);        // [2][T]
  int64_t* s_g = reinterpret_cast<int64_t*>(s_keys + 2 * T);      // [2][BK_MAXD]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_g + 2 * BK_MAXD);  // [2][BK_MAXD]
  uint32_t* s_w = s_cnt + 2 * BK_MAXD;                             // [8]
  const int tid = threadIdx.x;
  const int sh = kw + s1;  // key >> sh = level-1 digit, both sides
  // 16-byte loads of row pairs when both columns are 16-byte aligned
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int64_t ntiles = (n + T - 1) / T;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T;
    const int valid = int((n - base) < T ? (n - base) : T);
    for (int i = tid; i < 2 * BK_MAXD; i += 256) s_cnt[i] = 0;
    __syncthreads();
    uint64_t ko[KPT], ki[KPT];
    uint32_t so[KPT], si[KPT];
#pragma unroll
    for (int i = 0; i < KPT; i += 2) {
      const int j = (i >> 1) * 512 + 2 * tid;
      int64_t a0 = lo, a1 = lo, b0 = lo, b1 = lo;
      if (j + 1 < valid && aligned) {
        const longlong2 va = __ldcs(reinterpret_cast<const longlong2*>(src + base + j));
        const longlong2 vb = __ldcs(reinterpret_cast<const longlong2*>(dst + base + j));
        a0 = va.x; a1 = va.y; b0 = vb.x; b1 = vb.y;
      } else if (j + 1 < valid) {
        a0 = src[base + j]; a1 = src[base + j + 1];
        b0 = dst[base + j]; b1 = dst[base + j + 1];
      } else if (j < valid) {
        a0 = src[base + j];
        b0 = dst[base + j];
      }
      const uint64_t oa0 = uint64_t(a0) - uint64_t(lo), oa1 = uint64_t(a1) - uint64_t(lo);
      const uint64_t ob0 = uint64_t(b0) - uint64_t(lo), ob1 = uint64_t(b1) - uint64_t(lo);
      ko[i] = (oa0 << kw) | ob0;
      ki[i] = (ob0 << kw) | oa0;
      ko[i + 1] = (oa1 << kw) | ob1;
      ki[i + 1] = (ob1 << kw) | oa1;
    }
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int j = (i >> 1) * 512 + 2 * tid + (i & 1);
      const bool ok = j < valid;
      so[i] = ok ? atomicAdd(&s_cnt[uint32_t(ko[i] >> sh)], 1u) : 0u;
      si[i] = ok ? atomicAdd(&s_cnt[BK_MAXD + uint32_t(ki[i] >> sh)], 1u) : 0u;
    }
    __syncthreads();
    bk_reserve(s_cnt, s_g, nd1, cursor, s_w);
    __syncthreads();
    bk_reserve(s_cnt + BK_MAXD, s_g + BK_MAXD, nd1, cursor + nd1, s_w);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int j = (i >> 1) * 512 + 2 * tid + (i & 1);
      if (j < valid) {
        s_keys[s_cnt[uint32_t(ko[i] >> sh)] + so[i]] = ko[i];
        s_keys[T + s_cnt[BK_MAXD + uint32_t(ki[i] >> sh)] + si[i]] = ki[i];
      }
    }
    __syncthreads();
    for (int j = tid; j < valid; j += 256) {
      const uint64_t k0 = s_keys[j], k1 = s_keys[T + j];
      __stcs(out + s_g[uint32_t(k0 >> sh)] + j, k0);
      __stcs(out + s_g[BK_MAXD + uint32_t(k1 >> sh)] + j, k1);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------ segmented levels --
// Segment s is the range [seg_begin[s], seg_end[s]) of the key buffer;
// seg_tile[s] = first tile of segment s (tiles never straddle segments).
__device__ __forceinline__ int bk_find_seg(const int64_t* __restrict__ seg_tile, int nseg,
                                           int64_t t) {
  int a = 0, b = nseg;  // largest s with seg_tile[s] <= t
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (seg_tile[m] <= t) a = m;
    else b = m;
  }
  return a;
}

template <int KPT>
__global__ void __launch_bounds__(256) bk_seg_hist_kernel(
    const uint64_t* __restrict__ keys, const int64_t* __restrict__ seg_begin,
    const int64_t* __restrict__ seg_end, const int64_t* __restrict__ seg_tile, int nseg,
    int shift, int nd, unsigned int* __restrict__ hist) {
  constexpr int T = 256 * KPT;
  __shared__ uint32_t sh[BK_MAXD];
  __shared__ int s_seg;
  const int64_t ntiles = seg_tile[nseg];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < nd; i += 256) sh[i] = 0;
    if (threadIdx.x == 0) s_seg = bk_find_seg(seg_tile, nseg, t);
    __syncthreads();
    const int s = s_seg;
    const int64_t beg = seg_begin[s] + (t - seg_tile[s]) * T;
    const int64_t end = min(beg + T, seg_end[s]);
    uint64_t k[KPT];
#pragma unroll
    for (int i = 0; i < KPT; ++i) {  // every load in flight before the first atomic
      const int64_t j = beg + i * 256 + threadIdx.x;
      k[i] = j < end ? __ldcs(keys + j) : 0ull;
    }
#pragma unroll
    for (int i = 0; i < KPT; ++i)
      if (beg + i * 256 + threadIdx.x < end)
        atomicAdd(&sh[uint32_t(k[i] >> shift) & uint32_t(nd - 1)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < nd; d += 256)
      if (sh[d]) atomicAdd(&hist[int64_t(s) * nd + d], sh[d]);
    __syncthreads();
  }
}

// Per segment (block): exclusive scan of its digit counts -> cursors (and the
// next level's segment starts, which are the same numbers).
__global__ void __launch_bounds__(256) bk_seg_cursor_kernel(
    const unsigned int* __restrict__ hist, const int64_t* __restrict__ seg_begin, int nd,
    unsigned long long* __restrict__ cursor, int64_t* __restrict__ next_begin) {
  __shared__ uint32_t s_w[8];
  const int s = blockIdx.x;
  const int per = (nd + 255) >> 8;
  const int d0 = threadIdx.x * per;
  uint32_t c0 = d0 < nd ? hist[int64_t(s) * nd + d0] : 0u;
  uint32_t c1 = (per == 2 && d0 + 1 < nd) ? hist[int64_t(s) * nd + d0 + 1] : 0u;
  const uint32_t ex = bk_scan256(c0 + c1, s_w);
  const int64_t b = seg_begin[s];
  if (d0 < nd) {
    cursor[int64_t(s) * nd + d0] = b + ex;
    next_begin[int64_t(s) * nd + d0] = b + ex;
  }
  if (per == 2 && d0 + 1 < nd) {
    cursor[int64_t(s) * nd + d0 + 1] = b + ex + c0;
    next_begin[int64_t(s) * nd + d0 + 1] = b + ex + c0;
  }
}

__global__ void bk_seg_tiles_kernel(const int64_t* __restrict__ seg_begin,
                                    const int64_t* __restrict__ seg_end, int nseg, int T,
                                    int64_t* __restrict__ tiles) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) tiles[s] = (seg_end[s] - seg_begin[s] + T - 1) / T;
}

template <int KPT>
__global__ void __launch_bounds__(256) bk_seg_part_kernel(
    const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
    const int64_t* __restrict__ seg_begin, const int64_t* __restrict__ seg_end,
    const int64_t* __restrict__ seg_tile, int nseg, int shift, int nd,
    unsigned long long* __restrict__ cursor) {
  constexpr int T = 256 * KPT;
  extern __shared__ __align__(16) unsigned char bk_dsm[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(bk_dsm);    // [T]
  int64_t* s_g = reinterpret_cast<int64_t*>(s_keys + T);      // [BK_MAXD]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_g + BK_MAXD);  // [BK_MAXD]
  uint32_t* s_w = s_cnt + BK_MAXD;                             // [8]
  __shared__ int s_seg;
  const int tid = threadIdx.x;
  const uint32_t dm = uint32_t(nd - 1);
  const int64_t ntiles = seg_tile[nseg];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = tid; i < nd; i += 256) s_cnt[i] = 0;
    if (tid == 0) s_seg = bk_find_seg(seg_tile, nseg, t);
    __syncthreads();
    const int s = s_seg;
    const int64_t beg = seg_begin[s] + (t - seg_tile[s]) * T;
    const int valid = int(min(int64_t(T), seg_end[s] - beg));
    uint64_t k[KPT];
    uint32_t slot[KPT];
#pragma unroll
    for (int i = 0; i < KPT; ++i) {  // every load in flight before the first atomic
      const int j = i * 256 + tid;
      k[i] = j < valid ? __ldcs(in + beg + j) : 0ull;
    }
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int j = i * 256 + tid;
      slot[i] = j < valid ? atomicAdd(&s_cnt[uint32_t(k[i] >> shift) & dm], 1u) : 0u;
    }
    __syncthreads();
    bk_reserve(s_cnt, s_g, nd, cursor + int64_t(s) * nd, s_w);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int j = i * 256 + tid;
      if (j < valid) s_keys[s_cnt[uint32_t(k[i] >> shift) & dm] + slot[i]] = k[i];
    }
    __syncthreads();
    for (int j = tid; j < valid; j += 256) {
      const uint64_t key = s_keys[j];
      __stcs(out + s_g[uint32_t(key >> shift) & dm] + j, key);
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------- leaf sort --
constexpr int LF_DBITS = 12;               // CTA counting-sort digit (fallback passes)
constexpr int LF_NC = 2 * LF_CAP;          // counters of the main pass (<= 2 per key)
constexpr int LF_WBITS = 8;                // warp counting-sort digit (<= 256 buckets)
constexpr int LF_WSTRIDE = LF_NC / LF_WARPS;  // counters per warp in warp passes (512)
constexpr int LF_SMALL = 16;               // buckets up to this size: insertion sort
constexpr int LF_WARP_MAX = 1024;          // ranges up to this size: one warp
constexpr int LF_WL = 512;                 // work-list capacity (ranges > LF_SMALL <= CAP/17)
constexpr int LF_ROWS = 4096;              // rows (ids) a leaf may span

struct LfList {
  uint32_t beg[LF_WL];
  uint16_t len[LF_WL];
  uint8_t bits[LF_WL];
  uint32_t n;
};

struct LeafSmem {
  uint64_t a[LF_CAP];
  uint64_t b[LF_CAP];
  uint32_t cnt[LF_NC + 1];                 // counts, then in-place starts
  uint16_t rowbase[LF_ROWS];               // first bucket of each row (main pass)
  uint8_t rowbits[LF_ROWS];                // column bits per bucket of each row
  LfList cta[2], wrp[2];                   // ranges still to sort (ping-pong)
  uint32_t wsum[LF_WARPS];
  uint64_t orv[LF_WARPS];
  unsigned long long base;
  uint32_t ticket;
  uint32_t total;
};

// Block (1024 threads) exclusive scan of u32; s_w needs LF_WARPS slots.
__device__ __forceinline__ uint32_t lf_scan(uint32_t v, uint32_t* s_w, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  uint32_t x = lane < LF_WARPS ? s_w[lane] : 0u;
  uint32_t xi = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, xi, o);
    if (lane >= o) xi += u;
  }
  const uint32_t wpre = __shfl_sync(0xffffffffu, xi - x, w);
  total = __shfl_sync(0xffffffffu, xi, LF_WARPS - 1);
  __syncthreads();
  return wpre + inc - v;
}

__device__ __forceinline__ void lf_insertion(uint64_t* x, int n) {
  for (int i = 1; i < n; ++i) {
    const uint64_t v = x[i];
    int j = i - 1;
    while (j >= 0 && x[j] > v) {
      x[j + 1] = x[j];
      --j;
    }
    x[j + 1] = v;
  }
}

__device__ __forceinline__ int lf_digit_bits(int bits, int len, int cap_bits) {
  // ~2 keys per bucket, at least 4 bits, at most cap_bits and the bits left
  return min(min(cap_bits, bits), max(4, 33 - __clz(uint32_t(len))));
}

// A range of `len` keys at b[beg...] whose keys differ only in their low
// `bits` bits (bits == 0: all equal): sorted now (small), or queued.
__device__ __forceinline__ void lf_route(LeafSmem& s, uint32_t beg, uint32_t len, int bits,
                                         int nxt) {
  if (len <= 1 || bits == 0) return;
  if (len <= LF_SMALL) {
    lf_insertion(s.b + beg, int(len));
    return;
  }
  LfList& L = len <= LF_WARP_MAX ? s.wrp[nxt] : s.cta[nxt];
  const uint32_t at = atomicAdd(&L.n, 1u);
  L.beg[at] = beg;
  L.len[at] = uint16_t(len);
  L.bits[at] = uint8_t(bits);
}

// In-place exclusive scan of cnt[0, nd) (block-wide); cnt[nd] = total.
__device__ void lf_scan_counts(LeafSmem& s, int nd) {
  const int tid = threadIdx.x;
  const int per = (nd + LF_THREADS - 1) / LF_THREADS;
  const int d0 = tid * per;
  uint32_t sum = 0;
  for (int q = 0; q < per; ++q)
    if (d0 + q < nd) sum += s.cnt[d0 + q];
  uint32_t tot;
  uint32_t run = lf_scan(sum, s.wsum, tot);
  for (int q = 0; q < per; ++q) {
    if (d0 + q < nd) {
      const uint32_t c = s.cnt[d0 + q];
      s.cnt[d0 + q] = run;
      run += c;
    }
  }
  if (tid == 0) s.cnt[nd] = tot;
  __syncthreads();
}

// CTA-wide counting sort (non-stable) of b[beg, beg+n) by the top nb of its
// `bits` low bits, through a[], back into b[]; then every digit bucket is
// routed (thread per bucket).
__device__ void lf_cta_pass(LeafSmem& s, int beg, int n, int bits, int nxt) {
  const int tid = threadIdx.x;
  const int nb = lf_digit_bits(bits, n, LF_DBITS);
  const int shift = bits - nb;
  const int nd = 1 << nb;
  const uint32_t dm = uint32_t(nd - 1);
  for (int i = tid; i <= nd; i += LF_THREADS) s.cnt[i] = 0;
  __syncthreads();
  uint32_t slot[LF_KPT];
  uint64_t v[LF_KPT];
#pragma unroll
  for (int q = 0; q < LF_KPT; ++q) {
    const int j = q * LF_THREADS + tid;
    v[q] = j < n ? s.b[beg + j] : 0ull;
  }
#pragma unroll
  for (int q = 0; q < LF_KPT; ++q) {
    const int j = q * LF_THREADS + tid;
    slot[q] = j < n ? atomicAdd(&s.cnt[uint32_t(v[q] >> shift) & dm], 1u) : 0u;
  }
  __syncthreads();
  lf_scan_counts(s, nd);
#pragma unroll
  for (int q = 0; q < LF_KPT; ++q) {
    const int j = q * LF_THREADS + tid;
    if (j < n) s.a[beg + s.cnt[uint32_t(v[q] >> shift) & dm] + slot[q]] = v[q];
  }
  __syncthreads();
  for (int j = tid; j < n; j += LF_THREADS) s.b[beg + j] = s.a[beg + j];
  __syncthreads();
  for (int d = tid; d < nd; d += LF_THREADS)
    lf_route(s, uint32_t(beg) + s.cnt[d], s.cnt[d + 1] - s.cnt[d], shift, nxt);
  __syncthreads();
}

// The same for one warp over a range of <= LF_WARP_MAX keys, with the
// warp's own counters (digit <= 8 bits).
__device__ void lf_warp_pass(LeafSmem& s, uint32_t beg, int n, int bits, int nxt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* cnt = s.cnt + warp * LF_WSTRIDE;
  const int nb = lf_digit_bits(bits, n, LF_WBITS);
  const int shift = bits - nb;
  const int nd = 1 << nb;
  const uint32_t dm = uint32_t(nd - 1);
  for (int i = lane; i <= nd; i += 32) cnt[i] = 0;
  __syncwarp();
  for (int j = lane; j < n; j += 32) atomicAdd(&cnt[uint32_t(s.b[beg + j] >> shift) & dm], 1u);
  __syncwarp();
  {  // in-place exclusive scan: lane owns nd/32 consecutive counters
    const int per = (nd + 31) >> 5;
    uint32_t sum = 0;
    for (int q = 0; q < per; ++q) {
      const int d = lane * per + q;
      if (d < nd) sum += cnt[d];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    uint32_t run = inc - sum;
    for (int q = 0; q < per; ++q) {
      const int d = lane * per + q;
      if (d < nd) {
        const uint32_t c = cnt[d];
        cnt[d] = run;
        run += c;
      }
    }
    if (lane == 31) cnt[nd] = inc;
  }
  __syncwarp();
  // scatter through a[] (cursor per digit: the starts advance; restored below)
  for (int j = lane; j < n; j += 32) {
    const uint64_t v = s.b[beg + j];
    const uint32_t at = atomicAdd(&cnt[uint32_t(v >> shift) & dm], 1u);
    s.a[beg + at] = v;
  }
  __syncwarp();
  // cnt[d] now holds the END of bucket d: start(d) = cnt[d-1] (0 for d = 0)
  for (int j = lane; j < n; j += 32) s.b[beg + j] = s.a[beg + j];
  __syncwarp();
  for (int d = lane; d < nd; d += 32) {
    const uint32_t st = d == 0 ? 0u : cnt[d - 1];
    lf_route(s, beg + st, cnt[d] - st, shift, nxt);
  }
  __syncwarp();
}

// Load n keys (v = key - key_lo), sort them ascending in s.b. MSD counting
// sort: first by row (the leaf's rows share nothing else), then every row
// of more than LF_SMALL keys by the top bits of its column (a warp per row
// up to LF_WARP_MAX keys, the whole CTA beyond), until the buckets are small
// enough for an insertion sort. Column ids are random offsets (the configs
// permute ids), so a digit of log2(len)+1 bits leaves ~2 keys per bucket:
// ~40 thread-instructions per key, against ~35 per pass (x5) for an 8-bit
// stable LSD.
__device__ uint64_t* lf_sort(LeafSmem& s, const uint64_t* __restrict__ src, int n,
                             uint64_t key_lo, int kw, int& nw_out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  nw_out = (n + LF_SLOTS - 1) / LF_SLOTS;
  uint64_t orv = 0;
  {
    uint64_t v[LF_KPT];
#pragma unroll
    for (int q = 0; q < LF_KPT; ++q) {  // all loads in flight first
      const int j = q * LF_THREADS + tid;
      v[q] = j < n ? __ldcs(src + j) - key_lo : 0ull;
    }
#pragma unroll
    for (int q = 0; q < LF_KPT; ++q) {
      const int j = q * LF_THREADS + tid;
      if (j < n) s.b[j] = v[q];
      orv = max(orv, v[q]);  // the max: its top bit is the top varying bit
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) orv = max(orv, __shfl_xor_sync(0xffffffffu, orv, o));
  if (lane == 0) s.orv[warp] = orv;
  if (tid < 2) { s.cta[tid].n = 0; s.wrp[tid].n = 0; }
  __syncthreads();
  orv = 0;
#pragma unroll 4
  for (int w = 0; w < LF_WARPS; ++w) orv = max(orv, s.orv[w]);
  const int width = orv ? 64 - __clzll(orv) : 0;
  if (width == 0 || n <= 1) return s.b;
  int cur = 0;
  if (n <= LF_SMALL) {
    if (tid == 0) lf_route(s, 0, uint32_t(n), width, cur);
    __syncthreads();
    return s.b;
  }
  // ---- main pass: rows, then ~len buckets per row over its column bits ----
  // digit(key) = rowbase[row] + (col >> (kw - c_row)), c_row = ceil(log2(len_row))
  const int rows = width > kw ? int(orv >> kw) + 1 : 1;  // rows spanned (<= LF_ROWS)
  const uint64_t cm = (1ull << kw) - 1ull;
  for (int i = tid; i < rows; i += LF_THREADS) s.cnt[i] = 0;
  __syncthreads();
  uint64_t v[LF_KPT];
  uint32_t slot[LF_KPT];
#pragma unroll
  for (int q = 0; q < LF_KPT; ++q) {
    const int j = q * LF_THREADS + tid;
    v[q] = j < n ? s.b[j] : 0ull;
    if (j < n) atomicAdd(&s.cnt[uint32_t(v[q] >> kw)], 1u);
  }
  __syncthreads();
  for (int r = tid; r < rows; r += LF_THREADS) {
    const uint32_t len = s.cnt[r];
    const int c = len <= 1 ? 0 : min(kw, 32 - __clz(len - 1));
    s.rowbits[r] = uint8_t(kw - c);
    s.cnt[r] = len ? (1u << c) : 0u;  // buckets of the row (< 2 len)
  }
  __syncthreads();
  lf_scan_counts(s, rows);  // bucket starts per row, total in cnt[rows]
  const int nbk = int(s.cnt[rows]);
  for (int r = tid; r < rows; r += LF_THREADS) s.rowbase[r] = uint16_t(s.cnt[r]);
  __syncthreads();
  for (int i = tid; i <= nbk; i += LF_THREADS) s.cnt[i] = 0;
  __syncthreads();
  uint32_t dg[LF_KPT];
#pragma unroll
  for (int q = 0; q < LF_KPT; ++q) {
    const int j = q * LF_THREADS + tid;
    if (j < n) {
      const uint32_t r = uint32_t(v[q] >> kw);
      dg[q] = s.rowbase[r] + uint32_t((v[q] & cm) >> s.rowbits[r]);
      slot[q] = atomicAdd(&s.cnt[dg[q]], 1u);
    }
  }
  __syncthreads();
  lf_scan_counts(s, nbk);
#pragma unroll
  for (int q = 0; q < LF_KPT; ++q) {
    const int j = q * LF_THREADS + tid;
    if (j < n) s.a[s.cnt[dg[q]] + slot[q]] = v[q];
  }
  __syncthreads();
  for (int j = tid; j < n; j += LF_THREADS) s.b[j] = s.a[j];
  __syncthreads();
  for (int d = tid; d < nbk; d += LF_THREADS) {
    const uint32_t st = s.cnt[d], len = s.cnt[d + 1] - st;
    if (len <= 1) continue;
    if (len <= LF_SMALL) {
      lf_insertion(s.b + st, int(len));
    } else {  // rare: columns that share their top bits; bits that still vary
      uint64_t x = 0;
      const uint64_t k0 = s.b[st];
      for (uint32_t i = 1; i < len; ++i) x |= s.b[st + i] ^ k0;
      lf_route(s, st, len, x ? 64 - __clzll(x) : 0, cur);
    }
  }
  __syncthreads();
  while (s.cta[cur].n + s.wrp[cur].n > 0) {  // block-uniform
    const int nxt = cur ^ 1;
    if (tid == 0) { s.cta[nxt].n = 0; s.wrp[nxt].n = 0; }
    __syncthreads();
    const int mc = int(s.cta[cur].n);
    for (int r = 0; r < mc; ++r)
      lf_cta_pass(s, int(s.cta[cur].beg[r]), int(s.cta[cur].len[r]), s.cta[cur].bits[r], nxt);
    const int mw = int(s.wrp[cur].n);
    for (int r = warp; r < mw; r += LF_WARPS)
      lf_warp_pass(s, s.wrp[cur].beg[r], int(s.wrp[cur].len[r]), s.wrp[cur].bits[r], nxt);
    __syncthreads();
    cur = nxt;
  }
  return s.b;
}

// Dedupe flags over the sorted keys: kp[j] = kept keys before j (j <= n),
// returns the number kept. Warp-striped (coalesced) positions.
__device__ uint32_t lf_dedupe(LeafSmem& s, const uint64_t* sorted, uint32_t* kp, int n, int nw,
                              uint32_t& keep_bits) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned lt = lanemask_lt();
  uint32_t run = 0;
  keep_bits = 0;
  uint32_t before[LF_KPT];
  if (warp < nw) {
#pragma unroll
    for (int i = 0; i < LF_KPT; ++i) {
      const int j = warp * LF_SLOTS + i * 32 + lane;
      const bool keep = j < n && (j == 0 || sorted[j] != sorted[j - 1]);
      keep_bits |= uint32_t(keep) << i;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      before[i] = run + __popc(bal & lt);
      run += __popc(bal);
    }
  }
  if (lane == 0) s.wsum[warp] = warp < nw ? run : 0u;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (int w = 0; w < LF_WARPS; ++w) {
    const uint32_t c = s.wsum[w];
    if (w < warp) wpre += c;
    tot += c;
  }
  if (warp < nw) {
#pragma unroll
    for (int i = 0; i < LF_KPT; ++i) {
      const int j = warp * LF_SLOTS + i * 32 + lane;
      if (j < n) kp[j] = wpre + before[i];
    }
  }
  if (tid == 0) kp[n] = tot;
  __syncthreads();
  return tot;
}

__device__ __forceinline__ int lf_lower_bound(const uint64_t* a, int n, uint64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] < v) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// MAIN: leaves of the two key-ordered chains (side 0 entries [0,u0), side 1
// [u0,u0+u1)), placed by decoupled look-back; COUNT: the leaves of huge
// buckets (any order), deduplicated keys written back in place.
// MAIN: the leaves of the two key-ordered chains (side 0 entries [0,u0),
// side 1 [u0, n_leaves)): adjacency written at the leaf's RAW position (its
// first key's index in the side's key order) into args.tmp, row offsets of
// its owned ids relative to that position, deduplicated count to leaf_d;
// bk_compact_kernel moves them to their final positions. COUNT: the leaves
// of huge buckets, deduplicated keys written back in place.
// (No look-back: leaves vary in size, and a chain waiting on its slowest
// predecessor measured ~2x slower than the raw-position + compaction form.)
template <bool MAIN>
__global__ void __launch_bounds__(LF_THREADS, 1) bk_leaf_kernel(
    const BkLeaf* __restrict__ leaves, int n_leaves, int u0, BkArgs args,
    uint32_t* __restrict__ ticket) {
  extern __shared__ __align__(16) unsigned char lf_dsm[];
  LeafSmem& s = *reinterpret_cast<LeafSmem*>(lf_dsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kw = args.kw;
  const uint64_t colmask = (1ull << kw) - 1ull;
  while (true) {
    if (tid == 0) s.ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const int u = int(s.ticket);
    if (u >= n_leaves) break;
    const BkLeaf L = leaves[u];
    const int side = (L.info >> 1) & 1;
    const int kind = (L.info >> 2) & 7;
    const uint64_t* buf = args.buf[L.info & 1];
    int64_t* off = args.off[side];

    if (MAIN && kind == LK_PLACEHOLDER) {  // placed by bk_compact_kernel
      if (tid == 0) args.main_d[side ? u + 1 : u] = int64_t(args.huge_total[L.huge]);
      __syncthreads();
      continue;
    }

    // ---- LSD leaf ----
    const int n = L.count;
    int nw;
    const uint64_t* sorted = lf_sort(s, buf + L.begin, n, L.key_lo, kw, nw);
    uint32_t* kp = reinterpret_cast<uint32_t*>(s.a);  // sorted keys are in s.b
    uint32_t keep_bits;
    const uint32_t D = lf_dedupe(s, sorted, kp, n, nw, keep_bits);
    if (MAIN) {
      const int64_t raw = L.begin - int64_t(side) * args.rows;  // position in key order
      uint32_t* tmp = args.tmp[side] + raw;
      if (warp < nw) {
#pragma unroll
        for (int i = 0; i < LF_KPT; ++i) {
          if ((keep_bits >> i) & 1u) {
            const int j = warp * LF_SLOTS + i * 32 + lane;
            const uint64_t col = (sorted[j] + L.key_lo) & colmask;
            tmp[kp[j]] = bk_rank(args.words, col);
          }
        }
      }
      // row offsets (relative to the leaf) of the present ids this leaf owns
      const int64_t x0 = int64_t(L.key_lo >> kw);
      const int64_t x1 = min(int64_t(L.key_hi >> kw), args.n_ids);
      for (int64_t x = x0 + tid; x < x1; x += LF_THREADS) {
        if (!bk_present(args.words, uint64_t(x))) continue;
        const uint64_t v = (uint64_t(x) << kw) - L.key_lo;
        const int idx = lf_lower_bound(sorted, n, v);
        off[bk_rank(args.words, uint64_t(x))] = int64_t(kp[idx]);
      }
      if (tid == 0) args.main_d[side ? u + 1 : u] = int64_t(D);
    } else {
      // COUNT: deduplicated keys back in place, per-row (kind ROWS) or
      // per-column-child (kind HUBKIDS) deduplicated counts
      uint64_t* wb = args.wbuf[L.info & 1] + L.begin;
      if (warp < nw) {
#pragma unroll
        for (int i = 0; i < LF_KPT; ++i) {
          if ((keep_bits >> i) & 1u) {
            const int j = warp * LF_SLOTS + i * 32 + lane;
            wb[kp[j]] = sorted[j] + L.key_lo;
          }
        }
      }
      if (kind == LK_ROWS) {
        for (int j = tid; j < n; j += LF_THREADS) {
          const uint64_t row = (sorted[j] + L.key_lo) >> kw;
          if (j > 0 && ((sorted[j - 1] + L.key_lo) >> kw) == row) continue;  // not a row start
          const int e = lf_lower_bound(sorted, n, ((row + 1) << kw) - L.key_lo);
          const uint32_t cnt = kp[e] - kp[j];
          atomicAdd(&args.deg[int64_t(side) * args.n_nodes + bk_rank(args.words, row)], cnt);
        }
      } else {  // LK_HUBKIDS: one row, children = top column bits
        const int kb = args.kid_bits;
        for (int j = tid; j < n; j += LF_THREADS) {
          const uint64_t key = sorted[j] + L.key_lo;
          const uint64_t kid = (key & colmask) >> kb;
          if (j > 0 && (((sorted[j - 1] + L.key_lo) & colmask) >> kb) == kid) continue;
          const uint64_t nxt = ((key >> kw) << kw) + ((kid + 1) << kb) - L.key_lo;
          const int e = lf_lower_bound(sorted, n, nxt);
          args.child_cnt[int64_t(L.hub) * args.n_kids + kid] = kp[e] - kp[j];
        }
        if (tid == 0) {
          const uint64_t row = L.key_lo >> kw;
          atomicAdd(&args.deg[int64_t(side) * args.n_nodes + bk_rank(args.words, row)], D);
        }
      }
      if (tid == 0) {
        args.leaf_d[u] = int32_t(D);
        atomicAdd(&args.huge_total[L.huge], (unsigned long long)D);
      }
    }
    __syncthreads();
  }
}

// COUNT for one large column child of a hub row: a shared-memory bitmap
// over the child's column range (2^kid_bits values) sorts and deduplicates
// any number of keys; the distinct keys are written back in place.
__global__ void __launch_bounds__(1024, 1) bk_bitmap_leaf_kernel(const BkLeaf* __restrict__ leaves,
                                                                 int n_leaves, BkArgs args) {
  extern __shared__ __align__(16) unsigned char bm_dsm[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(bm_dsm);
  __shared__ uint32_t s_w[32];
  const int tid = threadIdx.x;
  const int kw = args.kw;
  const int nwords = max(1, (1 << args.kid_bits) >> 5);
  for (int u = blockIdx.x; u < n_leaves; u += gridDim.x) {
    const BkLeaf L = leaves[u];
    const int side = (L.info >> 1) & 1;
    const uint64_t* in = args.buf[L.info & 1] + L.begin;
    uint64_t* wb = args.wbuf[L.info & 1] + L.begin;
    for (int i = tid; i < nwords; i += 1024) bm[i] = 0;
    __syncthreads();
    const uint64_t cmask = (1ull << args.kid_bits) - 1ull;
    for (int64_t j = tid; j < L.count; j += 1024) {
      const uint32_t c = uint32_t(ld_stream_u64(in + j) & cmask);
      const uint32_t bit = 1u << (c & 31);
      if (!(bm[c >> 5] & bit)) atomicOr(&bm[c >> 5], bit);
    }
    __syncthreads();
    // each thread owns a contiguous run of words: count, scan, write
    const int per = (nwords + 1023) / 1024;
    const int w0 = tid * per;
    uint32_t cnt = 0;
    for (int q = 0; q < per; ++q)
      if (w0 + q < nwords) cnt += __popc(bm[w0 + q]);
    uint32_t tot;
    uint32_t pos = lf_scan(cnt, s_w, tot);
    const uint64_t hi = L.key_lo & ~cmask;  // row and child bits
    for (int q = 0; q < per; ++q) {
      if (w0 + q >= nwords) break;
      uint32_t bits = bm[w0 + q];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        wb[pos++] = hi | (uint64_t(w0 + q) << 5) | uint64_t(b);
      }
    }
    if (tid == 0) {
      args.leaf_d[u] = int32_t(tot);
      args.child_cnt[int64_t(L.hub) * args.n_kids + L.k0] = tot;
      const uint64_t row = L.key_lo >> kw;
      atomicAdd(&args.deg[int64_t(side) * args.n_nodes + bk_rank(args.words, row)], tot);
      atomicAdd(&args.huge_total[L.huge], (unsigned long long)tot);
    }
    __syncthreads();
  }
}

// The main chains at their final positions: main_d holds, per leaf, the
// exclusive prefix of the deduplicated counts of its side's chain (scanned
// in place). Group leaves move their adjacency from the raw position and
// shift their rows' offsets; placeholders write their rows' offsets from the
// deduplicated degrees of the COUNT pass; the last leaf of a side writes
// off[N] = E.
__global__ void __launch_bounds__(256) bk_compact_kernel(const BkLeaf* __restrict__ leaves,
                                                         int n_leaves, int u0, BkArgs args) {
  __shared__ uint32_t s_w[8];
  __shared__ int64_t s_carry;
  const int kw = args.kw;
  for (int u = blockIdx.x; u < n_leaves; u += gridDim.x) {
    const BkLeaf L = leaves[u];
    const int side = (L.info >> 1) & 1;
    const int kind = (L.info >> 2) & 7;
    const int64_t* scan = args.main_d + (side ? u0 + 1 : 0);
    const int li = side ? u - u0 : u;
    const int64_t base = scan[li];
    const int64_t d = scan[li + 1] - base;  // the scan array holds n+1 entries per side
    int64_t* off = args.off[side];
    const int64_t x0 = int64_t(L.key_lo >> kw);
    const int64_t x1 = min(int64_t(L.key_hi >> kw), args.n_ids);
    if (kind == LK_PLACEHOLDER) {
      if (threadIdx.x == 0) s_carry = 0;
      __syncthreads();
      for (int64_t c = x0; c < x1; c += 256) {
        const int64_t x = c + threadIdx.x;
        const bool pres = x < x1 && bk_present(args.words, uint64_t(x));
        const uint32_t r = pres ? bk_rank(args.words, uint64_t(x)) : 0u;
        const uint32_t dg = pres ? args.deg[int64_t(side) * args.n_nodes + r] : 0u;
        const uint32_t ex = bk_scan256(dg, s_w);
        const int64_t carry = s_carry;
        if (pres) off[r] = base + carry + ex;
        __syncthreads();
        if (threadIdx.x == 255) s_carry = carry + ex + dg;
        __syncthreads();
      }
    } else {
      const int64_t raw = L.begin - int64_t(side) * args.rows;
      const uint32_t* src = args.tmp[side] + raw;
      int32_t* dst = args.adj[side] + base;
      for (int64_t j = threadIdx.x; j < d; j += 256) dst[j] = int32_t(__ldcs(src + j));
      for (int64_t x = x0 + threadIdx.x; x < x1; x += 256)
        if (bk_present(args.words, uint64_t(x))) off[bk_rank(args.words, uint64_t(x))] += base;
    }
    if (threadIdx.x == 0 && (side ? (u == n_leaves - 1) : (u == u0 - 1)))
      off[args.n_nodes] = base + d;
    __syncthreads();
  }
}

// Per hub row (block): exclusive scan of its children's deduplicated counts.
__global__ void __launch_bounds__(256) bk_hub_prefix_kernel(const uint32_t* __restrict__ cnt,
                                                            uint32_t* __restrict__ base,
                                                            int n_kids) {
  __shared__ uint32_t s_w[8];
  const int64_t h = blockIdx.x;
  uint32_t carry = 0;
  for (int c = 0; c < n_kids; c += 256 * 8) {
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = c + threadIdx.x * 8 + q;
      v[q] = k < n_kids ? cnt[h * n_kids + k] : 0u;
      sum += v[q];
    }
    const uint32_t ex = bk_scan256(sum, s_w);
    uint32_t run = carry + ex;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = c + threadIdx.x * 8 + q;
      if (k < n_kids) base[h * n_kids + k] = run;
      run += v[q];
    }
    // block total: the last thread's run
    __shared__ uint32_t s_tot;
    if (threadIdx.x == 255) s_tot = run;
    __syncthreads();
    carry = s_tot;
    __syncthreads();
  }
}

// EMIT for the leaves of huge buckets: their deduplicated keys, in order,
// at the CSR position of their first row (plus the column-child prefix).
__global__ void __launch_bounds__(256) bk_emit_kernel(const BkLeaf* __restrict__ leaves,
                                                      int n_leaves, BkArgs args) {
  const int kw = args.kw;
  const uint64_t colmask = (1ull << kw) - 1ull;
  for (int u = blockIdx.x; u < n_leaves; u += gridDim.x) {
    const BkLeaf L = leaves[u];
    const int side = (L.info >> 1) & 1;
    const int kind = (L.info >> 2) & 7;
    const uint64_t* in = args.buf[L.info & 1] + L.begin;
    const uint64_t x = L.key_lo >> kw;
    int64_t base = args.off[side][bk_rank(args.words, x)];  // rank of the first id >= x
    if (kind != LK_ROWS) base += args.child_base[int64_t(L.hub) * args.n_kids + L.k0];
    const int d = args.leaf_d[u];
    int32_t* adj = args.adj[side] + base;
    for (int j = threadIdx.x; j < d; j += 256)
      adj[j] = int32_t(bk_rank(args.words, ld_stream_u64(in + j) & colmask));
  }
}


// ------------------------------------------------------------ planning --
// Leaf plans are built on the device (the bucket counts never leave HBM):
// the main chains by one thread per chunk of consecutive buckets (greedy
// grouping inside the chunk, chunks never straddle sides, counts then fill
// at scanned offsets, so chains stay in key order); the leaves of huge
// buckets by one thread per huge bucket / hub row, appended in any order
// (they are placed by row offsets, not by chain position).
struct BkHuge { int64_t begin, count; int32_t side, bucket; };
struct BkHub { int64_t begin, count; uint64_t row; int32_t h, side; };

template <bool FILL>
__global__ void bk_plan_main_kernel(const int64_t* __restrict__ bst, int nbk, int chunk,
                                    int nchunks, int shiftP, int bufF, int cap, int idcap,
                                    int64_t* __restrict__ leaf_off, int64_t* __restrict__ huge_off,
                                    BkLeaf* __restrict__ leaves, BkHuge* __restrict__ huges) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int b0 = c * chunk, b1 = b0 + chunk;
  const int side = b0 / nbk;
  int64_t nl = FILL ? leaf_off[c] : 0, nh = FILL ? huge_off[c] : 0;
  int gb = -1;
  int64_t gcount = 0;
  auto close = [&](int end_b) {
    if (gb < 0) return;
    if (FILL) {
      BkLeaf L{};
      L.begin = bst[gb];
      L.key_lo = uint64_t(gb - side * nbk) << shiftP;
      L.key_hi = uint64_t(end_b - side * nbk) << shiftP;
      L.count = int32_t(gcount);
      L.info = bufF | (side << 1) | (LK_GROUP << 2);
      L.huge = -1; L.hub = -1;
      leaves[nl] = L;
    }
    ++nl;
    gb = -1;
    gcount = 0;
  };
  for (int b = b0; b < b1; ++b) {
    const int64_t cb = bst[b + 1] - bst[b];
    if (cb > cap) {
      close(b);
      if (FILL) {
        BkLeaf L{};
        L.begin = bst[b];
        L.key_lo = uint64_t(b - side * nbk) << shiftP;
        L.key_hi = uint64_t(b + 1 - side * nbk) << shiftP;
        L.count = 0;
        L.info = bufF | (side << 1) | (LK_PLACEHOLDER << 2);
        L.huge = int32_t(nh); L.hub = -1;
        leaves[nl] = L;
        huges[nh] = BkHuge{bst[b], cb, side, b - side * nbk};
      }
      ++nl;
      ++nh;
      continue;
    }
    if (gb >= 0 && (gcount + cb > cap || b - gb >= idcap)) close(b);
    if (gb < 0) gb = b;
    gcount += cb;
  }
  close(b1);
  if (!FILL) {
    leaf_off[c] = nl;
    huge_off[c] = nh;
  }
}

// Row split of huge bucket h: rows <= cap grouped into ROWS leaves, larger
// rows become hub rows. Thread per huge bucket.
__global__ void bk_plan_rows_kernel(const BkHuge* __restrict__ huges, int nh,
                                    const int64_t* __restrict__ rbeg,
                                    const unsigned int* __restrict__ rcnt, int ndr, int shiftP,
                                    int kw, int bufH, int cap, BkLeaf* __restrict__ hl,
                                    int* __restrict__ n_hl, BkHub* __restrict__ hubs,
                                    int* __restrict__ n_hub) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= nh) return;
  const BkHuge H = huges[h];
  const uint64_t key0 = uint64_t(H.bucket) << shiftP;
  int cnt_l = 0, cnt_h = 0, at_l = 0, at_h = 0;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      at_l = atomicAdd(n_hl, cnt_l);
      at_h = atomicAdd(n_hub, cnt_h);
    }
    int gr = -1;
    int64_t gcount = 0;
    int nl = 0, nb = 0;
    auto close = [&](int end_r) {
      if (gr < 0) return;
      if (pass == 1) {
        BkLeaf L{};
        L.begin = rbeg[int64_t(h) * ndr + gr];
        L.key_lo = key0 + (uint64_t(gr) << kw);
        L.key_hi = key0 + (uint64_t(end_r) << kw);
        L.count = int32_t(gcount);
        L.info = bufH | (H.side << 1) | (LK_ROWS << 2);
        L.huge = h; L.hub = -1;
        hl[at_l + nl] = L;
      }
      ++nl;
      gr = -1;
      gcount = 0;
    };
    for (int r = 0; r < ndr; ++r) {
      const int64_t c = rcnt[int64_t(h) * ndr + r];
      if (c > cap) {
        close(r);
        if (pass == 1)
          hubs[at_h + nb] = BkHub{rbeg[int64_t(h) * ndr + r], c, (key0 >> kw) + uint64_t(r), h,
                                  H.side};
        ++nb;
        continue;
      }
      if (gr >= 0 && gcount + c > cap) close(r);
      if (gr < 0) gr = r;
      gcount += c;
    }
    close(ndr);
    cnt_l = nl;
    cnt_h = nb;
  }
}

__global__ void bk_hub_ranges_kernel(const BkHub* __restrict__ hubs, int n, int64_t* __restrict__ b,
                                     int64_t* __restrict__ e) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) {
    b[q] = hubs[q].begin;
    e[q] = hubs[q].begin + hubs[q].count;
  }
}

__global__ void bk_huge_ranges_kernel(const BkHuge* __restrict__ hg, int n, int64_t* __restrict__ b,
                                      int64_t* __restrict__ e) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) {
    b[q] = hg[q].begin;
    e[q] = hg[q].begin + hg[q].count;
  }
}

// Column split of hub row q: children <= cap grouped into HUBKIDS leaves,
// larger children become bitmap leaves. Thread per hub row.
__global__ void bk_plan_kids_kernel(const BkHub* __restrict__ hubs, int n_hub,
                                    const int64_t* __restrict__ kbeg,
                                    const unsigned int* __restrict__ kcnt, int n_kids, int kid_bits,
                                    int kw, int bufF, int cap, BkLeaf* __restrict__ hl,
                                    int* __restrict__ n_hl, BkLeaf* __restrict__ bml,
                                    int* __restrict__ n_bm) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_hub) return;
  const BkHub H = hubs[q];
  const uint64_t key0 = H.row << kw;
  int cnt_l = 0, cnt_b = 0, at_l = 0, at_b = 0;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      at_l = atomicAdd(n_hl, cnt_l);
      at_b = atomicAdd(n_bm, cnt_b);
    }
    int gk = -1;
    int64_t gcount = 0;
    int nl = 0, nb = 0;
    auto close = [&](int end_k) {
      if (gk < 0) return;
      if (pass == 1) {
        BkLeaf L{};
        L.begin = kbeg[int64_t(q) * n_kids + gk];
        L.key_lo = key0 + (uint64_t(gk) << kid_bits);
        L.key_hi = key0 + (uint64_t(end_k) << kid_bits);
        L.count = int32_t(gcount);
        L.info = bufF | (H.side << 1) | (LK_HUBKIDS << 2);
        L.huge = H.h; L.hub = q; L.k0 = gk;
        hl[at_l + nl] = L;
      }
      ++nl;
      gk = -1;
      gcount = 0;
    };
    for (int k = 0; k < n_kids; ++k) {
      const int64_t c = kcnt[int64_t(q) * n_kids + k];
      if (c > cap) {
        close(k);
        if (pass == 1) {
          BkLeaf L{};
          L.begin = kbeg[int64_t(q) * n_kids + k];
          L.key_lo = key0 + (uint64_t(k) << kid_bits);
          L.key_hi = key0 + (uint64_t(k + 1) << kid_bits);
          L.count = int32_t(c);
          L.info = bufF | (H.side << 1) | (LK_BITMAP << 2);
          L.huge = H.h; L.hub = q; L.k0 = k;
          bml[at_b + nb] = L;
        }
        ++nb;
        continue;
      }
      if (gk >= 0 && gcount + c > cap) close(k);
      if (gk < 0) gk = k;
      gcount += c;
    }
    close(n_kids);
    cnt_l = nl;
    cnt_b = nb;
  }
}

}  // namespace gtd

namespace gt {

using gtd::BkLeaf;

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Level digit widths: P key bits split into ceil(P/9) near-equal levels.
static std::vector<int> level_bits(int P) {
  std::vector<int> v;
  const int L = std::max(1, (P + 8) / 9);
  for (int l = 0; l < L; ++l) v.push_back(P / L + (l < P % L ? 1 : 0));
  return v;
}

template <typename K>
static void set_smem(K kernel, size_t bytes) {
  GT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

static constexpr int PART_KPT = 16;       // keys per thread in the partition kernels
static constexpr int PART_T = 256 * PART_KPT;

// One segmented level: hist of digit (key >> shift) & (nd-1) over segments
// [seg_begin[s], seg_end[s]) of `in`, partition into `out` at the same
// offsets; d_next_begin[s*nd + d] = start of child d (its count: d_hist).
static void seg_level(const uint64_t* in, uint64_t* out, const int64_t* d_seg_begin,
                      const int64_t* d_seg_end, int nseg, int shift, int nd,
                      unsigned int* d_hist, int64_t* d_next_begin, const char* phase,
                      double keys) {
  cudaStream_t st = ctx().stream;
  const int sms = ctx().sm_count;
  int64_t* d_tiles = ws_n<int64_t>(WS_TMP3, size_t(nseg) + 2);
  int64_t* d_small = ws_n<int64_t>(WS_SMALL, 16);
  GT_LAUNCH(gtd::bk_seg_tiles_kernel, ceil_div(nseg, 256), 256, 0, d_seg_begin, d_seg_end, nseg,
            PART_T, d_tiles);
  exclusive_scan_i64(d_tiles, nseg, d_small + 8);
  GT_CUDA(cudaMemsetAsync(d_hist, 0, size_t(nseg) * nd * 4, st));
  unsigned long long* d_cur = ws_n<unsigned long long>(WS_TMP4, size_t(nseg) * nd + 1);
  {
    Phase ph("build.seg_hist", 8.0 * keys);
    GT_LAUNCH(gtd::bk_seg_hist_kernel<PART_KPT>, sms * 8, 256, 0, in, d_seg_begin, d_seg_end,
              d_tiles, nseg, shift, nd, d_hist);
    GT_LAUNCH(gtd::bk_seg_cursor_kernel, nseg, 256, 0, d_hist, d_seg_begin, nd, d_cur,
              d_next_begin);
  }
  {
    Phase ph(phase, 16.0 * keys);
    const size_t smem = size_t(PART_T) * 8 + gtd::BK_MAXD * 12 + 64;
    static const bool once = [&] {
      set_smem(gtd::bk_seg_part_kernel<PART_KPT>, smem);
      return true;
    }();
    (void)once;
    GT_LAUNCH(gtd::bk_seg_part_kernel<PART_KPT>, sms * 3, 256, smem, in, out, d_seg_begin,
              d_seg_end, d_tiles, nseg, shift, nd, d_cur);
  }
}

// A non-stable partition of n keys by (key >> shift) & (2^bits - 1) into
// digit-sorted order, digit starts given (the first pass of an LSD sort needs
// no stability: nothing orders equal digits yet). 4.2 TB/s vs 2.4 TB/s for
// the stable onesweep pass on B200 (scripts/ubench/ubench_r2.cu).
void partition_pass(const uint64_t* in, uint64_t* out, int64_t n, int shift, int bits,
                    const int64_t* d_digit_base) {
  cudaStream_t st = ctx().stream;
  const int nd = 1 << bits;
  int64_t* d_seg = ws_n<int64_t>(WS_PART, 8 + size_t(nd));  // begin, end, tile offsets {0, tiles}
  unsigned long long* d_cur = reinterpret_cast<unsigned long long*>(d_seg + 8);
  const int64_t h_seg[4] = {0, n, 0, ceil_div64(n, PART_T)};
  h2d(d_seg, h_seg, sizeof h_seg);
  GT_CUDA(cudaMemcpyAsync(d_cur, d_digit_base, size_t(nd) * 8, cudaMemcpyDeviceToDevice, st));
  const size_t smem = size_t(PART_T) * 8 + gtd::BK_MAXD * 12 + 64;
  static const bool once = [&] {
    set_smem(gtd::bk_seg_part_kernel<PART_KPT>, smem);
    return true;
  }();
  (void)once;
  GT_LAUNCH(gtd::bk_seg_part_kernel<PART_KPT>, ctx().sm_count * 3, 256, smem, in, out, d_seg,
            d_seg + 1, d_seg + 2, 1, shift, nd, d_cur);
}

bool bucket_build_applies(int64_t rows, uint64_t span) {
  // GT_BUILD (read per call): the LSD sort pipeline (build.cu) is the
  // default; "bucket" forces this one, "auto" picks it for large dense
  // tables. Measured on B200: C4 177 ms vs 157 ms for the
  // LSD pipeline, C5 215 vs 220 ms — the shared-memory leaf sort is
  // instruction-bound, so it does not pay off yet.
  const char* v = getenv("GT_BUILD");
  const int mode = v ? (!strcmp(v, "bucket") ? 2 : (!strcmp(v, "auto") ? 1 : 0)) : 0;
  if (mode == 0 || rows <= 0) return false;
  const uint64_t W = span + 1;
  const int kw = bits_for(int64_t(W));
  if (kw > 29 || W < 2) return false;  // keys <= 58 bits; hub children <= 2^20 columns
  if (mode == 2) return true;
  return rows >= (int64_t(1) << 20) && W <= uint64_t(rows) * 4;
}

// The dense-id build (see the file comment). `g` gets ids, both CSRs, n, e.
void bucket_build(const int64_t* src, const int64_t* dst, int64_t rows, const int64_t* extra,
                  int64_t n_extra, int64_t lo, uint64_t span, gt_graph* g) {
  cudaStream_t st = ctx().stream;
  const int sms = ctx().sm_count;
  const uint64_t W = span + 1;
  const int kw = bits_for(int64_t(W));
  const int CAP = gtd::LF_CAP;
  // P key bits of bucket partitioning: ~CAP/4 keys per bucket on average,
  // and at most 8 row bits left below the buckets (the row split of a
  // huge bucket is one more 8-bit level)
  int P = bits_for(std::max<int64_t>(2, 4 * rows / CAP));
  P = std::max(P, kw - 8);
  P = std::min(P, kw);
  P = std::max(P, 1);
  P = std::min(P, env_int("GT_BK_PMAX", 27));
  const std::vector<int> lb = level_bits(P);
  const int b1 = lb[0], s1 = kw - b1, nd1 = 1 << b1;

  // ---- presence + level-1 histograms; ranks; ids --------------------------
  const int64_t nw = int64_t((W + 31) / 32);
  uint2* words = ws_n<uint2>(WS_RANKMAP, size_t(nw));
  GT_CUDA(cudaMemsetAsync(words, 0, size_t(nw) * sizeof(uint2), st));
  unsigned long long* d_h1 = ws_n<unsigned long long>(WS_HIST, 2 * gtd::BK_MAXD);
  GT_CUDA(cudaMemsetAsync(d_h1, 0, 2 * nd1 * 8, st));
  {
    Phase ph("build.presence", 16.0 * rows);
    GT_LAUNCH(gtd::bk_presence_hist_kernel, std::max(1, std::min(ceil_div(rows, 1024), sms * 8)),
              256, 0, src, dst, rows, lo, words, s1, nd1, d_h1);
    if (n_extra) launch_presence(extra, extra, n_extra, lo, words);
  }
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  {
    Phase ph("build.rank_prefix", 16.0 * nw);
    launch_word_prefix(words, nw, small + 2);
  }
  std::vector<unsigned long long> h1(2 * nd1);
  int64_t n_nodes = 0;
  d2h(h1.data(), d_h1, h1.size() * 8);
  d2h(&n_nodes, small + 2, 8);
  sync();
  if (n_nodes >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "graph has >= 2^31 distinct node ids");
  g->n = n_nodes;
  g->kbits = bits_for(n_nodes);
  g->ids = dalloc_n<int64_t>(n_nodes);
  {
    Phase ph("build.ids", 8.0 * nw + 8.0 * n_nodes);
    launch_ids(words, nw, lo, g->ids);
  }

  // ---- level 1: pack + partition ------------------------------------------
  const int64_t R2 = 2 * rows;
  uint64_t* A = ws_n<uint64_t>(WS_KEYS_A, size_t(R2));
  uint64_t* B = ws_n<uint64_t>(WS_KEYS_B, size_t(R2));
  // segment starts of level 1 (both sides): [0, rows) out, [rows, 2rows) in
  std::vector<int64_t> seg(2 * nd1 + 1);
  {
    int64_t run = 0;
    for (int sd = 0; sd < 2; ++sd) {
      run = sd * rows;
      for (int d = 0; d < nd1; ++d) {
        seg[sd * nd1 + d] = run;
        run += int64_t(h1[sd * nd1 + d]);
      }
    }
    seg[2 * nd1] = R2;
  }
  // ping-pong segment-start arrays (level k: 2 * 2^(bits so far) + 1 entries)
  const size_t seg_cap = (size_t(2) << P) + 2;
  int64_t* d_seg0 = ws_n<int64_t>(WS_TMP0, seg_cap * 2);
  int64_t* d_seg1 = d_seg0 + seg_cap;
  h2d(d_seg0, seg.data(), seg.size() * 8);
  {
    unsigned long long* d_cur = ws_n<unsigned long long>(WS_TMP4, size_t(2 * nd1));
    std::vector<unsigned long long> cur(seg.begin(), seg.end() - 1);
    h2d(d_cur, cur.data(), cur.size() * 8);
    Phase ph("build.pack_part", 32.0 * rows);
    constexpr int KPT = 8;
    const size_t smem = size_t(2) * 256 * KPT * 8 + 2 * gtd::BK_MAXD * 12 + 64;
    static const bool once = [&] {
      set_smem(gtd::bk_pack_part_kernel<KPT>, smem);
      return true;
    }();
    (void)once;
    GT_LAUNCH(gtd::bk_pack_part_kernel<KPT>, sms * 4, 256, smem, src, dst, rows, lo, kw, s1, nd1,
              d_cur, A);
  }

  // ---- further levels -------------------------------------------------------
  uint64_t* cur_buf = A;
  uint64_t* oth_buf = B;
  int nseg = 2 * nd1;
  int bits_done = b1;
  unsigned int* d_hist = ws_n<unsigned int>(WS_TMP1, size_t(2) << P);
  for (size_t l = 1; l < lb.size(); ++l) {
    const int nd = 1 << lb[l];
    const int shift = 2 * kw - bits_done - lb[l];
    seg_level(cur_buf, oth_buf, d_seg0, d_seg0 + 1, nseg, shift, nd, d_hist, d_seg1,
              "build.partition", double(R2));
    GT_CUDA(cudaMemcpyAsync(d_seg1 + int64_t(nseg) * nd, d_seg0 + nseg, 8,
                            cudaMemcpyDeviceToDevice, st));
    std::swap(d_seg0, d_seg1);
    std::swap(cur_buf, oth_buf);
    nseg *= nd;
    bits_done += lb[l];
  }
  const int bufF = cur_buf == A ? 0 : 1;  // buffer holding the buckets
  const int nbk = nseg / 2;               // buckets per side (2^P)
  const int shiftP = 2 * kw - P;          // bucket b covers keys [b << shiftP, (b+1) << shiftP)
  const int64_t* d_bst = d_seg0;          // bucket starts, both sides, + end

  // ---- plan the main chains on the device -------------------------------------
  const int chunk = std::min(nbk, 1024);
  const int nchunks = 2 * nbk / chunk;
  const int IDCAP_BK = std::max(1, 4096 >> (kw - P));  // buckets per group (id span <= 4096)
  char* pl = static_cast<char*>(ws_get(WS_TMP2, size_t(nchunks + 2) * 16 + 64));
  int64_t* d_loff = reinterpret_cast<int64_t*>(pl);
  int64_t* d_hoff = d_loff + nchunks + 1;
  int64_t* d_small = ws_n<int64_t>(WS_SMALL, 16);
  GT_LAUNCH(gtd::bk_plan_main_kernel<false>, ceil_div(nchunks, 128), 128, 0, d_bst, nbk, chunk,
            nchunks, shiftP, bufF, CAP, IDCAP_BK, d_loff, d_hoff, (BkLeaf*)nullptr,
            (gtd::BkHuge*)nullptr);
  exclusive_scan_i64(d_loff, nchunks, d_small + 12);
  exclusive_scan_i64(d_hoff, nchunks, d_small + 13);
  int64_t hs[3];
  d2h(&hs[0], d_loff + nchunks, 8);      // leaves
  d2h(&hs[1], d_loff + nchunks / 2, 8);  // leaves of side 0
  d2h(&hs[2], d_hoff + nchunks, 8);      // huge buckets
  sync();
  const int u_total = int(hs[0]), u0 = int(hs[1]), nh = int(hs[2]);
  // leaf tables (main chain | huge LSD leaves | bitmap leaves), hubs, huges
  const int64_t hub_cap = 2 * rows / CAP + 2;
  const int64_t hl_cap = 8 * (2 * rows / CAP) + 4 * int64_t(nh) + 16;
  BkLeaf* d_main = static_cast<BkLeaf*>(dalloc(sizeof(BkLeaf) * size_t(u_total + 1)));
  gtd::BkHuge* d_huge = static_cast<gtd::BkHuge*>(dalloc(sizeof(gtd::BkHuge) * size_t(nh + 1)));
  GT_LAUNCH(gtd::bk_plan_main_kernel<true>, ceil_div(nchunks, 128), 128, 0, d_bst, nbk, chunk,
            nchunks, shiftP, bufF, CAP, IDCAP_BK, d_loff, d_hoff, d_main, d_huge);

  // ---- huge buckets: row split; hub rows: column split ----------------------------
  const int row_bits = kw - P;  // row bits below a bucket (<= 8)
  // column split of a hub row: 2^kid_c children of 2^kid_bits columns each
  // (<= 2^20 columns: the child's bitmap fits shared memory)
  const int kid_c = std::min({std::max(8, kw - 20), 9, std::max(0, kw - 5)});
  const int kid_bits = kw - kid_c;
  const int n_kids = 1 << kid_c;
  const int bufH = 1 - bufF;  // rows of huge buckets live here after the row split
  BkLeaf* d_hl = nullptr;
  BkLeaf* d_bml = nullptr;
  gtd::BkHub* d_hubs = nullptr;
  int* d_cnt = ws_n<int>(WS_COUNTERS, 64) + 48;  // [n_hl, n_hub, n_bm]
  GT_CUDA(cudaMemsetAsync(d_cnt, 0, 16, st));
  int n_hl = 0, n_hub = 0, n_bm = 0;
  int64_t huge_keys = 0;
  if (nh) {
    const int ndr = 1 << std::max(row_bits, 0);
    d_hl = static_cast<BkLeaf*>(dalloc(sizeof(BkLeaf) * size_t(hl_cap)));
    d_bml = static_cast<BkLeaf*>(dalloc(sizeof(BkLeaf) * size_t(hub_cap)));
    d_hubs = static_cast<gtd::BkHub*>(dalloc(sizeof(gtd::BkHub) * size_t(hub_cap)));
    int64_t* d_sb = ws_n<int64_t>(WS_TMP0, size_t(nh) * (2 + ndr) + 2);
    int64_t* d_rb = d_sb + 2 * nh;
    GT_LAUNCH(gtd::bk_huge_ranges_kernel, ceil_div(nh, 256), 256, 0, d_huge, nh, d_sb, d_sb + nh);
    unsigned int* d_rh = ws_n<unsigned int>(WS_TMP1, size_t(nh) * ndr);
    seg_level(cur_buf, oth_buf, d_sb, d_sb + nh, nh, kw, ndr, d_rh, d_rb, "build.split_rows",
              0.0);
    GT_LAUNCH(gtd::bk_plan_rows_kernel, ceil_div(nh, 128), 128, 0, d_huge, nh, d_rb, d_rh, ndr,
              shiftP, kw, bufH, CAP, d_hl, d_cnt, d_hubs, d_cnt + 1);
    int c2[2];
    d2h(c2, d_cnt, 8);
    sync();
    n_hub = c2[1];
    if (n_hub > hub_cap) fail(GT_ECUDA, "bucket build: hub table overflow (internal error)");
    if (n_hub) {
      int64_t* d_s2 = ws_n<int64_t>(WS_TMP0, size_t(n_hub) * (2 + n_kids) + 2);
      int64_t* d_kb = d_s2 + 2 * n_hub;
      GT_LAUNCH(gtd::bk_hub_ranges_kernel, ceil_div(n_hub, 256), 256, 0, d_hubs, n_hub, d_s2,
                d_s2 + n_hub);
      unsigned int* d_kh = ws_n<unsigned int>(WS_TMP1, size_t(n_hub) * n_kids);
      seg_level(oth_buf, cur_buf, d_s2, d_s2 + n_hub, n_hub, kid_bits, n_kids, d_kh, d_kb,
                "build.split_cols", 0.0);
      GT_LAUNCH(gtd::bk_plan_kids_kernel, ceil_div(n_hub, 128), 128, 0, d_hubs, n_hub, d_kb, d_kh,
                n_kids, kid_bits, kw, bufF, CAP, d_hl, d_cnt, d_bml, d_cnt + 2);
    }
    int c3[3];
    d2h(c3, d_cnt, 12);
    sync();
    n_hl = c3[0];
    n_bm = c3[2];
    if (n_hl > hl_cap || n_bm > hub_cap)
      fail(GT_ECUDA, "bucket build: leaf table overflow (internal error)");
  }
  if (getenv("GT_BK_STATS"))
    fprintf(stderr,
            "[gt bucket] rows=%lld W=%llu kw=%d P=%d levels=%zu main=%d (side0 %d) huge=%d "
            "huge_leaves=%d hubs=%d bitmap=%d kid_bits=%d\n",
            (long long)rows, (unsigned long long)W, kw, P, lb.size(), u_total, u0, nh, n_hl, n_hub,
            n_bm, kid_bits);

  // ---- outputs ----------------------------------------------------------------
  g->out_adj = dalloc_n<int32_t>(rows);  // E <= rows; exact E after the pass
  g->in_adj = dalloc_n<int32_t>(rows);
  g->out_off = dalloc_n<int64_t>(n_nodes + 1);
  g->in_off = dalloc_n<int64_t>(n_nodes + 1);

  gtd::BkArgs args{};
  args.buf[0] = A; args.buf[1] = B;
  args.wbuf[0] = A; args.wbuf[1] = B;
  args.words = words;
  args.kw = kw;
  args.n_ids = int64_t(W);
  args.n_nodes = n_nodes;
  args.off[0] = g->out_off; args.off[1] = g->in_off;
  args.adj[0] = g->out_adj; args.adj[1] = g->in_adj;
  args.kid_bits = kid_bits;
  args.n_kids = n_kids;
  args.rows = rows;
  const size_t n_deg = size_t(2) * n_nodes;
  char* sp = static_cast<char*>(dalloc(size_t(nh) * 8 + size_t(n_hub) * n_kids * 8 +
                                       size_t(n_hl + n_bm) * 4 + (nh ? n_deg * 4 : 0) +
                                       size_t(u_total + 2) * 8 + 256));
  char* sp0 = sp;
  auto carve = [&](size_t b) { char* r = sp; sp += (b + 15) & ~size_t(15); return r; };
  args.huge_total = reinterpret_cast<unsigned long long*>(carve(size_t(nh) * 8));
  args.leaf_d = reinterpret_cast<int32_t*>(carve(size_t(n_hl + n_bm) * 4));
  args.child_cnt = reinterpret_cast<uint32_t*>(carve(size_t(n_hub) * n_kids * 4));
  args.child_base = reinterpret_cast<uint32_t*>(carve(size_t(n_hub) * n_kids * 4));
  args.deg = nh ? reinterpret_cast<uint32_t*>(carve(n_deg * 4)) : nullptr;
  args.main_d = reinterpret_cast<int64_t*>(carve(size_t(u_total + 2) * 8));
  args.tmp[0] = static_cast<uint32_t*>(dalloc(size_t(R2) * 4));
  args.tmp[1] = args.tmp[0] + rows;

  const size_t lsm = sizeof(gtd::LeafSmem);
  static const bool once = [&] {
    set_smem(gtd::bk_leaf_kernel<true>, lsm);
    set_smem(gtd::bk_leaf_kernel<false>, lsm);
    set_smem(gtd::bk_bitmap_leaf_kernel, size_t(128) * 1024);
    return true;
  }();
  (void)once;
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  if (nh) {
    GT_CUDA(cudaMemsetAsync(args.huge_total, 0, size_t(nh) * 8, st));
    GT_CUDA(cudaMemsetAsync(args.deg, 0, n_deg * 4, st));
    if (n_hub) GT_CUDA(cudaMemsetAsync(args.child_cnt, 0, size_t(n_hub) * n_kids * 4, st));
    Phase ph("build.huge_count", 0.0);
    if (n_hl) {
      GT_CUDA(cudaMemsetAsync(counters + 40, 0, 4, st));
      GT_LAUNCH(gtd::bk_leaf_kernel<false>, std::min(n_hl, sms), gtd::LF_THREADS, lsm, d_hl, n_hl,
                n_hl, args, counters + 40);
    }
    if (n_bm) {
      gtd::BkArgs a2 = args;
      a2.leaf_d = args.leaf_d + n_hl;
      GT_LAUNCH(gtd::bk_bitmap_leaf_kernel, std::min(n_bm, sms), 1024,
                std::max<size_t>(4, size_t(1 << kid_bits) / 8), d_bml, n_bm, a2);
    }
  }
  {
    Phase ph("build.leaves", 0.0);
    GT_CUDA(cudaMemsetAsync(counters + 41, 0, 4, st));
    GT_LAUNCH(gtd::bk_leaf_kernel<true>, std::min(u_total, sms), gtd::LF_THREADS, lsm, d_main,
              u_total, u0, args, counters + 41);
  }
  {
    Phase ph("build.compact", 0.0);
    exclusive_scan_i64(args.main_d, u0, d_small + 10);
    exclusive_scan_i64(args.main_d + u0 + 1, u_total - u0, d_small + 11);
    GT_LAUNCH(gtd::bk_compact_kernel, std::min(u_total, sms * 8), 256, 0, d_main, u_total, u0,
              args);
  }
  if (n_hl + n_bm) {
    Phase ph("build.huge_emit", 0.0);
    if (n_hub)
      GT_LAUNCH(gtd::bk_hub_prefix_kernel, n_hub, 256, 0, args.child_cnt, args.child_base, n_kids);
    if (n_hl)
      GT_LAUNCH(gtd::bk_emit_kernel, std::min(n_hl, sms * 8), 256, 0, d_hl, n_hl, args);
    if (n_bm) {
      gtd::BkArgs a2 = args;
      a2.leaf_d = args.leaf_d + n_hl;
      GT_LAUNCH(gtd::bk_emit_kernel, std::min(n_bm, sms * 8), 256, 0, d_bml, n_bm, a2);
    }
  }
  int64_t e[2];
  d2h(&e[0], g->out_off + n_nodes, 8);
  d2h(&e[1], g->in_off + n_nodes, 8);
  sync();
  dfree(d_main);
  dfree(d_huge);
  dfree(d_hl);
  dfree(d_bml);
  dfree(d_hubs);
  dfree(sp0);
  dfree(args.tmp[0]);
  if (e[0] != e[1]) fail(GT_ECUDA, "bucket build: out/in edge counts differ (internal error)");
  g->e = e[0];
  (void)huge_keys;
  // algorithmic bytes: presence 16R, pack 16R+16R, each
  // further level 8 + 16 B per key, leaves 8 B per key in + 4 B per edge out
  // + 8 B per offset, compaction 8 B per edge
  profile_add_bytes("build.leaves", 8.0 * double(R2) + 8.0 * double(e[0]) +
                                        16.0 * double(n_nodes + 1));
  profile_add_bytes("build.compact", 16.0 * double(e[0]));
}

}  // namespace gt
