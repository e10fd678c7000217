// radix_sort.cu — onesweep LSD radix sort (see radix_sort.cuh).
#include "radix_sort.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace gtd {

using gt::RS_KPT;
using gt::RS_THREADS;
using gt::RS_TILE;

// resident CTAs per SM the onesweep register budget is sized for
constexpr int RS_MIN_BLOCKS = 3;
// predecessor status words polled per look-back round trip (GT_LB_WIN: sweeps)
#ifndef GT_LB_WIN
#define GT_LB_WIN 4
#endif
constexpr int LB_WIN = GT_LB_WIN;

__global__ void __launch_bounds__(256) hist_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                   gt::SortPlan plan,
                                                   unsigned long long* __restrict__ ghist) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    plan_hist_add(sh, plan, ld_stream_u64(keys + i));
  __syncthreads();
  plan_hist_flush(sh, plan, ghist);
}

// grid = passes, block = 256: exclusive scan of each pass's 256 digit counts.
__global__ void __launch_bounds__(256) digit_scan_kernel(const unsigned long long* __restrict__ ghist,
                                                         int64_t* __restrict__ base) {
  __shared__ int64_t sm[8];
  const int q = blockIdx.x;
  int64_t v = int64_t(ghist[q * 256 + threadIdx.x]);
  int64_t tot;
  int64_t ex = block_excl_scan_256<int64_t>(v, sm, tot);
  base[q * 256 + threadIdx.x] = ex;
}

// One onesweep LSD pass over a BITS-wide digit (BITS is a template parameter
// so the per-bit ballot loop is fully unrolled). RS_MATCH of the RS_KPT keys
// of a thread are ranked with __match_any_sync (ADU pipe), the rest with one
// ballot per digit bit (ALU pipe): splitting the ranking across the two pipes
// keeps either from being the bottleneck (ncu: all-MATCH ranking was 68%
// ADU-bound, all-ballot ranking doubled the instruction count).
struct OnesweepSmem {
  uint64_t keys[RS_TILE];  // staged by index during the look-back, then by position
  uint32_t whist[RS_THREADS / 32][256];
  int64_t gbase[256];
  uint32_t scan[8];
  uint32_t tile;
};

// One tile of a onesweep pass. FULL: the tile holds RS_TILE keys, so every
// per-key bounds test compiles away (all tiles but the last).
template <int BITS, int RS_MATCH, bool FULL>
__device__ __forceinline__ void onesweep_tile(OnesweepSmem& s, const uint64_t* __restrict__ in,
                                              uint64_t* __restrict__ out, int64_t n, int shift,
                                              const int64_t* __restrict__ digit_base,
                                              uint64_t* __restrict__ status, int tile,
                                              uint32_t epoch) {
  constexpr int NW = RS_THREADS / 32;
  constexpr uint32_t mask = (1u << BITS) - 1u;
  int64_t* s_gbase = s.gbase;
  uint32_t* s_scan = s.scan;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t base = int64_t(tile) * RS_TILE;
  const int woff = warp * 32 * RS_KPT + lane;  // key i of this thread: tile element woff + 32*i

  int rem = 32 * RS_KPT;
  if (!FULL) {
    const int64_t rem64 = n - (base + woff);
    rem = rem64 > 32 * RS_KPT ? 32 * RS_KPT : (rem64 < 0 ? 0 : int(rem64));
  }
  const uint64_t* src = in + (base + woff);
  uint64_t k[RS_KPT];
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) k[i] = 32 * i < rem ? ld_stream_u64(src + 32 * i) : ~0ull;

  // Peer masks: lanes of this warp whose key i has the same digit (invalid
  // tail keys are in no mask).
  uint32_t rank[RS_KPT];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) {
    const uint32_t d = uint32_t(k[i] >> shift) & mask;
    if (i < RS_MATCH) {
      rank[i] = FULL ? __match_any_sync(0xffffffffu, d)
                     : __match_any_sync(0xffffffffu, 32 * i < rem ? d : 0xFFFFu) &
                           __ballot_sync(0xffffffffu, 32 * i < rem);
    } else {
      uint32_t peers = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, 32 * i < rem);
#pragma unroll
      for (int b = 0; b < BITS; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
      }
      rank[i] = peers;
    }
  }
  // Stable ranks: key by key, the highest peer adds the group size to the
  // warp's private counter with one shared atomic; the old value is
  // broadcast to the group.
  uint32_t* wh = s.whist[warp];
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) {
    const uint32_t peers = rank[i];
    const int leader = 31 - __clz(peers);
    uint32_t before = 0;
    if (32 * i < rem && lane == leader)
      before = atomicAdd(&wh[uint32_t(k[i] >> shift) & mask], __popc(peers));
    before = __shfl_sync(0xffffffffu, before, leader);
    rank[i] = before + __popc(peers & lt);
  }
  // park the keys in shared memory (by index) so that they do not hold 32
  // registers across the look-back
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) s.keys[woff + 32 * i] = k[i];
  __syncthreads();

  // Per digit (thread == digit): warp offsets, tile count, look-back.
  if (tid < (1 << BITS)) {
    const int d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = s.whist[w][d];
      s.whist[w][d] = run;
      run += c;
    }
    const uint32_t tile_cnt = run;
    uint64_t* st = status + int64_t(tile) * 256 + d;
    if (tile == 0) st_status_u64(st, lb_pack(LB_INC, epoch, tile_cnt));
    else st_status_u64(st, lb_pack(LB_AGG, epoch, tile_cnt));
    s.whist[0][d] = run;  // tile count, for the in-tile digit scan below (w=0 offset is 0)
    // Decoupled look-back, LB_WIN predecessors polled per round trip.
    uint64_t excl = 0;
    if (tile > 0) {
      const uint64_t ep = uint64_t(epoch & 0x3FFFFFu);
      int t = tile - 1;
      bool done = false;
      while (!done) {
        uint64_t v[LB_WIN];
#pragma unroll
        for (int q = 0; q < LB_WIN; ++q)
          v[q] = t - q >= 0 ? ld_status_u64(status + int64_t(t - q) * 256 + d) : 0ull;
#pragma unroll
        for (int q = 0; q < LB_WIN; ++q) {
          if (done || t < 0) break;
          if (((v[q] >> 40) & 0x3FFFFFu) != ep || (v[q] >> 62) == 0) break;  // re-poll
          excl += v[q] & ((1ull << 40) - 1);
          if ((v[q] >> 62) == 2) done = true;
          else --t;
        }
      }
      st_status_u64(st, lb_pack(LB_INC, epoch, excl + tile_cnt));
    }
    s_gbase[d] = digit_base[d] + int64_t(excl);
  }
  __syncthreads();
  // in-tile digit starts (exclusive scan of the tile counts over the digits)
  {
    const uint32_t c = tid < (1 << BITS) ? s.whist[0][tid] : 0u;
    uint32_t tot;
    const uint32_t start = block_excl_scan_256<uint32_t>(c, s_scan, tot);
    if (tid < (1 << BITS)) {
      s.whist[0][tid] = 0;
      s_gbase[tid] -= int64_t(start);
#pragma unroll
      for (int w = 0; w < NW; ++w) s.whist[w][tid] += start;
    }
  }
  __syncthreads();

  uint32_t pos[RS_KPT];
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) {
    k[i] = s.keys[woff + 32 * i];
    pos[i] = s.whist[warp][uint32_t(k[i] >> shift) & mask] + rank[i];
  }
  __syncthreads();  // every key read back before the buffer is reused by position
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i)
    if (32 * i < rem) s.keys[pos[i]] = k[i];
  __syncthreads();

  if (FULL) {
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i) {
      const int j = tid + i * RS_THREADS;
      const uint64_t key = s.keys[j];
      out[s_gbase[uint32_t(key >> shift) & mask] + j] = key;
    }
  } else {
    const int nvalid = (n - base) < RS_TILE ? int(n - base) : RS_TILE;
    for (int j = tid; j < nvalid; j += RS_THREADS) {
      const uint64_t key = s.keys[j];
      out[s_gbase[uint32_t(key >> shift) & mask] + j] = key;
    }
  }
}

template <int BITS, int RS_MATCH>
__global__ void __launch_bounds__(RS_THREADS, RS_MIN_BLOCKS)
    onesweep_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t n,
                    int shift, const int64_t* __restrict__ digit_base,
                    uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter,
                    uint32_t epoch) {
  extern __shared__ __align__(16) unsigned char os_dsm[];  // dynamic: tiles may exceed 48 KB
  OnesweepSmem& s = *reinterpret_cast<OnesweepSmem*>(os_dsm);
  if (threadIdx.x == 0) s.tile = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < (RS_THREADS / 32) * 256; i += RS_THREADS) (&s.whist[0][0])[i] = 0;
  __syncthreads();
  const int tile = int(s.tile);
  if (int64_t(tile + 1) * RS_TILE <= n)
    onesweep_tile<BITS, RS_MATCH, true>(s, in, out, n, shift, digit_base, status, tile, epoch);
  else
    onesweep_tile<BITS, RS_MATCH, false>(s, in, out, n, shift, digit_base, status, tile, epoch);
}

// ---- onesweep pass that ranks from shared memory -----------------------------
// The kernel above loads its tile into registers and then ranks it; the keys
// (32 registers) are what caps it at 80 registers = 3 CTAs per SM (ncu at C4:
// 37% warps active, 2.6 TB/s, a fifth of the stall samples at the barrier
// after the look-back). This one brings its tile into shared memory with ONE
// bulk asynchronous copy (cp.async.bulk, completion counted on an mbarrier)
// issued by one thread, and ranks it straight from there: no register
// staging, no parking store, 64 registers. NT = 256 (4096-key tiles, 4 CTAs
// per SM) or 512 (8192-key tiles, 2 CTAs per SM: half the look-backs).
// Measured alternatives, not kept (profiles/r2s2_sort_kernel_variants.txt):
// persistent CTAs double-buffering the next tile (the drawn tile waits a tile
// time before publishing its aggregate, so successors' look-backs walk
// further: slower in every placement of the draw), and a dedicated look-back
// warp overlapping the in-tile scatter (one lane per 8 digits polls one
// predecessor per round trip: 1.5x slower).
#ifndef GT_SMEM_LB_WIN
#define GT_SMEM_LB_WIN 2
#endif
constexpr int SMEM_LB_WIN = GT_SMEM_LB_WIN;

template <int NT>
struct OnesweepSmemT {
  uint64_t keys[NT * RS_KPT];  // the tile by index, then scattered in place by position
  uint32_t whist[NT / 32][256];
  int64_t gbase[256];
  unsigned long long bar;
  uint32_t scan[NT / 32];
  int tile;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
// Arm `bar` for `bytes` and start the bulk global->shared copy that completes it.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Exclusive scan across an NT-thread block; `sm` needs NT/32 slots.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_nt(uint32_t v, uint32_t* sm) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t inc = warp_incl_scan(v);
  if (l == 31) sm[w] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i)
    if (i < w) wpre += sm[i];
  __syncthreads();
  return wpre + inc - v;
}

// Tiles are drawn in ticket order, so the tile `pf_dist` tickets ahead is one
// that some CTA draws about one residency wave from now: its keys are pulled
// into L2 here (cp.async.bulk.prefetch.L2), so that CTA's bulk copy finds them
// there instead of waiting on DRAM. 0 = off.
template <int BITS, int RS_MATCH, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)
    onesweep_smem_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t n,
                         int shift, const int64_t* __restrict__ digit_base,
                         uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter,
                         uint32_t epoch, int pf_dist) {
  constexpr int NW = NT / 32;
  constexpr int TILE = NT * RS_KPT;
  constexpr uint32_t mask = (1u << BITS) - 1u;
  extern __shared__ __align__(128) unsigned char os1_dsm[];
  OnesweepSmemT<NT>& s = *reinterpret_cast<OnesweepSmemT<NT>*>(os1_dsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    const int t = int(atomicAdd(tile_counter, 1u));
    s.tile = t;
    if (int64_t(t + 1) * TILE <= n) {
      mbar_init(&s.bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      bulk_load(s.keys, in + int64_t(t) * TILE, TILE * 8, &s.bar);
    }
    if (pf_dist > 0 && int64_t(t + pf_dist + 1) * TILE <= n)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(in + int64_t(t + pf_dist) * TILE),
                   "r"(TILE * 8)
                   : "memory");
  }
  for (int i = tid; i < NW * 256; i += NT) (&s.whist[0][0])[i] = 0;
  __syncthreads();
  const int cur = s.tile;
  const int64_t base = int64_t(cur) * TILE;
  const bool full = base + TILE <= n;
  const int nvalid = full ? TILE : int(n - base);
  const int woff = warp * 32 * RS_KPT + lane;  // key i of this thread: tile element woff + 32*i
  int rem = nvalid - woff;
  rem = rem > 32 * RS_KPT ? 32 * RS_KPT : (rem < 0 ? 0 : rem);
  if (full) {
    mbar_wait(&s.bar, 0);
  } else {  // the last, partial tile: plain loads
    for (int j = tid; j < nvalid; j += NT) s.keys[j] = ld_stream_u64(in + base + j);
    __syncthreads();
  }

  // Stable ranks: peer masks (MATCH for RS_MATCH keys, one ballot per digit
  // bit for the rest), then key by key the highest peer adds the group size to
  // the warp's counter with one shared atomic and broadcasts the old value.
  uint32_t rank[RS_KPT];
  {
    const unsigned lt = lanemask_lt();
    uint32_t d[RS_KPT];
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i) d[i] = uint32_t(s.keys[woff + 32 * i] >> shift) & mask;
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i) {
      if (i < RS_MATCH) {
        rank[i] = full ? __match_any_sync(0xffffffffu, d[i])
                       : __match_any_sync(0xffffffffu, 32 * i < rem ? d[i] : 0xFFFFu) &
                             __ballot_sync(0xffffffffu, 32 * i < rem);
      } else {
        uint32_t peers = full ? 0xffffffffu : __ballot_sync(0xffffffffu, 32 * i < rem);
#pragma unroll
        for (int q = 0; q < BITS; ++q) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (d[i] >> q) & 1u);
          peers &= ((d[i] >> q) & 1u) ? bal : ~bal;
        }
        rank[i] = peers;
      }
    }
    uint32_t* wh = s.whist[warp];
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i) {
      const uint32_t peers = rank[i];
      const int leader = 31 - __clz(peers);
      uint32_t before = 0;
      if (32 * i < rem && lane == leader) before = atomicAdd(&wh[d[i]], __popc(peers));
      before = __shfl_sync(0xffffffffu, before, leader);
      rank[i] = before + __popc(peers & lt);
    }
  }
  __syncthreads();

  uint32_t tile_cnt = 0;
  if (tid < (1 << BITS)) {  // per digit: warp offsets, tile count, decoupled look-back
    const int d = tid;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = s.whist[w][d];
      s.whist[w][d] = tile_cnt;
      tile_cnt += c;
    }
    uint64_t* st = status + int64_t(cur) * 256 + d;
    st_status_u64(st, lb_pack(cur == 0 ? LB_INC : LB_AGG, epoch, tile_cnt));
    uint64_t excl = 0;
    if (cur > 0) {
      const uint64_t ep = uint64_t(epoch & 0x3FFFFFu);
      int t = cur - 1;
      bool done = false;
      while (!done) {
        uint64_t v[SMEM_LB_WIN];
#pragma unroll
        for (int q = 0; q < SMEM_LB_WIN; ++q)
          v[q] = t - q >= 0 ? ld_status_u64(status + int64_t(t - q) * 256 + d) : 0ull;
#pragma unroll
        for (int q = 0; q < SMEM_LB_WIN; ++q) {
          if (done || t < 0) break;
          if (((v[q] >> 40) & 0x3FFFFFu) != ep || (v[q] >> 62) == 0) break;  // re-poll
          excl += v[q] & ((1ull << 40) - 1);
          if ((v[q] >> 62) == 2) done = true;
          else --t;
        }
      }
      st_status_u64(st, lb_pack(LB_INC, epoch, excl + tile_cnt));
    }
    s.gbase[d] = digit_base[d] + int64_t(excl);
  }
#ifdef GT_SMEM_LB_SYNC
  __syncthreads();
#endif
  {  // in-tile digit starts (exclusive scan of the tile counts over the digits)
    const uint32_t start = block_excl_scan_nt<NT>(tile_cnt, s.scan);
    if (tid < (1 << BITS)) {
      s.gbase[tid] -= int64_t(start);
#pragma unroll
      for (int w = 0; w < NW; ++w) s.whist[w][tid] += start;
    }
  }
  __syncthreads();
  {
    uint64_t k[RS_KPT];
    uint32_t pos[RS_KPT];
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i) {
      k[i] = s.keys[woff + 32 * i];
      pos[i] = s.whist[warp][uint32_t(k[i] >> shift) & mask] + rank[i];
    }
    __syncthreads();  // every key read before the buffer is reused by position
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i)
      if (32 * i < rem) s.keys[pos[i]] = k[i];
  }
  __syncthreads();
  if (full) {
#pragma unroll
    for (int i = 0; i < RS_KPT; ++i) {
      const int j = tid + i * NT;
      const uint64_t key = s.keys[j];
      out[s.gbase[uint32_t(key >> shift) & mask] + j] = key;
    }
  } else {
    for (int j = tid; j < nvalid; j += NT) {
      const uint64_t key = s.keys[j];
      out[s.gbase[uint32_t(key >> shift) & mask] + j] = key;
    }
  }
}

}  // namespace gtd

namespace gt {

SortPlan make_plan(int lo_bit, int hi_bit) {
  SortPlan p;
  int width = hi_bit - lo_bit;
  if (width <= 0) return p;
  p.passes = (width + 7) / 8;
  int shift = lo_bit;
  for (int q = 0; q < p.passes; ++q) {
    int b = width / p.passes + (q < width % p.passes ? 1 : 0);
    p.shift[q] = shift;
    p.bits[q] = b;
    shift += b;
  }
  return p;
}

SortHist sort_hist_begin(int slot_index) {
  char* base = static_cast<char*>(ws_get(WS_HIST, 2 * (RS_MAX_PASSES * 256 * 16)));
  base += slot_index * (RS_MAX_PASSES * 256 * 16);
  SortHist h;
  h.hist = reinterpret_cast<unsigned long long*>(base);
  h.digit_base = reinterpret_cast<int64_t*>(base + RS_MAX_PASSES * 256 * 8);
  GT_CUDA(cudaMemsetAsync(h.hist, 0, RS_MAX_PASSES * 256 * 8, ctx().stream));
  return h;
}

void sort_histogram(const uint64_t* keys, int64_t n, const SortPlan& plan, SortHist h) {
  if (n == 0 || plan.passes == 0) return;
  Phase ph("sort.histogram", 8.0 * n);
  int grid = static_cast<int>(std::min<int64_t>(ctx().sm_count * 4, ceil_div64(n, 256)));
  GT_LAUNCH(gtd::hist_kernel, grid, 256, 0, keys, n, plan, h.hist);
}

template <int BITS, int M>
static void launch_bits(int grid, const uint64_t* src, uint64_t* dst, int64_t n, int shift,
                        const int64_t* digit_base, uint64_t* status, uint32_t* counter,
                        uint32_t epoch) {
  // thread-safe one-time set-up (lanes may launch from two threads)
  static const bool attr_set = [] {
    GT_CUDA(cudaFuncSetAttribute(gtd::onesweep_kernel<BITS, M>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sizeof(gtd::OnesweepSmem))));
    return true;
  }();
  (void)attr_set;
  GT_LAUNCH((gtd::onesweep_kernel<BITS, M>), grid, RS_THREADS, sizeof(gtd::OnesweepSmem), src, dst,
            n, shift, digit_base, status, counter, epoch);
}

// onesweep_smem_kernel with NT threads per CTA (tiles of NT * RS_KPT keys)
template <int BITS, int M, int NT>
static void launch_smem_bits(const uint64_t* src, uint64_t* dst, int64_t n, int shift,
                             const int64_t* digit_base, uint64_t* status, uint32_t* counter,
                             uint32_t epoch) {
  constexpr auto kern = gtd::onesweep_smem_kernel<BITS, M, NT>;
  constexpr size_t smem = sizeof(gtd::OnesweepSmemT<NT>);
  static const bool once = [] {  // thread-safe one-time set-up
    GT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    GT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (getenv("GT_SORT_DEBUG")) {
      int b = 0;
      GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, NT, smem));
      fprintf(stderr, "onesweep_smem<%d,%d,%d>: %d CTAs/SM, %zu B smem\n", BITS, M, NT, b, smem);
    }
    return true;
  }();
  (void)once;
  // GT_SORT_PF: prefetch distance in tiles (default: one residency wave)
  static const int pf_dist = [] {
    const char* env = getenv("GT_SORT_PF");
    if (env) return atoi(env);
    int b = 0;
    GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, NT, smem));
    return b * ctx().sm_count;
  }();
  GT_LAUNCH(kern, static_cast<int>(ceil_div64(n, int64_t(NT) * RS_KPT)), NT, smem, src, dst, n,
            shift, digit_base, status, counter, epoch, pf_dist);
}

template <int NT>
static void launch_smem(int bits, const uint64_t* src, uint64_t* dst, int64_t n, int shift,
                        const int64_t* digit_base, uint64_t* status, uint32_t* counter,
                        uint32_t epoch) {
  switch (bits) {
#define GT_SMEM_CASE(B)                                                                      \
  case B:                                                                                    \
    launch_smem_bits<B, 6, NT>(src, dst, n, shift, digit_base, status, counter, epoch);      \
    break;
    GT_SMEM_CASE(1) GT_SMEM_CASE(2) GT_SMEM_CASE(3) GT_SMEM_CASE(4)
    GT_SMEM_CASE(5) GT_SMEM_CASE(6) GT_SMEM_CASE(7) GT_SMEM_CASE(8)
#undef GT_SMEM_CASE
    default: fail(GT_EINVAL, "radix digit width must be 1..8");
  }
}

template <int M>
static void launch_m(int bits, int grid, const uint64_t* src, uint64_t* dst, int64_t n, int shift,
                     const int64_t* digit_base, uint64_t* status, uint32_t* counter,
                     uint32_t epoch) {
  switch (bits) {
    case 1: launch_bits<1, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 2: launch_bits<2, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 3: launch_bits<3, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 4: launch_bits<4, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 5: launch_bits<5, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 6: launch_bits<6, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 7: launch_bits<7, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    case 8: launch_bits<8, M>(grid, src, dst, n, shift, digit_base, status, counter, epoch); break;
    default: fail(GT_EINVAL, "radix digit width must be 1..8");
  }
}

static void launch_onesweep(int bits, int nmatch, int grid, const uint64_t* src, uint64_t* dst,
                            int64_t n, int shift, const int64_t* digit_base, uint64_t* status,
                            uint32_t* counter, uint32_t epoch) {
  // GT_SORT_KERNEL (A/B measurements): 0 = the register-staged kernel,
  // 1 = the shared-memory-ranked kernel with 256-thread CTAs, 2 = with
  // 512-thread CTAs. The bulk copy needs 16-byte aligned tiles.
  static const int kind = [] {
    const char* env = getenv("GT_SORT_KERNEL");
    return env ? atoi(env) : 1;
  }();
  if (kind > 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    if (kind == 2) launch_smem<512>(bits, src, dst, n, shift, digit_base, status, counter, epoch);
    else launch_smem<256>(bits, src, dst, n, shift, digit_base, status, counter, epoch);
    return;
  }
  if (nmatch <= 0)
    launch_m<0>(bits, grid, src, dst, n, shift, digit_base, status, counter, epoch);
  else if (nmatch >= RS_KPT)
    launch_m<RS_KPT>(bits, grid, src, dst, n, shift, digit_base, status, counter, epoch);
  else if (nmatch <= 6)
    launch_m<6>(bits, grid, src, dst, n, shift, digit_base, status, counter, epoch);
  else if (nmatch <= 8)
    launch_m<8>(bits, grid, src, dst, n, shift, digit_base, status, counter, epoch);
  else
    launch_m<11>(bits, grid, src, dst, n, shift, digit_base, status, counter, epoch);
}

uint64_t* radix_sort(uint64_t* a, uint64_t* b, int64_t n, const SortPlan& plan, SortHist h,
                     const char* phase, bool first_unstable) {
  if (n <= 1 || plan.passes == 0) return a;
  const int64_t tiles = ceil_div64(n, RS_TILE);
  if (tiles >= (1ll << 31)) fail(GT_ECAPACITY, "radix sort: too many tiles");
  uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) * 256);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  GT_CUDA(cudaMemsetAsync(counters, 0, RS_MAX_PASSES * sizeof(uint32_t), ctx().stream));
  {
    Phase ph("sort.digit_scan", 0.0);
    GT_LAUNCH(gtd::digit_scan_kernel, plan.passes, 256, 0, h.hist, h.digit_base);
  }
  uint64_t* src = a;
  uint64_t* dst = b;
  static const int nmatch = [] {  // GT_SORT_MATCH: keys per thread ranked by MATCH (tuning)
    const char* env = getenv("GT_SORT_MATCH");
    return env ? atoi(env) : 6;
  }();
  static const bool stable_only = [] {  // GT_SORT_STABLE_FIRST=1: onesweep for every pass
    const char* env = getenv("GT_SORT_STABLE_FIRST");
    return env && atoi(env);
  }();
  for (int q = 0; q < plan.passes; ++q) {
    Phase ph(phase, 16.0 * n);
    if (q == 0 && first_unstable && !stable_only) {
      partition_pass(src, dst, n, plan.shift[q], plan.bits[q], h.digit_base + q * 256);
      std::swap(src, dst);
      continue;
    }
    const uint32_t epoch = next_epoch();
    launch_onesweep(plan.bits[q], nmatch, static_cast<int>(tiles), src, dst, n, plan.shift[q],
                    h.digit_base + q * 256, status, counters + q, epoch);
    std::swap(src, dst);
  }
  return src;
}

}  // namespace gt
