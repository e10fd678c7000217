// radix_sort.cuh — LSD radix sort of 64-bit keys over an arbitrary bit range.
//
// One "onesweep" kernel per 8-bit digit: tiles of 4096 keys are ranked with
// warp-ballot multi-split into per-warp shared-memory histograms, the tile's
// digit counts are chained to the preceding tiles by decoupled look-back, and
// keys are scattered through shared memory so that every run of equal digits
// leaves the SM as contiguous stores. The per-pass digit histograms are
// computed up front for all passes at once — by the producer kernel that
// writes the keys (pack / dedupe) or by hist_kernel — so each pass reads and
// writes every key exactly once (16 B/key/pass of HBM traffic).
//
// This replaces the reference's sample sort + threaded np.sort
// (parallel.py:52-93) and its lexsort fallback (convert.py:82-89).
#pragma once

#include "common.cuh"

namespace gt {

constexpr int RS_THREADS = 256;
constexpr int RS_KPT = 16;
constexpr int RS_TILE = RS_THREADS * RS_KPT;  // 4096 keys
constexpr int RS_MAX_PASSES = 8;

struct SortPlan {
  int passes = 0;
  int shift[RS_MAX_PASSES] = {0};
  int bits[RS_MAX_PASSES] = {0};
};

// Split [lo_bit, hi_bit) into ceil(width/8) near-equal digits, LSD first.
SortPlan make_plan(int lo_bit, int hi_bit);

// Device scratch for a sort: histograms [passes][256] (u64), digit bases.
struct SortHist {
  unsigned long long* hist;  // zeroed by sort_hist_begin
  int64_t* digit_base;
};
SortHist sort_hist_begin(int slot_index);  // slot_index 0/1: two independent sorts may overlap

// Histogram all passes of `plan` over keys (when no producer kernel fused it).
void sort_histogram(const uint64_t* keys, int64_t n, const SortPlan& plan, SortHist h);

// Sort n keys (in `a`) by `plan`; `b` is scratch of the same size. The
// histogram `h` must already hold the digit counts of the keys. Returns the
// buffer that holds the sorted result (a or b).
// first_unstable: the caller's input order does not matter (full-key sorts),
// so the first pass may be a non-stable partition (partition_pass).
uint64_t* radix_sort(uint64_t* a, uint64_t* b, int64_t n, const SortPlan& plan, SortHist h,
                     const char* phase, bool first_unstable = false);

// bucket_build.cu
void partition_pass(const uint64_t* in, uint64_t* out, int64_t n, int shift, int bits,
                    const int64_t* d_digit_base);

}  // namespace gt

namespace gtd {

// ---- block-level helpers (256 threads) -------------------------------------

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive scan across a 256-thread block; `sm` needs 8 slots of T.
// Also returns the block total in `total`. Contains __syncthreads.
template <typename T>
__device__ __forceinline__ T block_excl_scan_256(T v, T* sm, T& total) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  T inc = warp_incl_scan(v);
  if (l == 31) sm[w] = inc;
  __syncthreads();
  T wpre = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    T x = sm[i];
    if (i < w) wpre += x;
    tot += x;
  }
  __syncthreads();
  total = tot;
  return wpre + inc - v;
}

// Deterministic block sum (fixed tree) across NW warps; `sm` needs NW slots.
template <int NW, typename T>
__device__ __forceinline__ T block_sum_warps(T v, T* sm) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_sum(v);
  if (l == 0) sm[w] = v;
  __syncthreads();
  T tot = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) tot += sm[i];
  __syncthreads();
  return tot;
}

// Deterministic block sum (fixed tree) across 256 threads.
template <typename T>
__device__ __forceinline__ T block_sum_256(T v, T* sm) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_sum(v);
  if (l == 0) sm[w] = v;
  __syncthreads();
  T tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot += sm[i];
  __syncthreads();
  return tot;
}

// Accumulate the digits of `key` for all passes of a plan into a block-local
// shared histogram sh[passes][256].
__device__ __forceinline__ void plan_hist_add(uint32_t* sh, const gt::SortPlan& p, uint64_t key) {
#pragma unroll
  for (int q = 0; q < gt::RS_MAX_PASSES; ++q) {
    if (q < p.passes) {
      uint32_t d = uint32_t(key >> p.shift[q]) & ((1u << p.bits[q]) - 1u);
      atomicAdd(&sh[q * 256 + d], 1u);
    }
  }
}

__device__ __forceinline__ void plan_hist_flush(const uint32_t* sh, const gt::SortPlan& p,
                                                unsigned long long* g) {
  for (int i = threadIdx.x; i < p.passes * 256; i += blockDim.x) {
    uint32_t c = sh[i];
    if (c) atomicAdd(&g[i], (unsigned long long)c);
  }
}

}  // namespace gtd
