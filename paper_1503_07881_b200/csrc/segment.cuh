// segment.cuh — sorted packed keys (row<<k | col) -> CSR rows.
//
// Shared by the ToGraph build (out- and in-CSR, convert.py:154-164) and the
// triangle-count orientation (oriented CSR). One tile = 4096 keys read once;
// kept positions come from warp ballots + decoupled look-back, row offsets
// are written at row starts (empty rows filled warp-cooperatively).
#pragma once

#include "radix_sort.cuh"

namespace gtd {

using gt::SortPlan;

constexpr int SEG_KPT = 16;
#ifndef GT_SEG_MIN_CTAS
#define GT_SEG_MIN_CTAS 4
#endif
constexpr int SEG_MIN_CTAS = GT_SEG_MIN_CTAS;  // resident CTAs per SM the register budget is sized for
constexpr int SEG_TILE = 256 * SEG_KPT;

// Warp-cooperative fill of off[first..last] = v for the lanes that own a gap.
__device__ __forceinline__ void warp_fill_gaps(bool have, int64_t first, int64_t last, int64_t v,
                                               int64_t* __restrict__ off) {
  uint32_t m = __ballot_sync(0xffffffffu, have);
  while (m) {
    const int l = __ffs(m) - 1;
    m &= m - 1;
    const int64_t f = __shfl_sync(0xffffffffu, first, l);
    const int64_t e = __shfl_sync(0xffffffffu, last, l);
    const int64_t val = __shfl_sync(0xffffffffu, v, l);
    for (int64_t r = f + (threadIdx.x & 31); r <= e; r += 32) off[r] = val;
  }
}

// Sorted packed keys -> CSR rows. DEDUPE: drop repeated keys (convert.py:76-80)
// and emit in-keys (dst<<k|src); the kept keys before each tile come from
// dedupe_count_kernel + a scan (tile_base[t], tile_base[tiles] = total), so no
// tile waits on its predecessors.
template <bool DEDUPE>
__global__ void __launch_bounds__(256, SEG_MIN_CTAS) segment_kernel(
    const uint64_t* __restrict__ keys, int64_t n, int kbits, int64_t n_rows,
    int32_t* __restrict__ adj, int64_t* __restrict__ off, uint64_t* __restrict__ in_keys,
    const int64_t* __restrict__ tile_base) {
  __shared__ uint32_t s_warp[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = int(blockIdx.x);
  const int64_t wbase = int64_t(tile) * SEG_TILE + int64_t(warp) * 32 * SEG_KPT;
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
  uint32_t kept_before[SEG_KPT];  // warp-local kept count before item i (dedupe)
  uint32_t keep_bits = 0, row_bits = 0;
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    const bool valid = idx < n;
    uint64_t prev = __shfl_up_sync(0xffffffffu, k[i], 1);
    const uint64_t last_prev = __shfl_sync(0xffffffffu, i > 0 ? k[i > 0 ? i - 1 : 0] : first_prev, 31);
    if (lane == 0) prev = (i == 0) ? first_prev : last_prev;
    const bool has_prev = idx > 0;
    const bool keep = valid && (!DEDUPE || !has_prev || k[i] != prev);
    const bool newrow = valid && (!has_prev || (k[i] >> kbits) != (prev >> kbits));
    keep_bits |= uint32_t(keep) << i;
    row_bits |= uint32_t(newrow) << i;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    kept_before[i] = run + __popc(bal & lt);
    run += __popc(bal);
  }

  int64_t base_pos;  // position of this warp's first kept item
  int64_t total = n;
  if (DEDUPE) {
    if (lane == 0) s_warp[warp] = run;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w)
      if (w < warp) wpre += s_warp[w];
    base_pos = tile_base[tile] + wpre;
    total = tile_base[gridDim.x];
  } else {
    base_pos = wbase;
  }

#pragma unroll
  for (int i = 0; i < SEG_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    const bool keep = (keep_bits >> i) & 1u;
    const bool newrow = (row_bits >> i) & 1u;
    const int64_t pos = DEDUPE ? base_pos + kept_before[i] : idx;
    const int64_t row = int64_t(k[i] >> kbits);
    const uint64_t col = k[i] & lowmask;
    if (keep) {
      adj[pos] = int32_t(col);
      if (DEDUPE) in_keys[pos] = (col << kbits) | uint64_t(row);
    }
    // Row starts: rows (prev_row, row] begin at pos (empty rows share it).
    uint64_t prev = __shfl_up_sync(0xffffffffu, k[i], 1);
    const uint64_t last_prev = __shfl_sync(0xffffffffu, i > 0 ? k[i > 0 ? i - 1 : 0] : first_prev, 31);
    if (lane == 0) prev = (i == 0) ? first_prev : last_prev;
    const int64_t prev_row = idx > 0 ? int64_t(prev >> kbits) : -1;
    const bool single = newrow && row - prev_row == 1;
    if (single) off[row] = pos;
    warp_fill_gaps(newrow && !single, prev_row + 1, row, pos, off);
    // Trailing rows (last_row, n_rows] end at the edge count.
    const bool tail = idx == n - 1;
    warp_fill_gaps(tail, row + 1, n_rows, total, off);
  }
}

}  // namespace gtd
