// scan.cu — exclusive scan of int64 counts (see scan.cuh).
#include "radix_sort.cuh"
#include "scan.cuh"

namespace gtd {

constexpr int SCAN_PER = 8;
constexpr int SCAN_TILE = 256 * SCAN_PER;

__global__ void __launch_bounds__(256) scan_i64_kernel(int64_t* __restrict__ data, int64_t n,
                                                       uint64_t* __restrict__ status,
                                                       uint32_t* __restrict__ counter,
                                                       uint32_t epoch,
                                                       int64_t* __restrict__ total_out) {
  __shared__ uint32_t s_tile;
  __shared__ int64_t s_scan[8];
  __shared__ uint64_t s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = int(s_tile);
  const int64_t first = int64_t(tile) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_PER;
  int64_t v[SCAN_PER];
  int64_t sum = 0;
#pragma unroll
  for (int j = 0; j < SCAN_PER; ++j) {
    v[j] = first + j < n ? data[first + j] : 0;
    sum += v[j];
  }
  int64_t tot;
  const int64_t ex = block_excl_scan_256<int64_t>(sum, s_scan, tot);
  if (threadIdx.x == 0) s_excl = lookback_single(status, tile, epoch, uint64_t(tot));
  __syncthreads();
  int64_t run = int64_t(s_excl) + ex;
#pragma unroll
  for (int j = 0; j < SCAN_PER; ++j) {
    if (first + j < n) data[first + j] = run;
    run += v[j];
  }
  if (first <= n - 1 && n - 1 < first + SCAN_PER) {
    data[n] = run;
    *total_out = run;
  }
}

}  // namespace gtd

namespace gt {

void exclusive_scan_i64(int64_t* data, int64_t n, int64_t* total_out) {
  if (n <= 0) {
    GT_CUDA(cudaMemsetAsync(total_out, 0, 8, ctx().stream));
    GT_CUDA(cudaMemsetAsync(data, 0, 8, ctx().stream));
    return;
  }
  const int64_t tiles = ceil_div64(n, gtd::SCAN_TILE);
  uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) * 256);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  GT_CUDA(cudaMemsetAsync(counters + 30, 0, 4, ctx().stream));
  GT_LAUNCH(gtd::scan_i64_kernel, static_cast<int>(tiles), 256, 0, data, n, status, counters + 30,
            next_epoch(), total_out);
}

}  // namespace gt
