// radix_sort.cu — onesweep LSD radix sort (see radix_sort.cuh).
#include "radix_sort.cuh"

#include <algorithm>

namespace gtd {

using gt::RS_KPT;
using gt::RS_THREADS;
using gt::RS_TILE;

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

__global__ void __launch_bounds__(RS_THREADS, 3)
    onesweep_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t n,
                    int shift, int bits, const int64_t* __restrict__ digit_base,
                    uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter,
                    uint32_t epoch) {
  constexpr int NW = RS_THREADS / 32;
  __shared__ union {
    uint64_t keys[RS_TILE];
    uint32_t whist[NW][256];
  } s;
  __shared__ int64_t s_gbase[256];
  __shared__ uint32_t s_scan[8];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < NW * 256; i += RS_THREADS) (&s.whist[0][0])[i] = 0;
  __syncthreads();
  const int tile = int(s_tile);
  const int64_t base = int64_t(tile) * RS_TILE;
  const int64_t wbase = base + int64_t(warp) * 32 * RS_KPT;
  const uint32_t mask = (1u << bits) - 1u;

  uint64_t k[RS_KPT];
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    k[i] = idx < n ? ld_stream_u64(in + idx) : ~0ull;
  }

  // Warp-level multi-split: rank every key among the equal digits of its
  // warp in lane order (stable). __match_any_sync finds the peers of a digit
  // in one instruction; invalid tail keys match only each other (digit 256).
  uint32_t rank[RS_KPT];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) {
    const bool valid = (wbase + i * 32 + lane) < n;
    const uint32_t d = valid ? uint32_t(k[i] >> shift) & mask : 256u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = 0;
    if (valid) before = s.whist[warp][d];
    rank[i] = before + __popc(peers & lt);
    const int leader = 31 - __clz(peers);
    __syncwarp();
    if (valid && lane == leader) s.whist[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // Per digit (thread == digit): warp offsets, tile count, look-back.
  {
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

    uint32_t tot;
    const uint32_t local_start = block_excl_scan_256<uint32_t>(tile_cnt, s_scan, tot);

    uint64_t excl = 0;
    if (tile > 0) {
      const uint64_t ep = uint64_t(epoch & 0x3FFFFFu);
      int t = tile - 1;
      while (true) {
        const uint64_t v = ld_status_u64(status + int64_t(t) * 256 + d);
        if (((v >> 40) & 0x3FFFFFu) != ep || (v >> 62) == 0) continue;
        excl += v & ((1ull << 40) - 1);
        if ((v >> 62) == 2) break;
        --t;
      }
      st_status_u64(st, lb_pack(LB_INC, epoch, excl + tile_cnt));
    }
    s_gbase[d] = digit_base[d] + int64_t(excl) - int64_t(local_start);
#pragma unroll
    for (int w = 0; w < NW; ++w) s.whist[w][d] += local_start;
  }
  __syncthreads();

  uint32_t pos[RS_KPT];
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i) {
    const uint32_t d = uint32_t(k[i] >> shift) & mask;
    pos[i] = s.whist[warp][d] + rank[i];
  }
  __syncthreads();  // whist aliases the key staging buffer
#pragma unroll
  for (int i = 0; i < RS_KPT; ++i)
    if (wbase + i * 32 + lane < n) s.keys[pos[i]] = k[i];
  __syncthreads();

  const int nvalid = (n - base) < RS_TILE ? int(n - base) : RS_TILE;
  for (int j = tid; j < nvalid; j += RS_THREADS) {
    const uint64_t key = s.keys[j];
    const uint32_t d = uint32_t(key >> shift) & mask;
    out[s_gbase[d] + j] = key;
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

uint64_t* radix_sort(uint64_t* a, uint64_t* b, int64_t n, const SortPlan& plan, SortHist h,
                     const char* phase) {
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
  for (int q = 0; q < plan.passes; ++q) {
    Phase ph(phase, 16.0 * n);
    const uint32_t epoch = next_epoch();
    GT_LAUNCH(gtd::onesweep_kernel, static_cast<int>(tiles), RS_THREADS, 0, src, dst, n,
              plan.shift[q], plan.bits[q], h.digit_base + q * 256, status, counters + q, epoch);
    std::swap(src, dst);
  }
  return src;
}

}  // namespace gt
