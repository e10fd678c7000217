// merge.cu — stable merge of sorted key runs (multi-GPU build, receive side).
//
// After the row shuffle of the sharded build every rank holds `world` runs,
// one per source rank, each already sorted (distributed.py: build_csr). The
// reference re-sorts the concatenation (parallel.py:52-93 sample sort: the
// received buckets go through np.sort again); here the runs are merged
// pairwise instead: ceil(log2 runs) merge rounds of 16 B/key each, against
// 16 B/key for every 8-bit radix pass of a re-sort (2k/8 passes, k the key
// half width).
//
// One round merges run pairs (0,1), (2,3), ... with a merge-path kernel: each
// CTA owns a tile of 2048 outputs, finds where its tile boundaries cut the two
// runs by binary search along the cross diagonal, stages both slices in
// shared memory with coalesced loads, and every thread merges 8 outputs
// serially from its own diagonal. Ties take the left run first (stable).
#include "common.cuh"

#include <vector>

namespace gtd {

constexpr int MG_THREADS = 256;
constexpr int MG_VT = 8;
constexpr int MG_TILE = MG_THREADS * MG_VT;

// Number of a-items among the first d outputs of merge(a, b), a before b on ties.
template <typename Ptr, typename Idx>
__device__ __forceinline__ Idx merge_path(Ptr a, Idx na, Ptr b, Idx nb, Idx d) {
  Idx lo = d > nb ? d - nb : Idx(0);
  Idx hi = d < na ? d : na;
  while (lo < hi) {
    const Idx mid = (lo + hi) >> 1;
    if (a[mid] <= b[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(MG_THREADS)
merge_pair_kernel(const uint64_t* __restrict__ a, int64_t na, const uint64_t* __restrict__ b,
                  int64_t nb, uint64_t* __restrict__ c) {
  __shared__ uint64_t s[MG_TILE];
  __shared__ int64_t cut[2];
  const int64_t n = na + nb;
  const int64_t d0 = int64_t(blockIdx.x) * MG_TILE;
  const int64_t d1 = d0 + MG_TILE < n ? d0 + MG_TILE : n;
  if (threadIdx.x < 2) cut[threadIdx.x] = merge_path(a, na, b, nb, threadIdx.x ? d1 : d0);
  __syncthreads();
  const int64_t i0 = cut[0], i1 = cut[1];
  const int la = int(i1 - i0), lb = int((d1 - i1) - (d0 - i0));
  const uint64_t* ga = a + i0;
  const uint64_t* gb = b + (d0 - i0);
  for (int k = threadIdx.x; k < la + lb; k += MG_THREADS) s[k] = k < la ? ga[k] : gb[k - la];
  __syncthreads();

  const int tot = la + lb;
  const int diag = min(int(threadIdx.x) * MG_VT, tot);
  int ia = merge_path(s, la, s + la, lb, diag);
  int ib = diag - ia;
  uint64_t out[MG_VT];
#pragma unroll
  for (int k = 0; k < MG_VT; ++k) {
    const bool take_a = ib >= lb || (ia < la && s[ia] <= s[la + ib]);
    const uint64_t va = ia < la ? s[ia] : 0, vb = ib < lb ? s[la + ib] : 0;
    out[k] = take_a ? va : vb;
    ia += take_a;
    ib += !take_a;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < MG_VT; ++k)
    if (diag + k < tot) s[diag + k] = out[k];
  __syncthreads();
  uint64_t* gc = c + d0;
  for (int k = threadIdx.x; k < tot; k += MG_THREADS) gc[k] = s[k];
}

}  // namespace gtd

namespace gt {

// Merge the runs [off[r], off[r+1]) of `a` (each sorted ascending) into one
// sorted sequence; `b` is scratch of n keys. Returns the buffer holding it.
static uint64_t* merge_runs(uint64_t* a, uint64_t* b, const std::vector<int64_t>& off) {
  std::vector<int64_t> cur = off;
  uint64_t* src = a;
  uint64_t* dst = b;
  while (cur.size() > 2) {
    const size_t runs = cur.size() - 1;
    std::vector<int64_t> next{0};
    for (size_t r = 0; r < runs; r += 2) {
      const int64_t lo = cur[r];
      if (r + 1 == runs) {  // odd run out: carried over unchanged
        const int64_t len = cur[r + 1] - lo;
        if (len)
          GT_CUDA(cudaMemcpyAsync(dst + lo, src + lo, size_t(len) * 8, cudaMemcpyDeviceToDevice,
                                  ctx().stream));
        next.push_back(cur[r + 1]);
        continue;
      }
      const int64_t na = cur[r + 1] - lo, nb = cur[r + 2] - cur[r + 1];
      if (na + nb)
        GT_LAUNCH(gtd::merge_pair_kernel, ceil_div(na + nb, gtd::MG_TILE), gtd::MG_THREADS, 0,
                  src + lo, na, src + cur[r + 1], nb, dst + lo);
      next.push_back(cur[r + 2]);
    }
    cur.swap(next);
    std::swap(src, dst);
  }
  return src;
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_merge_runs(uint64_t* d_keys, uint64_t* d_tmp, int64_t n, const int64_t* h_run_off,
                  int nruns, int* result_in_tmp) {
  GT_API_BEGIN
  require_init();
  if (!result_in_tmp || !h_run_off || nruns < 1) fail(GT_EINVAL, "bad arguments");
  if (h_run_off[0] != 0 || h_run_off[nruns] != n) fail(GT_EINVAL, "run offsets must span [0, n)");
  for (int r = 0; r < nruns; ++r)
    if (h_run_off[r + 1] < h_run_off[r]) fail(GT_EINVAL, "run offsets must be non-decreasing");
  std::vector<int64_t> off(h_run_off, h_run_off + nruns + 1);
  Phase ph("dist.merge", 0);
  uint64_t* out = merge_runs(d_keys, d_tmp, off);
  *result_in_tmp = out == d_tmp ? 1 : 0;
  sync();
  GT_API_END
}

}  // extern "C"
