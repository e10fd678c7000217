// rmat.cu — counter-based R-MAT edge generator (bench / test inputs).
//
// The reference ships only a uniform generator (synth.py:20-29); BASELINE.json
// configs 1-4 are R-MAT tables, so both sides generate them from this
// definition (numpy twin: paper_1503_07881_b200/synth.py:rmat_edges):
//   key      = splitmix64(seed ^ 0x5851F42D4C957F2D)
//   x(e, l)  = splitmix64(key + e*scale + l)            l = 0 .. scale-1 (MSB first)
//   u        = x >> 11                                   (53-bit uniform)
//   quadrant = a if u < A, b if u < A+B, c if u < A+B+C, else d
//              (A, A+B, A+B+C = thresholds * 2^53; b sets the dst bit,
//               c the src bit, d both)
//   permute  : 4-round Feistel on 2h bits (h = ceil(scale/2)), round key
//              splitmix64(key ^ (0xA0761D6478BD642F * (r+1))), cycle-walked
//              into [0, 2^scale).
#include "common.cuh"

#include <algorithm>

namespace gtd {

struct RmatParams {
  int scale;
  int h;
  uint64_t key;
  uint64_t ta, tab, tabc;
  uint64_t rk[4];
};

__device__ __forceinline__ uint64_t feistel_perm(uint64_t x, const RmatParams& p) {
  const uint64_t mh = (1ull << p.h) - 1ull;
  const uint64_t limit = 1ull << p.scale;
  do {
    uint64_t L = x >> p.h, R = x & mh;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t nl = R;
      R = L ^ (splitmix64(R ^ p.rk[r]) & mh);
      L = nl;
    }
    x = (L << p.h) | R;
  } while (x >= limit);
  return x;
}

__global__ void __launch_bounds__(256) rmat_kernel(int64_t start, int64_t rows, RmatParams p,
                                                   int permute,
                                                   int64_t* __restrict__ src,
                                                   int64_t* __restrict__ dst) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows; e += stride) {
    uint64_t s = 0, d = 0;
    const uint64_t base = p.key + uint64_t(start + e) * uint64_t(p.scale);
    for (int l = 0; l < p.scale; ++l) {
      const uint64_t u = splitmix64(base + uint64_t(l)) >> 11;
      const uint64_t sb = u >= p.tab ? 1ull : 0ull;                  // quadrants c, d
      const uint64_t db = (u >= p.ta && u < p.tab) || u >= p.tabc;   // quadrants b, d
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    if (permute) {
      s = feistel_perm(s, p);
      d = feistel_perm(d, p);
    }
    src[e] = int64_t(s);
    dst[e] = int64_t(d);
  }
}

// Uniform (Erdős–Rényi) rows, the stand-in for BASELINE config 4's
// synth.random_edges table (numpy twin: synth.uniform_edges):
//   key = splitmix64(seed ^ 0xD1B54A32D192ED03)
//   src = hi64(splitmix64(key + 2e) * n),  dst = hi64(splitmix64(key + 2e + 1) * n)
__global__ void __launch_bounds__(256) uniform_kernel(int64_t start, int64_t rows, uint64_t key,
                                                      uint64_t n, int64_t* __restrict__ src,
                                                      int64_t* __restrict__ dst) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows; e += stride) {
    const uint64_t b = key + 2ull * uint64_t(start + e);
    src[e] = int64_t(__umul64hi(splitmix64(b), n));
    dst[e] = int64_t(__umul64hi(splitmix64(b + 1ull), n));
  }
}

}  // namespace gtd

using namespace gt;

extern "C" int gt_uniform_generate_range(int64_t n_nodes, int64_t start, int64_t rows,
                                         uint64_t seed, int64_t* d_src, int64_t* d_dst) {
  GT_API_BEGIN
  require_init();
  if (n_nodes < 1 || rows < 0 || start < 0) fail(GT_EINVAL, "need n_nodes >= 1, rows >= 0");
  if (rows == 0) return GT_OK;
  if (!d_src || !d_dst) fail(GT_EINVAL, "output pointers must not be NULL");
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div64(rows, 256), 16LL * ctx().sm_count));
  {
    Phase ph("synth.uniform", 16.0 * rows);
    GT_LAUNCH(gtd::uniform_kernel, grid, 256, 0, start, rows,
              gtd::splitmix64(seed ^ 0xD1B54A32D192ED03ull), uint64_t(n_nodes), d_src, d_dst);
  }
  sync();
  GT_API_END
}

extern "C" int gt_rmat_generate_range(int scale, int64_t start, int64_t rows, double a, double b,
                                      double c, uint64_t seed, int permute, int64_t* d_src,
                                      int64_t* d_dst) {
  GT_API_BEGIN
  require_init();
  if (scale < 1 || scale > 40) fail(GT_EINVAL, "scale must be in [1, 40]");
  if (rows < 0 || start < 0) fail(GT_EINVAL, "rows and start must be >= 0");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
    fail(GT_EINVAL, "R-MAT probabilities must be >= 0 and a+b+c <= 1");
  if (rows == 0) return GT_OK;
  if (!d_src || !d_dst) fail(GT_EINVAL, "output pointers must not be NULL");
  gtd::RmatParams p;
  p.scale = scale;
  p.h = (scale + 1) / 2;
  p.key = gtd::splitmix64(seed ^ 0x5851F42D4C957F2Dull);
  const double two53 = 9007199254740992.0;
  p.ta = uint64_t(a * two53);
  p.tab = uint64_t((a + b) * two53);
  p.tabc = uint64_t((a + b + c) * two53);
  for (int r = 0; r < 4; ++r) p.rk[r] = gtd::splitmix64(p.key ^ (0xA0761D6478BD642Full * uint64_t(r + 1)));
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div64(rows, 256), 16LL * ctx().sm_count));
  {
    Phase ph("synth.rmat", 16.0 * rows);
    GT_LAUNCH(gtd::rmat_kernel, grid, 256, 0, start, rows, p, permute, d_src, d_dst);
  }
  sync();
  GT_API_END
}

extern "C" int gt_rmat_generate(int scale, int64_t rows, double a, double b, double c,
                                uint64_t seed, int permute, int64_t* d_src, int64_t* d_dst) {
  return gt_rmat_generate_range(scale, 0, rows, a, b, c, seed, permute, d_src, d_dst);
}
