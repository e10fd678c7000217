// ubench_r2.cu — round-2 design probes on B200 (not product code).
//
//  part : non-stable MSD partition pass of 64-bit keys (the candidate build
//         primitive) — plain shared atomics vs MATCH-aggregated ranking,
//         8/9/10-bit digits, on R-MAT-skewed keys.
//  cub  : CUB onesweep SortKeys on the same keys (calibration only: what a
//         tuned stable LSD pass reaches on this part).
//  gather: random fp64 gathers (the PageRank SpMV bound): LDG (L1 allocate /
//         no-allocate) vs TMA tile::gather4 into shared memory.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//        -o ubench_r2 ubench_r2.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// R-MAT-like key: src/dst of `scale` bits each, (src<<scale)|dst, src ids
// scrambled by a multiplicative bijection (like the permuted configs).
__global__ void gen_keys(uint64_t* k, int64_t n, int scale, uint64_t seed) {
  const uint64_t ta = uint64_t(0.57 * 9007199254740992.0), tab = uint64_t(0.76 * 9007199254740992.0),
                 tabc = uint64_t(0.95 * 9007199254740992.0);
  const uint64_t m = (1ull << scale) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t s = 0, d = 0;
    for (int l = 0; l < scale; ++l) {
      uint64_t u = sm64(seed + uint64_t(i) * 64 + l) >> 11;
      int q = u < ta ? 0 : u < tab ? 1 : u < tabc ? 2 : 3;
      s = (s << 1) | (q >> 1);
      d = (d << 1) | (q & 1);
    }
    s = (s * 0x9E3779B1ull) & m;
    d = (d * 0x85EBCA77ull) & m;
    k[i] = (s << scale) | d;
  }
}

// ----------------------------------------------------------------- partition
template <int BITS>
__global__ void __launch_bounds__(256) hist_kernel(const uint64_t* __restrict__ k, int64_t n,
                                                   int shift, unsigned long long* __restrict__ h) {
  constexpr int D = 1 << BITS;
  __shared__ uint32_t sh[D];
  for (int i = threadIdx.x; i < D; i += 256) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(256) + threadIdx.x; i < n; i += int64_t(gridDim.x) * 256)
    atomicAdd(&sh[(k[i] >> shift) & (D - 1)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < D; i += 256)
    if (sh[i]) atomicAdd(&h[i], (unsigned long long)sh[i]);
}

__global__ void scan_kernel(const unsigned long long* h, unsigned long long* cur, int D) {
  if (threadIdx.x == 0) {
    unsigned long long r = 0;
    for (int i = 0; i < D; ++i) { cur[i] = r; r += h[i]; }
  }
}

// MODE 0: per-lane shared atomics; MODE 1: MATCH-aggregated leader atomics
template <int BITS, int KPT, int MODE>
__global__ void __launch_bounds__(256) part_kernel(const uint64_t* __restrict__ in,
                                                   uint64_t* __restrict__ out, int64_t n,
                                                   int shift,
                                                   unsigned long long* __restrict__ cursor) {
  constexpr int D = 1 << BITS, T = 256 * KPT;
  extern __shared__ __align__(16) unsigned char dsm[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_keys + T);
  int64_t* s_g = reinterpret_cast<int64_t*>(s_cnt + D + 32);
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t ntiles = (n + T - 1) / T;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T;
    const int valid = int((n - base) < T ? (n - base) : T);
    for (int i = tid; i < D; i += 256) s_cnt[i] = 0;
    __syncthreads();
    uint64_t k[KPT];
    uint32_t slot[KPT];
#pragma unroll
    for (int i = 0; i < KPT; i += 2) {
      const int j = (i / 2) * 512 + 2 * tid;
      if (j + 1 < valid) {
        const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in + base + j));
        k[i] = v.x;
        k[i + 1] = v.y;
      } else {
        k[i] = j < valid ? in[base + j] : ~0ull;
        k[i + 1] = ~0ull;
      }
    }
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int j = (i / 2) * 512 + 2 * tid + (i & 1);
      const bool ok = j < valid;
      const uint32_t d = uint32_t(k[i] >> shift) & (D - 1);
      if (MODE == 0) {
        slot[i] = ok ? atomicAdd(&s_cnt[d], 1u) : 0u;
      } else {
        const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0xFFFFFFFFu);
        const int leader = 31 - __clz(peers);
        uint32_t b = 0;
        if (ok && lane == leader) b = atomicAdd(&s_cnt[d], __popc(peers));
        b = __shfl_sync(0xffffffffu, b, leader);
        slot[i] = b + __popc(peers & lt);
      }
    }
    __syncthreads();
    // in-tile starts (exclusive scan over D counts) + global reservation
    {
      constexpr int PER = (D + 255) / 256;
      uint32_t c[PER], sum = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int d = tid * PER + q;
        c[q] = d < D ? s_cnt[d] : 0u;
        sum += c[q];
      }
      // block exclusive scan of `sum`
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      uint32_t* s_w = s_cnt + D;
      if (lane == 31) s_w[tid >> 5] = inc;
      __syncthreads();
      uint32_t wpre = 0;
      for (int w = 0; w < (tid >> 5); ++w) wpre += s_w[w];
      uint32_t run = wpre + inc - sum;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int d = tid * PER + q;
        if (d < D) {
          int64_t g = 0;
          if (c[q]) g = int64_t(atomicAdd(&cursor[d], (unsigned long long)c[q]));
          s_g[d] = g - int64_t(run);
          s_cnt[d] = run;
        }
        run += c[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int j = (i / 2) * 512 + 2 * tid + (i & 1);
      if (j < valid) s_keys[s_cnt[uint32_t(k[i] >> shift) & (D - 1)] + slot[i]] = k[i];
    }
    __syncthreads();
    for (int j = tid; j < valid; j += 256) {
      const uint64_t key = s_keys[j];
      out[s_g[uint32_t(key >> shift) & (D - 1)] + j] = key;
    }
    __syncthreads();
  }
}

template <int BITS, int KPT, int MODE>
float run_part(const uint64_t* in, uint64_t* out, int64_t n, int shift,
               unsigned long long* hist, unsigned long long* cur, int sms, int occ) {
  constexpr int D = 1 << BITS, T = 256 * KPT;
  const size_t smem = size_t(T) * 8 + (D + 32) * 4 + D * 8;
  CK(cudaFuncSetAttribute(part_kernel<BITS, KPT, MODE>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, part_kernel<BITS, KPT, MODE>, 256, smem));
  const int blocks = sms * (occ > 0 ? std::min(occ, maxb) : maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemset(hist, 0, D * 8));
    hist_kernel<BITS><<<sms * 4, 256>>>(in, n, shift, hist);
    scan_kernel<<<1, 32>>>(hist, cur, D);
    cudaEventRecord(a);
    part_kernel<BITS, KPT, MODE><<<blocks, 256, smem>>>(in, out, n, shift, cur);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  printf("part bits=%d kpt=%d mode=%s occ=%d blocks=%d: %.3f ms  %.1f GB/s (16 B/key)\n", BITS,
         KPT, MODE ? "match" : "atomic", maxb, blocks, best, 16.0 * n / best / 1e6);
  return best;
}

// verify: every output digit run matches the histogram order
__global__ void check_part(const uint64_t* out, int64_t n, int shift, int D, int* bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i + 1 < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (((out[i] >> shift) & (D - 1)) > ((out[i + 1] >> shift) & (D - 1))) atomicAdd(bad, 1);
}

// -------------------------------------------------------------------- gather
__global__ void gen_idx(int32_t* idx, int64_t e, int32_t n, int skew, uint64_t seed) {
  const double ln = log(double(n));
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < e;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double u = double(sm64(seed + i) >> 11) / 9007199254740992.0;
    int64_t v = skew ? int64_t(exp(u * ln)) - 1 : int64_t(u * n);
    idx[i] = int32_t(v < 0 ? 0 : (v >= n ? n - 1 : v));
  }
}

template <int NA>
__global__ void __launch_bounds__(256) gather_ldg(const int32_t* __restrict__ idx, int64_t e,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ out) {
  double acc = 0;
  const int64_t stride = int64_t(gridDim.x) * 256 * 8;
  for (int64_t i = (blockIdx.x * int64_t(256) + threadIdx.x) * 8; i < e; i += stride) {
    const int4 a = __ldcs(reinterpret_cast<const int4*>(idx + i));
    const int4 b = __ldcs(reinterpret_cast<const int4*>(idx + i + 4));
    const int j[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (NA) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[q]) : "l"(x + j[q]));
      else v[q] = __ldg(x + j[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += v[q];
  }
  if (acc == 12345.678) out[0] = acc;
}

// TMA gather4: x viewed as [n/2][2] doubles (16-B rows); each lane gathers the
// 4 rows holding its 4 indices into shared memory (64 B), 2 stages per warp.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__global__ void __launch_bounds__(128) gather_tma4(const __grid_constant__ CUtensorMap tm,
                                                   const int32_t* __restrict__ idx, int64_t e,
                                                   double* __restrict__ out) {
  __shared__ __align__(128) double buf[4][2][32 * 16];  // warp, stage, lane*16 doubles (128 B)
  __shared__ __align__(8) uint64_t bar[4][2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int s = 0; s < 2; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = blockIdx.x * 4 + w, nwarps = int64_t(gridDim.x) * 4;
  const int64_t per = 128;  // indices per warp round
  uint32_t phase[2] = {0, 0};
  double acc = 0;
  int64_t r = gw * per;
  auto issue = [&](int s, int64_t at) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_u32(&bar[w][s])), "r"(32 * 64) : "memory");
    __syncwarp();
    const int4 q = *reinterpret_cast<const int4*>(idx + at + lane * 4);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&buf[w][s][lane * 16])),
        "l"(&tm), "r"(0), "r"(q.x >> 1), "r"(q.y >> 1), "r"(q.z >> 1), "r"(q.w >> 1),
        "r"(smem_u32(&bar[w][s]))
        : "memory");
  };
  int s = 0;
  if (r < e) issue(0, r);
  while (r < e) {
    const int64_t nx = r + nwarps * per;
    if (nx < e) issue(s ^ 1, nx);
    // wait stage s
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[w][s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    const int4 q = *reinterpret_cast<const int4*>(idx + r + lane * 4);
    const double* b = &buf[w][s][lane * 16];
    acc += b[0 + (q.x & 1)] + b[2 + (q.y & 1)] + b[4 + (q.z & 1)] + b[6 + (q.w & 1)];
    __syncwarp();
    r = nx;
    s ^= 1;
  }
  if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const char* what = argc > 1 ? argv[1] : "all";
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  printf("SMs %d\n", sms);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);

  if (!strcmp(what, "all") || !strcmp(what, "part") || !strcmp(what, "cub")) {
    const int64_t n = int64_t(1470) * 1000 * 1000;
    const int scale = 26;
    uint64_t *k0, *k1;
    unsigned long long *hist, *cur;
    CK(cudaMalloc(&k0, n * 8));
    CK(cudaMalloc(&k1, n * 8));
    CK(cudaMalloc(&hist, 1024 * 8));
    CK(cudaMalloc(&cur, 1024 * 8));
    int* bad;
    CK(cudaMalloc(&bad, 4));
    gen_keys<<<sms * 8, 256>>>(k0, n, scale, 3);
    CK(cudaDeviceSynchronize());
    if (strcmp(what, "cub")) {
      const int top = 2 * scale;
      auto chk = [&](int bits) {
        CK(cudaMemset(bad, 0, 4));
        check_part<<<sms * 8, 256>>>(k1, n, top - bits, 1 << bits, bad);
        int h;
        CK(cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost));
        printf("  check: %d inversions\n", h);
      };
      run_part<8, 16, 0>(k0, k1, n, top - 8, hist, cur, sms, 0); chk(8);
      run_part<8, 16, 1>(k0, k1, n, top - 8, hist, cur, sms, 0); chk(8);
      run_part<9, 16, 0>(k0, k1, n, top - 9, hist, cur, sms, 0); chk(9);
      run_part<9, 16, 1>(k0, k1, n, top - 9, hist, cur, sms, 0); chk(9);
      run_part<10, 16, 0>(k0, k1, n, top - 10, hist, cur, sms, 0); chk(10);
      run_part<10, 16, 1>(k0, k1, n, top - 10, hist, cur, sms, 0); chk(10);
      run_part<9, 8, 0>(k0, k1, n, top - 9, hist, cur, sms, 0);
      run_part<9, 24, 0>(k0, k1, n, top - 9, hist, cur, sms, 0);
      run_part<9, 32, 0>(k0, k1, n, top - 9, hist, cur, sms, 0);
      // second-level digit (bits below the top 9): less skew
      run_part<9, 16, 0>(k0, k1, n, top - 18, hist, cur, sms, 0);
      run_part<9, 16, 1>(k0, k1, n, top - 18, hist, cur, sms, 0);
    }
    {  // CUB onesweep calibration (stable LSD, 8-bit digits)
      size_t tmp = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0, k1, n, 0, 52);
      void* t;
      CK(cudaMalloc(&t, tmp));
      for (int nb : {8, 16, 52}) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          cub::DeviceRadixSort::SortKeys(t, tmp, k0, k1, n, 0, nb);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep) best = std::min(best, ms);
        }
        const int passes = (nb + 7) / 8;
        printf("cub SortKeys u64 bits=%d: %.3f ms  (%d passes; %.1f GB/s at 16 B/key/pass + 8 B hist)\n",
               nb, best, passes, (16.0 * passes + 8.0) * n / best / 1e6);
      }
      cudaFree(t);
    }
    cudaFree(k0);
    cudaFree(k1);
  }

  if (!strcmp(what, "all") || !strcmp(what, "gather")) {
    const int32_t nn = 35400000;
    const int64_t e = int64_t(1) << 30;
    double *x, *o;
    int32_t* idx;
    CK(cudaMalloc(&x, size_t(nn + 16) * 8));
    CK(cudaMalloc(&o, 64));
    CK(cudaMalloc(&idx, e * 4));
    CK(cudaMemset(x, 0, size_t(nn + 16) * 8));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, cuuint64_t((nn + 1) / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = reinterpret_cast<EncodeTiled>(fn)(
        &tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map encode: %d\n", int(cr));
    const int nsk = (argc > 3) ? 3 : 2;
    for (int skew = 0; skew < nsk; ++skew) {
      // skew 2: uniform over the first 8M doubles (64 MB: L2-resident)
      gen_idx<<<sms * 8, 256>>>(idx, e, skew == 2 ? (8 << 20) : nn, skew == 1, 7);
      CK(cudaDeviceSynchronize());
      for (int v = 0; v < 3; ++v) {
        if (v == 2 && (cr != CUDA_SUCCESS || (argc > 2 && !strcmp(argv[2], "notma")))) continue;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          if (v == 0) gather_ldg<0><<<sms * 8, 256>>>(idx, e, x, o);
          else if (v == 1) gather_ldg<1><<<sms * 8, 256>>>(idx, e, x, o);
          else gather_tma4<<<sms * 8, 128>>>(tm, idx, e, o);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          CK(cudaGetLastError());
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep) best = std::min(best, ms);
        }
        printf("gather %s %s: %.3f ms  %.1f G gathers/s  %.3f gathers/cycle/SM@1.965GHz\n",
               skew == 2 ? "uniform64MB" : skew ? "logskew" : "uniform", v == 0 ? "ldg" : v == 1 ? "ldg.na" : "tma.gather4",
               best, e / best / 1e6, e / best / 1e6 / (sms * 1.965));
      }
    }
  }
  return 0;
}
