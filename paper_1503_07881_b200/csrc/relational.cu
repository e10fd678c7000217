// relational.cu — device Select and Join feeding ToGraph.
//
// The reference builds the demo's edge table with two relational operators
// on host numpy columns (demo.py:40-44):
//   select (tables.py:325-344)  mask = cmp(column, constant); _take(flatnonzero(mask))
//   join   (tables.py:397-426)  hash join building on the smaller input; pairs
//                               come out in probe-row order, and for each probe
//                               row in ascending build-row order (the bucket
//                               lists are appended in row order, :413-421)
// Here both run on device-resident columns:
//   gt_select_rows   one pass counts the hits of every 2048-row tile, a
//                    decoupled-look-back scan turns the counts into offsets,
//                    a second pass writes the ascending row indices.
//   gt_gather_u64    _take / _paired_table (tables.py:232-240, 385-394): one
//                    8-byte column gathered by a row-index list, optionally
//                    through a code remap (merged string pools, tables.py:393).
//   gt_join_build    open-addressing hash table of the build keys (64-bit CAS),
//                    build rows grouped by slot with a stable radix sort over the
//                    slot bits only (row order inside a slot is kept), probe
//                    rows count their matches, an exclusive scan gives every
//                    probe row its output offset, and the pairs are expanded in
//                    the reference's order. Exact for every key, including
//                    collisions of the hash.
// Keys: INT and (pool-remapped) STRING columns compare as int64; FLOAT keys
// compare as Python floats do in a dict: -0.0 == 0.0, NaN never matches.
#include "graph.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"

#include <algorithm>

namespace gtd {

constexpr int SEL_THREADS = 256;
constexpr int SEL_PER = 8;
constexpr int SEL_TILE = SEL_THREADS * SEL_PER;

struct SelPred {
  int kind;  // 0 int64, 1 float64, 2 int64 code -> lut
  int op;    // GT_CMP_*
  int64_t iv;
  double fv;
  const uint8_t* lut;
  int64_t lut_n;
};

template <typename T>
__device__ __forceinline__ bool sel_cmp(T a, T b, int op) {
  switch (op) {
    case GT_CMP_EQ: return a == b;
    case GT_CMP_NE: return a != b;
    case GT_CMP_LT: return a < b;
    case GT_CMP_LE: return a <= b;
    case GT_CMP_GT: return a > b;
    default: return a >= b;
  }
}

__device__ __forceinline__ bool sel_eval(const void* col, int64_t i, const SelPred& p) {
  if (p.kind == 0) return sel_cmp<int64_t>(__ldcs(static_cast<const int64_t*>(col) + i), p.iv, p.op);
  if (p.kind == 1) return sel_cmp<double>(__ldcs(static_cast<const double*>(col) + i), p.fv, p.op);
  const int64_t code = __ldcs(static_cast<const int64_t*>(col) + i);
  return code >= 0 && code < p.lut_n && p.lut[code] != 0;
}

// Hits of each tile (rows tile*SEL_TILE + [0, SEL_TILE)).
__global__ void __launch_bounds__(SEL_THREADS) select_count_kernel(const void* col, int64_t n,
                                                                   SelPred p,
                                                                   int64_t* __restrict__ counts) {
  __shared__ int64_t s_red[8];
  const int64_t r0 = int64_t(blockIdx.x) * SEL_TILE + threadIdx.x;
  int64_t c = 0;
#pragma unroll
  for (int i = 0; i < SEL_PER; ++i) {
    const int64_t r = r0 + i * SEL_THREADS;
    if (r < n && sel_eval(col, r, p)) ++c;
  }
  c = block_sum_256(c, s_red);
  if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

// Ascending row indices of the hits: per slab of 256 rows, ballots give each
// hit its place among the slab's hits; slabs are laid out in order.
__global__ void __launch_bounds__(SEL_THREADS) select_write_kernel(const void* col, int64_t n,
                                                                   SelPred p,
                                                                   const int64_t* __restrict__ offs,
                                                                   int64_t* __restrict__ out) {
  __shared__ uint32_t s_w[SEL_PER][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = int64_t(blockIdx.x) * SEL_TILE + threadIdx.x;
  uint32_t hit = 0, below[SEL_PER];
#pragma unroll
  for (int i = 0; i < SEL_PER; ++i) {
    const int64_t r = r0 + i * SEL_THREADS;
    const bool h = r < n && sel_eval(col, r, p);
    const uint32_t b = __ballot_sync(0xffffffffu, h);
    below[i] = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) s_w[i][warp] = __popc(b);
    hit |= uint32_t(h) << i;
  }
  __syncthreads();
  int64_t base = offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SEL_PER; ++i) {
    uint32_t before = 0, slab = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t c = s_w[i][w];
      before += w < warp ? c : 0u;
      slab += c;
    }
    if ((hit >> i) & 1u) out[base + before + below[i]] = r0 + i * SEL_THREADS;
    base += slab;
  }
}

__global__ void __launch_bounds__(256) gather_u64_kernel(const uint64_t* __restrict__ src,
                                                         const int64_t* __restrict__ idx, int64_t n,
                                                         const int64_t* __restrict__ remap,
                                                         uint64_t* __restrict__ out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t j = idx ? __ldcs(idx + i) : i;
    uint64_t v = src[j];
    if (remap) v = uint64_t(remap[int64_t(v)]);
    __stcs(out + i, v);
  }
}

// ---- join -------------------------------------------------------------------

constexpr uint64_t JN_EMPTY = 0x8000000000000000ull;  // keys equal to it use slot `cap`

// Canonical 64-bit key; false when the key can never match (NaN).
__device__ __forceinline__ bool jn_key(const void* col, int64_t i, int kind, uint64_t& k) {
  if (kind == 0) {
    k = uint64_t(static_cast<const int64_t*>(col)[i]);
    return true;
  }
  double v = static_cast<const double*>(col)[i];
  if (v != v) return false;
  if (v == 0.0) v = 0.0;  // -0.0 == 0.0 as dict keys
  k = uint64_t(__double_as_longlong(v));
  return true;
}

__device__ __forceinline__ uint64_t jn_hash(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// Insert the build keys; every build row gets the composite sort key
// (slot << 32 | row). NaN rows go to the dead slot cap+1 (never probed).
__global__ void __launch_bounds__(256) join_insert_kernel(const void* col, int64_t nb, int kind,
                                                          uint64_t* __restrict__ table,
                                                          uint64_t cap_mask, int sbits,
                                                          gt::SortPlan plan,
                                                          unsigned long long* __restrict__ hist,
                                                          uint64_t* __restrict__ comp) {
  __shared__ uint32_t sh[gt::RS_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t cap = cap_mask + 1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb; i += stride) {
    uint64_t k;
    uint64_t s;
    if (!jn_key(col, i, kind, k)) {
      s = cap + 1;
    } else if (k == JN_EMPTY) {
      s = cap;
    } else {
      uint64_t h = jn_hash(k) & cap_mask;
      while (true) {
        const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + h),
                                        (unsigned long long)JN_EMPTY, (unsigned long long)k);
        if (prev == JN_EMPTY || prev == k) break;
        h = (h + 1) & cap_mask;
      }
      s = h;
    }
    const uint64_t key = (s << 32) | uint64_t(i);
    comp[i] = key;
    plan_hist_add(sh, plan, key);
  }
  __syncthreads();
  plan_hist_flush(sh, plan, hist);
}

// First position (head of the run) and length (tail of the run) of every
// slot's run in the sorted composite keys; two launches so the tail reads a
// start the head has already written.
__global__ void __launch_bounds__(256) join_runs_kernel(const uint64_t* __restrict__ sorted,
                                                        int64_t nb, int64_t* __restrict__ start) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nb) return;
  const uint64_t s = sorted[p] >> 32;
  if (p == 0 || (sorted[p - 1] >> 32) != s) start[s] = p;
}

__global__ void __launch_bounds__(256) join_len_kernel(const uint64_t* __restrict__ sorted,
                                                       int64_t nb, const int64_t* __restrict__ start,
                                                       int64_t* __restrict__ cnt) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nb) return;
  const uint64_t s = sorted[p] >> 32;
  if (p == nb - 1 || (sorted[p + 1] >> 32) != s) cnt[s] = p + 1 - start[s];
}

// Matches of every probe row: count (into counts[j], scanned afterwards) and
// the start of its slot's run.
__global__ void __launch_bounds__(256) join_probe_kernel(const void* col, int64_t np, int kind,
                                                         const uint64_t* __restrict__ table,
                                                         uint64_t cap_mask,
                                                         const int64_t* __restrict__ start,
                                                         const int64_t* __restrict__ cnt,
                                                         int64_t* __restrict__ counts,
                                                         int64_t* __restrict__ pstart) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < np; j += stride) {
    uint64_t k;
    int64_t c = 0, st = 0;
    if (jn_key(col, j, kind, k)) {
      int64_t s = -1;
      if (k == JN_EMPTY) {
        s = int64_t(cap_mask + 1);
      } else {
        uint64_t h = jn_hash(k) & cap_mask;
        while (true) {
          const uint64_t t = table[h];
          if (t == k) { s = int64_t(h); break; }
          if (t == JN_EMPTY) break;
          h = (h + 1) & cap_mask;
        }
      }
      if (s >= 0) {
        c = cnt[s];
        st = start[s];
      }
    }
    counts[j] = c;
    pstart[j] = st;
  }
}

// Pairs in the reference's order: probe row ascending, then build row
// ascending. Thread per probe row; rows with more than 32 matches are written
// by the whole warp.
__global__ void __launch_bounds__(256) join_expand_kernel(const int64_t* __restrict__ offs,
                                                          const int64_t* __restrict__ pstart,
                                                          int64_t np,
                                                          const uint64_t* __restrict__ sorted,
                                                          int build_left,
                                                          int64_t* __restrict__ li,
                                                          int64_t* __restrict__ ri) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j0 = int64_t(blockIdx.x) * blockDim.x; j0 < np; j0 += stride) {
    const int64_t j = j0 + threadIdx.x;
    int64_t o = 0, c = 0, st = 0;
    if (j < np) {
      o = offs[j];
      c = offs[j + 1] - o;
      st = pstart[j];
    }
    const bool big = c > 32;
    if (!big) {
      for (int64_t t = 0; t < c; ++t) {
        const int64_t b = int64_t(sorted[st + t] & 0xffffffffull);
        li[o + t] = build_left ? b : j;
        ri[o + t] = build_left ? j : b;
      }
    }
    uint32_t bigs = __ballot_sync(0xffffffffu, big);
    while (bigs) {
      const int src = __ffs(bigs) - 1;
      bigs &= bigs - 1;
      const int64_t jj = __shfl_sync(0xffffffffu, j, src);
      const int64_t oo = __shfl_sync(0xffffffffu, o, src);
      const int64_t cc = __shfl_sync(0xffffffffu, c, src);
      const int64_t ss = __shfl_sync(0xffffffffu, st, src);
      for (int64_t t = lane; t < cc; t += 32) {
        const int64_t b = int64_t(sorted[ss + t] & 0xffffffffull);
        li[oo + t] = build_left ? b : jj;
        ri[oo + t] = build_left ? jj : b;
      }
    }
  }
}

__global__ void fill_u64_kernel(uint64_t* __restrict__ p, int64_t n, uint64_t v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

}  // namespace gtd

struct gt_join {
  int64_t n_pairs = 0;
  int64_t* li = nullptr;
  int64_t* ri = nullptr;
};

namespace gt {

static int grid_rows(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div64(n, 256),
                                                                   8LL * ctx().sm_count)));
}

static int64_t select_rows(const void* col, int64_t n, int kind, int op, int64_t iv, double fv,
                           const uint8_t* lut, int64_t lut_n, int64_t* out_idx) {
  if (n == 0) return 0;
  const int64_t tiles = ceil_div64(n, gtd::SEL_TILE);
  int64_t* offs = ws_n<int64_t>(WS_TMP0, size_t(tiles) + 2);
  int64_t* total = ws_n<int64_t>(WS_SMALL, 16) + 9;
  gtd::SelPred p{kind, op, iv, fv, lut, lut_n};
  Phase ph("rel.select", 16.0 * n);
  GT_LAUNCH(gtd::select_count_kernel, static_cast<int>(tiles), gtd::SEL_THREADS, 0, col, n, p,
            offs);
  exclusive_scan_i64(offs, tiles, total);
  GT_LAUNCH(gtd::select_write_kernel, static_cast<int>(tiles), gtd::SEL_THREADS, 0, col, n, p,
            offs, out_idx);
  int64_t m = 0;
  d2h(&m, total, 8);
  sync();
  return m;
}

static gt_join* join_build(const void* left, int64_t nl, const void* right, int64_t nr,
                           int kind) {
  gt_join* j = new gt_join();
  const bool build_left = nl <= nr;  // tables.py:411
  const void* bcol = build_left ? left : right;
  const void* pcol = build_left ? right : left;
  const int64_t nb = build_left ? nl : nr, np = build_left ? nr : nl;
  if (nb == 0 || np == 0) return j;
  if (nb >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "join: build side must have < 2^31 rows");
  uint64_t cap = 1024;
  while (cap < uint64_t(2 * nb)) cap <<= 1;
  const int sbits = bits_for(int64_t(cap + 2));
  uint64_t* table = ws_n<uint64_t>(WS_TMP1, size_t(cap));
  uint64_t* ka = ws_n<uint64_t>(WS_KEYS_A, size_t(nb));
  uint64_t* kb = ws_n<uint64_t>(WS_KEYS_B, size_t(nb));
  int64_t* start = ws_n<int64_t>(WS_TMP2, size_t(cap + 2) * 2);
  int64_t* cnt = start + (cap + 2);
  int64_t* counts = ws_n<int64_t>(WS_TMP3, size_t(np) + 2);
  int64_t* pstart = ws_n<int64_t>(WS_TMP4, size_t(np) + 1);
  int64_t* total = ws_n<int64_t>(WS_SMALL, 16) + 10;
  SortPlan plan = make_plan(32, 32 + sbits);  // stable over the slot bits: row order kept
  SortHist h = sort_hist_begin(0);
  {
    Phase ph("rel.join_build", 16.0 * nb + 8.0 * cap);
    GT_LAUNCH(gtd::fill_u64_kernel, grid_rows(int64_t(cap)), 256, 0, table, int64_t(cap),
              gtd::JN_EMPTY);
    GT_CUDA(cudaMemsetAsync(cnt, 0, size_t(cap + 2) * 8, ctx().stream));
    GT_LAUNCH(gtd::join_insert_kernel, grid_rows(nb), 256, 0, bcol, nb, kind, table, cap - 1,
              sbits, plan, h.hist, ka);
  }
  uint64_t* sorted = radix_sort(ka, kb, nb, plan, h, "rel.join_sort");
  {
    Phase ph("rel.join_build", 24.0 * nb);
    GT_LAUNCH(gtd::join_runs_kernel, ceil_div(nb, 256), 256, 0, sorted, nb, start);
    GT_LAUNCH(gtd::join_len_kernel, ceil_div(nb, 256), 256, 0, sorted, nb, start, cnt);
  }
  {
    Phase ph("rel.join_probe", 8.0 * np + 24.0 * np);
    GT_LAUNCH(gtd::join_probe_kernel, grid_rows(np), 256, 0, pcol, np, kind, table, cap - 1,
              start, cnt, counts, pstart);
    exclusive_scan_i64(counts, np, total);
  }
  int64_t m = 0;
  d2h(&m, total, 8);
  sync();
  j->n_pairs = m;
  if (m > 0) {
    try {
      j->li = dalloc_n<int64_t>(size_t(m));
      j->ri = dalloc_n<int64_t>(size_t(m));
    } catch (...) {
      if (j->li) dfree(j->li);
      delete j;
      throw;
    }
    Phase ph("rel.join_expand", 16.0 * np + 24.0 * m);
    GT_LAUNCH(gtd::join_expand_kernel, grid_rows(np), 256, 0, counts, pstart, np, sorted,
              build_left ? 1 : 0, j->li, j->ri);
  }
  sync();
  return j;
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_select_rows(const void* d_col, int64_t n, int kind, int op, int64_t ival, double fval,
                   const uint8_t* d_lut, int64_t lut_n, int64_t* d_out_idx, int64_t* n_out) {
  GT_API_BEGIN
  require_init();
  if (n < 0 || !n_out) fail(GT_EINVAL, "bad arguments");
  if (kind < 0 || kind > 2) fail(GT_EINVAL, "select: kind must be 0 (int64), 1 (float64) or 2 (lut)");
  if (op < GT_CMP_EQ || op > GT_CMP_GE) fail(GT_EINVAL, "select: unknown comparison operator");
  if (n > 0 && (!d_col || !d_out_idx)) fail(GT_EINVAL, "select: null column or output");
  if (kind == 2 && lut_n > 0 && !d_lut) fail(GT_EINVAL, "select: null lookup table");
  *n_out = select_rows(d_col, n, kind, op, ival, fval, d_lut, lut_n, d_out_idx);
  GT_API_END
}

int gt_gather_u64(const uint64_t* d_src, const int64_t* d_idx, int64_t n, const int64_t* d_remap,
                  uint64_t* d_out) {
  GT_API_BEGIN
  require_init();
  if (n < 0) fail(GT_EINVAL, "gather: n must be >= 0");
  if (n > 0) {
    if (!d_src || !d_out) fail(GT_EINVAL, "gather: null column or output");
    Phase ph("rel.gather", 16.0 * n + (d_idx ? 8.0 * n : 0.0));
    GT_LAUNCH(gtd::gather_u64_kernel, grid_rows(n), 256, 0, d_src, d_idx, n, d_remap, d_out);
  }
  sync();
  GT_API_END
}

int gt_join_build(const void* d_left, int64_t nl, const void* d_right, int64_t nr, int kind,
                  gt_join** out, int64_t* n_pairs) {
  GT_API_BEGIN
  require_init();
  if (!out || !n_pairs || nl < 0 || nr < 0) fail(GT_EINVAL, "bad arguments");
  if (kind < 0 || kind > 1) fail(GT_EINVAL, "join: kind must be 0 (int64) or 1 (float64)");
  if ((nl > 0 && !d_left) || (nr > 0 && !d_right)) fail(GT_EINVAL, "join: null key column");
  gt_join* j = join_build(d_left, nl, d_right, nr, kind);
  *out = j;
  *n_pairs = j->n_pairs;
  GT_API_END
}

int gt_join_export(const gt_join* j, int64_t* d_li, int64_t* d_ri) {
  GT_API_BEGIN
  require_init();
  if (!j) fail(GT_EINVAL, "null join");
  if (j->n_pairs > 0) {
    if (!d_li || !d_ri) fail(GT_EINVAL, "join export: null output");
    GT_CUDA(cudaMemcpyAsync(d_li, j->li, size_t(j->n_pairs) * 8, cudaMemcpyDeviceToDevice,
                            ctx().stream));
    GT_CUDA(cudaMemcpyAsync(d_ri, j->ri, size_t(j->n_pairs) * 8, cudaMemcpyDeviceToDevice,
                            ctx().stream));
  }
  sync();
  GT_API_END
}

void gt_join_free(gt_join* j) {
  if (!j) return;
  try {
    if (j->li) dfree(j->li);
    if (j->ri) dfree(j->ri);
  } catch (...) {
  }
  delete j;
}

}  // extern "C"
