// tsv.cu — LoadTableTSV for all-int schemas on the device.
//
// Reference (tables.py:246-284): headerless UTF-8 TSV read in text mode
// (universal newlines: "\n", "\r\n" and a lone "\r" end a line), one row per
// line, `line.rstrip("\n").split("\t")` must give exactly one field per
// column, each field converted with Python's int() (surrounding whitespace,
// optional sign, single underscores between digits), errors reported for the
// first offending line (field count first, then the leftmost bad column).
// Device pipeline (the file bytes already in HBM):
//   tsv_count_kernel / tsv_ends_kernel   line ends by decoupled look-back
//                                        compaction over 4096-byte tiles
//   tsv_parse_kernel                     thread per line: split on tabs,
//                                        parse, write the int64 columns;
//                                        the first error by atomicMin on
//                                        (line, column) keys
// Bytes >= 0x80 (non-ASCII digits / spaces that int() accepts) are left to
// the host parser by the Python caller.
#include "common.cuh"
#include "radix_sort.cuh"

#include <algorithm>

namespace gtd {

constexpr int TSV_TILE = 4096;
constexpr int TSV_MAX_COLS = 16;

struct TsvCols {
  int64_t* col[TSV_MAX_COLS];
};

__device__ __forceinline__ bool tsv_is_end(const uint8_t* __restrict__ b, int64_t n, int64_t i) {
  const uint8_t c = b[i];
  return c == '\n' || (c == '\r' && (i + 1 >= n || b[i + 1] != '\n'));
}

// Pass 1 (count) and pass 2 (write the end positions) of the compaction.
template <bool WRITE>
__global__ void __launch_bounds__(256) tsv_ends_kernel(const uint8_t* __restrict__ b, int64_t n,
                                                       int64_t* __restrict__ ends,
                                                       uint64_t* __restrict__ status,
                                                       uint32_t* __restrict__ counter,
                                                       uint32_t epoch,
                                                       int64_t* __restrict__ total_out) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[8];
  __shared__ uint64_t s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t base = int64_t(s_tile) * TSV_TILE + int64_t(threadIdx.x) * 16;
  uint32_t bits = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (base + q < n && tsv_is_end(b, n, base + q)) bits |= 1u << q;
  uint32_t tot;
  const uint32_t pre = block_excl_scan_256<uint32_t>(__popc(bits), s_scan, tot);
  if (threadIdx.x == 0) {
    s_excl = lookback_single(status, int(s_tile), epoch, tot);
    if (int64_t(s_tile) == (n - 1) / TSV_TILE) *total_out = int64_t(s_excl) + tot;
  }
  __syncthreads();
  if (WRITE) {
    int64_t pos = int64_t(s_excl) + pre;
    while (bits) {
      const int q = __ffs(bits) - 1;
      bits &= bits - 1;
      ends[pos++] = base + q;
    }
  }
}

__device__ __forceinline__ bool tsv_space(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' ||
         (c >= 0x1c && c <= 0x1f);  // str.strip()/int() whitespace in ASCII
}

// int(field) for an ASCII field [p, q): 0 ok, 1 not an integer, 2 out of
// int64 range (Python would parse it; numpy's int64 conversion then fails).
__device__ __forceinline__ int tsv_int(const uint8_t* __restrict__ b, int64_t p, int64_t q,
                                       int64_t& out) {
  while (p < q && tsv_space(b[p])) ++p;
  while (q > p && tsv_space(b[q - 1])) --q;
  if (p >= q) return 1;
  bool neg = false;
  if (b[p] == '+' || b[p] == '-') {
    neg = b[p] == '-';
    ++p;
  }
  if (p >= q) return 1;
  unsigned long long mag = 0;
  bool big = false, prev_digit = false;
  for (int64_t i = p; i < q; ++i) {
    const uint8_t c = b[i];
    if (c == '_') {  // single underscores between digits only
      if (!prev_digit || i + 1 >= q || b[i + 1] < '0' || b[i + 1] > '9') return 1;
      prev_digit = false;
      continue;
    }
    if (c < '0' || c > '9') return 1;
    prev_digit = true;
    if (mag > (~0ull - 9) / 10) big = true;
    else mag = mag * 10 + (c - '0');
  }
  const unsigned long long lim = neg ? (1ull << 63) : (1ull << 63) - 1;
  if (big || mag > lim) return 2;
  out = neg ? int64_t(0 - mag) : int64_t(mag);
  return 0;
}

// err: min over (line << 8 | code), code 0 = field count, 1 + j = column j.
__global__ void __launch_bounds__(256) tsv_parse_kernel(const uint8_t* __restrict__ b, int64_t n,
                                                        const int64_t* __restrict__ ends,
                                                        int64_t n_lines, int ncols, TsvCols cols,
                                                        unsigned long long* __restrict__ err,
                                                        int* __restrict__ overflow) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t l = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; l < n_lines; l += stride) {
    const int64_t s = l == 0 ? 0 : ends[l - 1] + 1;
    int64_t e = ends[l];  // exclusive: the line end byte ("\n" or lone "\r")
    if (e > s && b[e] == '\n' && b[e - 1] == '\r') --e;  // "\r\n" -> one newline
    // field count first (line.rstrip("\n").split("\t"))
    int nf = 1;
    for (int64_t i = s; i < e; ++i) nf += b[i] == '\t';
    if (nf != ncols) {
      atomicMin(err, (unsigned long long)(l) << 8);
      continue;
    }
    int64_t p = s;
    for (int j = 0; j < ncols; ++j) {
      int64_t q = p;
      while (q < e && b[q] != '\t') ++q;
      int64_t v = 0;
      const int rc = tsv_int(b, p, q, v);
      if (rc == 1) {
        atomicMin(err, ((unsigned long long)(l) << 8) | unsigned(1 + j));
        break;
      }
      if (rc == 2) *overflow = 1;
      cols.col[j][l] = v;
      p = q + 1;
    }
  }
}

}  // namespace gtd

namespace gt {

// Line ends of the buffer; returns the number of lines (a final line without
// a terminator counts when non-empty).
static int64_t tsv_index(const uint8_t* buf, int64_t nbytes, int64_t** ends_out) {
  if (nbytes <= 0) {
    *ends_out = nullptr;
    return 0;
  }
  const int64_t tiles = ceil_div64(nbytes, gtd::TSV_TILE);
  if (tiles >= (int64_t(1) << 31)) fail(GT_ECAPACITY, "TSV buffer too large");
  uint64_t* status = ws_n<uint64_t>(WS_LOOKBACK, size_t(tiles) + 1);
  uint32_t* counters = ws_n<uint32_t>(WS_COUNTERS, 64);
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  GT_CUDA(cudaMemsetAsync(counters + 24, 0, 8, ctx().stream));
  GT_LAUNCH(gtd::tsv_ends_kernel<false>, static_cast<int>(tiles), 256, 0, buf, nbytes,
            (int64_t*)nullptr, status, counters + 24, next_epoch(), small + 1);
  int64_t n_ends = 0;
  d2h(&n_ends, small + 1, 8);
  sync();
  uint8_t last = 0;
  d2h(&last, buf + nbytes - 1, 1);
  sync();
  const bool tail = !(last == '\n' || last == '\r');
  int64_t* ends = ws_n<int64_t>(WS_TMP0, size_t(n_ends) + 1);
  GT_LAUNCH(gtd::tsv_ends_kernel<true>, static_cast<int>(tiles), 256, 0, buf, nbytes, ends,
            status, counters + 25, next_epoch(), small + 1);
  if (tail) h2d(ends + n_ends, &nbytes, 8);  // virtual end after the last byte
  *ends_out = ends;
  return n_ends + (tail ? 1 : 0);
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_tsv_count_lines(const uint8_t* d_buf, int64_t nbytes, int64_t* n_lines) {
  GT_API_BEGIN
  require_init();
  if (!n_lines || nbytes < 0 || (nbytes > 0 && !d_buf)) fail(GT_EINVAL, "bad arguments");
  int64_t* ends = nullptr;
  Phase ph("tsv.index", 2.0 * nbytes);
  *n_lines = tsv_index(d_buf, nbytes, &ends);
  sync();
  GT_API_END
}

int gt_tsv_parse_int64(const uint8_t* d_buf, int64_t nbytes, int ncols, int64_t* const* d_cols,
                       int64_t* n_lines, int64_t* err_line, int* err_column, int* overflow) {
  GT_API_BEGIN
  require_init();
  if (!n_lines || !err_line || !err_column || !overflow || ncols < 1 ||
      ncols > gtd::TSV_MAX_COLS || !d_cols)
    fail(GT_EINVAL, "bad arguments (1 <= ncols <= 16)");
  *err_line = -1;
  *err_column = -1;
  *overflow = 0;
  int64_t* ends = nullptr;
  int64_t lines = 0;
  {
    Phase ph("tsv.index", 2.0 * nbytes);
    lines = tsv_index(d_buf, nbytes, &ends);
  }
  *n_lines = lines;
  if (lines == 0) {
    sync();
    return GT_OK;
  }
  gtd::TsvCols cols;
  for (int j = 0; j < ncols; ++j) cols.col[j] = d_cols[j];
  int64_t* small = ws_n<int64_t>(WS_SMALL, 16);
  const unsigned long long none = ~0ull;
  h2d(small + 6, &none, 8);
  GT_CUDA(cudaMemsetAsync(small + 7, 0, 8, ctx().stream));
  {
    Phase ph("tsv.parse", double(nbytes) + 8.0 * lines * (ncols + 1));
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div64(lines, 256), 16LL * ctx().sm_count));
    GT_LAUNCH(gtd::tsv_parse_kernel, grid, 256, 0, d_buf, nbytes, ends, lines, ncols, cols,
              reinterpret_cast<unsigned long long*>(small + 6), reinterpret_cast<int*>(small + 7));
  }
  unsigned long long h[2];
  d2h(h, small + 6, sizeof h);
  sync();
  if (h[0] != ~0ull) {
    *err_line = int64_t(h[0] >> 8);
    *err_column = int(h[0] & 0xff) - 1;  // -1: field count
  }
  *overflow = int(h[1] & 0xffffffff) != 0;
  GT_API_END
}

}  // extern "C"
