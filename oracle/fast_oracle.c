/*
 * fast_oracle.c — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * C restatement of the reference triangle count (graphtables
 * algorithms.py:90-119) for parity checks at sizes where the numpy
 * restatement (oracle/reference_port.py: one np.intersect1d per oriented
 * edge) would take minutes:
 *   und(i)   = (in(i) ∪ out(i)) \ {i}             graphs.py:163-167
 *   rank     = order by (|und(i)|, i)             algorithms.py:103-106
 *   higher(i)= {u ∈ und(i) : rank(u) > rank(i)}   algorithms.py:108 (id order)
 *   total    = Σ_i Σ_{j ∈ higher(i)} |higher(i) ∩ higher(j)|   algorithms.py:110-116
 * Inputs are the dense-index CSR pair (0..n-1), rows ascending.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int64_t merge_union(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t self,
                           int64_t* out) {
  int64_t i = 0, j = 0, k = 0;
  while (i < na || j < nb) {
    int64_t v;
    if (j >= nb || (i < na && a[i] < b[j])) v = a[i++];
    else if (i >= na || b[j] < a[i]) v = b[j++];
    else { v = a[i]; ++i; ++j; }
    if (v != self) {
      if (out) out[k] = v;
      ++k;
    }
  }
  return k;
}

static int64_t merge_count(const int64_t* a, int64_t na, const int64_t* b, int64_t nb) {
  int64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

int64_t oracle_triangles(int64_t n, const int64_t* out_off, const int64_t* out_adj,
                         const int64_t* in_off, const int64_t* in_adj, int threads) {
  if (n <= 0) return 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* uoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    deg[i] = merge_union(out_adj + out_off[i], out_off[i + 1] - out_off[i], in_adj + in_off[i],
                         in_off[i + 1] - in_off[i], i, NULL);
  uoff[0] = 0;
  for (int64_t i = 0; i < n; ++i) uoff[i + 1] = uoff[i] + deg[i];
  int64_t* und = (int64_t*)malloc(sizeof(int64_t) * (size_t)(uoff[n] + 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    merge_union(out_adj + out_off[i], out_off[i + 1] - out_off[i], in_adj + in_off[i],
                in_off[i + 1] - in_off[i], i, und + uoff[i]);
  /* higher(i): keep neighbours ranked above i by (degree, id), id order */
  int64_t* hoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* hcnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t p = uoff[i]; p < uoff[i + 1]; ++p) {
      int64_t u = und[p];
      if (deg[u] > deg[i] || (deg[u] == deg[i] && u > i)) ++c;
    }
    hcnt[i] = c;
  }
  hoff[0] = 0;
  for (int64_t i = 0; i < n; ++i) hoff[i + 1] = hoff[i] + hcnt[i];
  int64_t* hi = (int64_t*)malloc(sizeof(int64_t) * (size_t)(hoff[n] + 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    int64_t k = hoff[i];
    for (int64_t p = uoff[i]; p < uoff[i + 1]; ++p) {
      int64_t u = und[p];
      if (deg[u] > deg[i] || (deg[u] == deg[i] && u > i)) hi[k++] = u;
    }
  }
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t* a = hi + hoff[i];
    const int64_t na = hoff[i + 1] - hoff[i];
    for (int64_t p = 0; p < na; ++p) {
      const int64_t j = a[p];
      total += merge_count(a, na, hi + hoff[j], hoff[j + 1] - hoff[j]);
    }
  }
  free(deg); free(uoff); free(und); free(hoff); free(hcnt); free(hi);
  return total;
}
