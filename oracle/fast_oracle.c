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

/* ---- large-size checkers (BASELINE configs[3] / configs[4]) ------------- *
 * Same restatements over the dense-index CSR pair with int32 adjacency (the
 * layout the device exports), so that a 1.47 B-edge graph fits host RAM.  */

static int cmp_deg_id(const void* pa, const void* pb) {
  const int64_t* a = (const int64_t*)pa;
  const int64_t* b = (const int64_t*)pb;
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  return a[1] < b[1] ? -1 : (a[1] > b[1]);
}

static int cmp_i32(const void* pa, const void* pb) {
  const int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  return a < b ? -1 : (a > b);
}

static int64_t merge_union32(const int32_t* a, int64_t na, const int32_t* b, int64_t nb,
                             int32_t self, int32_t* out) {
  int64_t i = 0, j = 0, k = 0;
  while (i < na || j < nb) {
    int32_t v;
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

static int64_t merge_count32(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
  int64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

/* Triangles whose MIDDLE vertex, in the (undirected degree, id) order of
 * algorithms.py:103-106, has rank r with r % nparts == part: the slice the
 * device's gt_triangles_part counts. Orientation built here, independently of
 * the device's: higher(i) in rank space, sorted; Σ_u Σ_{v∈N+(u)} |N+(u) ∩ N+(v)|
 * restricted to the slice (algorithms.py:110-116). */
int64_t oracle_triangles_slice32(int64_t n, const int64_t* out_off, const int32_t* out_adj,
                                 const int64_t* in_off, const int32_t* in_adj, int64_t part,
                                 int64_t nparts, int threads) {
  if (n <= 0) return 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i)
    deg[i] = merge_union32(out_adj + out_off[i], out_off[i + 1] - out_off[i], in_adj + in_off[i],
                           in_off[i + 1] - in_off[i], (int32_t)i, NULL);
  int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)n);
  for (int64_t i = 0; i < n; ++i) { ord[2 * i] = deg[i]; ord[2 * i + 1] = i; }
  qsort(ord, (size_t)n, 2 * sizeof(int64_t), cmp_deg_id);
  int32_t* rank = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t r = 0; r < n; ++r) rank[ord[2 * r + 1]] = (int32_t)r;
  free(ord);
  /* N+(rank r): neighbours of higher rank, as ranks, sorted */
  int64_t* hoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* hcnt = (int64_t*)calloc((size_t)n, sizeof(int64_t));
#pragma omp parallel
  {
    int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * 1024);
    int64_t cap = 1024;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      if (deg[i] > cap) { cap = deg[i]; buf = (int32_t*)realloc(buf, sizeof(int32_t) * cap); }
      int64_t k = merge_union32(out_adj + out_off[i], out_off[i + 1] - out_off[i],
                                in_adj + in_off[i], in_off[i + 1] - in_off[i], (int32_t)i, buf);
      int64_t c = 0;
      for (int64_t p = 0; p < k; ++p) c += rank[buf[p]] > rank[i];
      hcnt[rank[i]] = c;
    }
    free(buf);
  }
  hoff[0] = 0;
  for (int64_t r = 0; r < n; ++r) hoff[r + 1] = hoff[r] + hcnt[r];
  int32_t* hi = (int32_t*)malloc(sizeof(int32_t) * (size_t)(hoff[n] + 1));
#pragma omp parallel
  {
    int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * 1024);
    int64_t cap = 1024;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      if (deg[i] > cap) { cap = deg[i]; buf = (int32_t*)realloc(buf, sizeof(int32_t) * cap); }
      int64_t k = merge_union32(out_adj + out_off[i], out_off[i + 1] - out_off[i],
                                in_adj + in_off[i], in_off[i + 1] - in_off[i], (int32_t)i, buf);
      const int32_t ri = rank[i];
      int32_t* row = hi + hoff[ri];
      int64_t c = 0;
      for (int64_t p = 0; p < k; ++p)
        if (rank[buf[p]] > ri) row[c++] = rank[buf[p]];
      qsort(row, (size_t)c, sizeof(int32_t), cmp_i32);  /* id order -> rank order */
    }
    free(buf);
  }
  free(deg); free(rank); free(hcnt);
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : total)
  for (int64_t u = 0; u < n; ++u) {
    const int32_t* a = hi + hoff[u];
    const int64_t na = hoff[u + 1] - hoff[u];
    for (int64_t p = 0; p < na; ++p) {
      const int32_t v = a[p];
      if ((int64_t)v % nparts != part) continue;
      total += merge_count32(a, na, hi + hoff[v], hoff[v + 1] - hoff[v]);
    }
  }
  free(hoff); free(hi);
  return total;
}

/* PageRank of algorithms.py:45-85 over the dense in-CSR: start 1/N,
 * contrib = score / outdeg (0 for dangling), base = (1-d)/N + d*dangling/N,
 * new[v] = base + d * Σ_{u ∈ in(v)} contrib[u] (ascending u). */
void oracle_pagerank32(int64_t n, const int64_t* in_off, const int32_t* in_adj,
                       const int64_t* out_off, double damping, int iterations, double* score,
                       int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  double* contrib = (double*)malloc(sizeof(double) * (size_t)n);
  double* next = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) score[i] = 1.0 / (double)n;
  for (int it = 0; it < iterations; ++it) {
    double dangling = 0.0;
#pragma omp parallel for reduction(+ : dangling)
    for (int64_t i = 0; i < n; ++i) {
      const int64_t od = out_off[i + 1] - out_off[i];
      contrib[i] = od ? score[i] / (double)od : 0.0;
      if (!od) dangling += score[i];
    }
    const double base = (1.0 - damping) / (double)n + damping * dangling / (double)n;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) {
      double acc = 0.0;
      for (int64_t p = in_off[v]; p < in_off[v + 1]; ++p) acc += contrib[in_adj[p]];
      next[v] = base + damping * acc;
    }
    for (int64_t i = 0; i < n; ++i) score[i] = next[i];
  }
  free(contrib); free(next);
}
