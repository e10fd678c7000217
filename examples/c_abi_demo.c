/* Plain-C use of the drop-in boundary (include/gtb200.h): no Python, no torch.
 * Builds the graph of a small edge table with duplicates and a self-loop,
 * exports the CSR, runs PageRank and the triangle count, and checks them
 * against the reference's known answers (test_algorithms.py:28-37, 80-90):
 * K4 has 4 triangles, the self-loop is ignored, PageRank sums to 1.
 * Build: gcc -std=c99 c_abi_demo.c -I../include -L../paper_1503_07881_b200 -lgtb200 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "gtb200.h"

#define CHECK(call)                                                         \
  do {                                                                      \
    int rc_ = (call);                                                       \
    if (rc_ != GT_OK) {                                                     \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, gt_last_error()); \
      return 1;                                                             \
    }                                                                       \
  } while (0)

int main(void) {
  /* K4 on ids {10, 20, 30, 40} in both directions, plus a duplicate row and a
   * self-loop on 40 */
  const int64_t src[] = {10, 10, 10, 20, 20, 30, 20, 30, 40, 30, 40, 40, 10, 40};
  const int64_t dst[] = {20, 30, 40, 30, 40, 40, 10, 10, 10, 20, 20, 30, 20, 40};
  const int64_t rows = (int64_t)(sizeof src / sizeof src[0]);
  gt_graph* g = NULL;
  int64_t n = 0, e = 0, tri = 0;
  CHECK(gt_init(0));
  CHECK(gt_build_csr(src, dst, rows, 0, &g));
  CHECK(gt_graph_sizes(g, &n, &e));
  int64_t* ids = malloc(sizeof(int64_t) * n);
  int64_t* out_off = malloc(sizeof(int64_t) * (n + 1));
  int64_t* out_adj = malloc(sizeof(int64_t) * e);
  int64_t* in_off = malloc(sizeof(int64_t) * (n + 1));
  int64_t* in_adj = malloc(sizeof(int64_t) * e);
  double* scores = malloc(sizeof(double) * n);
  CHECK(gt_graph_export(g, ids, out_off, out_adj, in_off, in_adj));
  CHECK(gt_pagerank(g, 0.85, 10, scores, 0));
  CHECK(gt_triangles(g, &tri));
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += scores[i];
  printf("nodes %lld edges %lld triangles %lld pagerank_sum %.12f ids %lld..%lld\n",
         (long long)n, (long long)e, (long long)tri, total, (long long)ids[0],
         (long long)ids[n - 1]);
  /* 12 K4 arcs + the self-loop = 13 distinct edges (the duplicate collapses) */
  const int ok = n == 4 && e == 13 && tri == 4 && fabs(total - 1.0) < 1e-12 && ids[0] == 10 &&
                 out_off[n] == e && in_off[n] == e;
  gt_graph_free(g);
  free(ids); free(out_off); free(out_adj); free(in_off); free(in_adj); free(scores);
  puts(ok ? "c abi demo ok" : "c abi demo MISMATCH");
  return ok ? 0 : 2;
}
