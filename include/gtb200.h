/*
 * gtb200.h — C ABI of the B200-native graphtables hot path.
 *
 * One shared library (libgtb200.so, sm_100a) replaces the three numpy
 * routines that dominate Ringo-style analytics in the reference package
 * (`/root/reference/pkg/src/graphtables`):
 *
 *   gt_build_csr   replaces convert.table_to_graph          (convert.py:128-175)
 *                  together with _dense_ids / _pack / _sorted_unique_pairs /
 *                  parallel_sort / _fill_pool                (convert.py:45-125,
 *                                                             parallel.py:52-93)
 *   gt_pagerank    replaces algorithms.pagerank             (algorithms.py:36-87)
 *   gt_triangles   replaces algorithms.triangle_count       (algorithms.py:90-119)
 *   gt_graph_export materialises the reference's in/out pools + offsets
 *                  (convert.py:154-174) in host memory, ids ascending
 *                  (graphs.py:80-82: Graph.node_ids()).
 *
 * Conventions
 *  - Every call is synchronous with respect to the caller: it enqueues work on
 *    the library stream (gt_stream()) and synchronises before returning,
 *    unless the name ends in `_async`.
 *  - Return value: GT_OK (0) or one of the GT_E* codes below; the message of
 *    the last failure on the calling thread is gt_last_error().
 *  - Pointers named `d_*` are device pointers (HBM), `h_*` host pointers.
 *    Pointers that may be either carry an explicit `*_is_device` flag.
 *  - A gt_graph owns all of its device buffers; gt_graph_free releases them.
 *    Input columns are borrowed and never written (convert.py:138-139).
 *  - Dense node index = rank of the id among the distinct ids of src ∪ dst in
 *    ascending signed order (convert.py:51-52); adjacency is stored as int32
 *    dense indices, offsets as int64 (convert.py:156-157).
 */
#ifndef GTB200_H
#define GTB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped to the reference's exception types by the host shim) */
#define GT_OK        0
#define GT_EINVAL    1   /* ValueError / TypeMismatchError                     */
#define GT_ENOMEM    2   /* MemoryError (device allocation failed)             */
#define GT_ECUDA     3   /* RuntimeError (CUDA launch / runtime failure)       */
#define GT_ENCCL     4   /* RuntimeError (collective failure)                  */
#define GT_ECAPACITY 5   /* CapacityError: N >= 2^31 distinct ids              */
#define GT_ENODEV    6   /* RuntimeError: no CUDA device / wrong architecture  */

#if defined(__GNUC__)
#define GT_API __attribute__((visibility("default")))
#else
#define GT_API
#endif

typedef struct gt_graph gt_graph;
typedef struct gt_join gt_join;

/* ---- context ------------------------------------------------------------ */

/* Select the CUDA device for this process and create the library stream.
 * Idempotent for the same device. Fails with GT_ENODEV when no sm_100 device
 * is visible. */
GT_API int gt_init(int device);

/* Library version string and the cudaStream_t (as void*) every kernel runs on. */
GT_API const char* gt_version(void);
GT_API void* gt_stream(void);

/* Message of the last failing call on this thread ("" if none). */
GT_API const char* gt_last_error(void);

/* Bind the calling thread to a lane (0 or 1; default 0). A lane has its own
 * stream and workspace, so two threads on different lanes can run calls on
 * the same graph at once (e.g. gt_pagerank next to gt_triangles); calls on
 * one lane stay serialised. */
GT_API int gt_set_lane(int lane);

/* Release cached scratch memory (radix-sort buffers, look-back state). */
GT_API int gt_release_workspace(void);

/* ---- table -> CSR  (convert.table_to_graph, convert.py:128-175) ---------- */

/* Build the directed simple graph of the edge table (src[i], dst[i]), i<rows:
 * node set = distinct ids of src ∪ dst, edge set = distinct (src,dst) pairs,
 * out-CSR sorted by (src,dst), in-CSR sorted by (dst,src). rows == 0 yields an
 * empty graph. `cols_are_device` = 1 if src/dst are device pointers, 0 for
 * host pointers (copied to HBM inside the call). */
GT_API int gt_build_csr(const int64_t* src, const int64_t* dst, int64_t rows,
                 int cols_are_device, gt_graph** out);

/* Same, with additional node ids that become nodes even without edges (a
 * host Graph's isolated nodes, graphs.py:92-96 add_node): node set = distinct
 * ids of src ∪ dst ∪ nodes. Used to move any Graph to the device. */
GT_API int gt_build_csr_nodes(const int64_t* src, const int64_t* dst, int64_t rows,
                              const int64_t* nodes, int64_t n_nodes, int cols_are_device,
                              gt_graph** out);

/* Node and distinct-edge counts (Graph.node_count / Graph.edge_count,
 * graphs.py:62-68). */
GT_API int gt_graph_sizes(const gt_graph* g, int64_t* n_nodes, int64_t* n_edges);

/* Copy the CSR to host memory in the reference's layout: ids[N] ascending,
 * out_off[N+1], out_adj[E] (original ids, per-node ascending), in_off[N+1],
 * in_adj[E]. Any pointer may be NULL to skip that array. */
GT_API int gt_graph_export(const gt_graph* g, int64_t* h_ids, int64_t* h_out_off,
                    int64_t* h_out_adj, int64_t* h_in_off, int64_t* h_in_adj);

/* Device views of the CSR (dense int32 adjacency), owned by the graph. */
GT_API int gt_graph_device_views(const gt_graph* g, const int64_t** d_ids,
                          const int64_t** d_out_off, const int32_t** d_out_adj,
                          const int64_t** d_in_off, const int32_t** d_in_adj);

/* Per-node lookups without exporting the CSR (Graph.record / has_node /
 * has_edge, graphs.py:62-88, 148-167; DeviceGraph uses them until a full
 * host copy exists). gt_graph_find: dense index of each of k node ids (-1
 * if absent). gt_graph_row: the out (in_side = 0) or in (1) neighbours of
 * dense index `index` as original ids, ascending; *h_len = row length, the
 * row is copied when h_nbrs != NULL and cap >= length. gt_graph_has_edge:
 * *h_result = 1 if the directed edge src_id -> dst_id exists. */
GT_API int gt_graph_find(const gt_graph* g, const int64_t* h_ids, int64_t k, int64_t* h_index);
GT_API int gt_graph_row(const gt_graph* g, int64_t index, int in_side, int64_t* h_nbrs,
                        int64_t cap, int64_t* h_len);
GT_API int gt_graph_has_edge(const gt_graph* g, int64_t src_id, int64_t dst_id, int* h_result);

GT_API void gt_graph_free(gt_graph* g);

/* ---- graph -> table (convert.py:178-217) ----------- */

/* The edge table of the graph, sorted by (src, dst), original ids
 * (graph_to_edge_table, convert.py:178-197): src[E], dst[E], host or device
 * buffers. */
GT_API int gt_graph_edge_table(const gt_graph* g, int64_t* src, int64_t* dst, int out_is_device);

/* The node table (node, out_deg, in_deg), ascending by id
 * (graph_to_node_table, convert.py:200-217): three int64[N] buffers. */
GT_API int gt_graph_node_table(const gt_graph* g, int64_t* node, int64_t* out_deg,
                               int64_t* in_deg, int out_is_device);

/* ---- TSV ingest (tables.load_tsv, tables.py:246-284) ---- */

/* Number of lines of a headerless TSV held in HBM (universal newlines: "\n",
 * "\r\n" and a lone "\r" end a line; a final unterminated line counts). */
GT_API int gt_tsv_count_lines(const uint8_t* d_buf, int64_t nbytes, int64_t* n_lines);

/* Parse an all-int TSV (ASCII) into ncols (<= 16) device int64 columns of
 * n_lines rows (size them with gt_tsv_count_lines). int() semantics per
 * field. On a bad line: *err_line = its 0-based index and *err_column = -1
 * (wrong field count) or the 0-based column of the leftmost bad field; the
 * first bad line is reported. *overflow = 1 when a value does not fit int64. */
GT_API int gt_tsv_parse_int64(const uint8_t* d_buf, int64_t nbytes, int ncols,
                              int64_t* const* d_cols, int64_t* n_lines, int64_t* err_line,
                              int* err_column, int* overflow);

/* ---- PageRank (algorithms.pagerank, algorithms.py:36-87) --------------- */

/* Damped power iteration, fp64, start 1/N, dangling mass redistributed
 * uniformly; scores[i] belongs to the i-th smallest node id.
 * `scores_is_device` selects a device or host output buffer of N doubles.
 * Errors: GT_EINVAL for damping ∉ (0,1), iterations < 1, empty graph
 * (algorithms.py:45-50). */
GT_API int gt_pagerank(const gt_graph* g, double damping, int iterations,
                double* scores, int scores_is_device);

/* ---- triangle count (algorithms.triangle_count, algorithms.py:90-119) -- */

/* Number of unordered mutually adjacent triples of the symmetrised graph,
 * self-loops ignored; 0 for an empty graph (algorithms.py:100-101). */
GT_API int gt_triangles(const gt_graph* g, int64_t* count);

/* Degree-ordered orientation used by gt_triangles (algorithms.py:103-108),
 * for parity tests: h_deg[N] = undirected degree |in ∪ out \ {i}| by dense
 * index (graphs.py:163-167); h_rank[N] = position of node i in (degree, id)
 * order (algorithms.py:104-106); the oriented CSR in RANK space, N+(r) = the
 * higher-ranked neighbours of the node of rank r, ascending: h_off_p[N+1],
 * h_adj_p[m] (m = undirected edge count, returned in *m; call once with
 * h_adj_p = NULL to size it). Any output pointer may be NULL; GT_EINVAL for a
 * graph without edges. */
GT_API int gt_triangle_orientation(const gt_graph* g, int32_t* h_deg, int32_t* h_rank,
                                   int64_t* h_off_p, int32_t* h_adj_p, int64_t* m);

/* ---- other CSR consumers (algorithms.py:122-248) ---- */

/* Hop distances from the node of dense index `source_index` along out-edges
 * (algorithms.sssp, algorithms.py:125-141): dist[N] int32, -1 = unreachable
 * (the reference's None); host or device buffer. GT_EINVAL for an index
 * outside [0, N). */
GT_API int gt_bfs(const gt_graph* g, int64_t source_index, int32_t* dist, int dist_is_device);

/* Weakly connected components of the symmetrised graph
 * (algorithms.connected_components, algorithms.py:232-248): labels[N] int64,
 * dense, numbered in the order of each component's smallest node id (the
 * reference labels components as it meets them scanning ids ascending);
 * *n_components (may be NULL) = number of components. */
GT_API int gt_connected_components(const gt_graph* g, int64_t* labels, int labels_is_device,
                                   int64_t* n_components);

/* Strongly connected components (algorithms.scc, algorithms.py:144-203):
 * labels[N] int64 aligned with the dense order, numbered in ascending order of
 * each component's smallest id (the reference relabels its Tarjan components
 * by first occurrence over ascending ids); *n_components (may be NULL) = their
 * number. */
GT_API int gt_scc(const gt_graph* g, int64_t* labels, int labels_is_device,
                  int64_t* n_components);

/* k-core (algorithms.k_core, algorithms.py:206-229): the induced subgraph
 * (graphs.py:169-183, every original edge between survivors) on the maximal
 * node set whose members keep >= k distinct undirected neighbours inside it,
 * as a new graph (free with gt_graph_free). GT_EINVAL for k < 1. */
GT_API int gt_kcore(const gt_graph* g, int k, gt_graph** out);

/* Batched dynamic update (graphs.py:92-144) into a new graph (*out; free with
 * gt_graph_free; g is unchanged). The batch means these reference calls in
 * this order: del_node(x) for x in d_del_nodes; del_edge(s, d) for the
 * deletion pairs; add_node(x) for x in d_add_nodes; add_edge(s, d) for the
 * addition pairs. Ids that are absent are ignored as the reference's calls
 * ignore them. All arrays are device int64. */
GT_API int gt_graph_update(const gt_graph* g, const int64_t* d_add_src, const int64_t* d_add_dst,
                           int64_t n_add, const int64_t* d_del_src, const int64_t* d_del_dst,
                           int64_t n_del, const int64_t* d_add_nodes, int64_t n_add_nodes,
                           const int64_t* d_del_nodes, int64_t n_del_nodes, gt_graph** out);

/* ---- relational operators feeding ToGraph -------- */

/* Predicate comparison codes (tables.py:32-39 _COMPARATORS). */
#define GT_CMP_EQ 0
#define GT_CMP_NE 1
#define GT_CMP_LT 2
#define GT_CMP_LE 3
#define GT_CMP_GT 4
#define GT_CMP_GE 5

/* Select (tables.py:325-344): ascending indices of the rows of the device
 * column d_col[n] whose value satisfies `value op constant`.
 *   kind 0: int64 column vs ival (INT; STRING = / != on pool codes)
 *   kind 1: float64 column vs fval (IEEE, as numpy: NaN only satisfies !=)
 *   kind 2: int64 codes, row selected iff 0 <= code < lut_n and d_lut[code]
 *           (STRING ordering comparisons, evaluated on the decoded pool)
 * d_out_idx holds n entries; *n_out (host) = number of rows selected. */
GT_API int gt_select_rows(const void* d_col, int64_t n, int kind, int op, int64_t ival,
                          double fval, const uint8_t* d_lut, int64_t lut_n, int64_t* d_out_idx,
                          int64_t* n_out);

/* Row gather of one 8-byte column (ColumnTable._take tables.py:232-240,
 * _paired_table tables.py:385-394): d_out[i] = d_src[d_idx[i]] (d_idx NULL:
 * identity), then, if d_remap is not NULL, d_out[i] = d_remap[d_out[i]]
 * (right-pool string codes into the merged pool, tables.py:393). */
GT_API int gt_gather_u64(const uint64_t* d_src, const int64_t* d_idx, int64_t n,
                         const int64_t* d_remap, uint64_t* d_out);

/* Equi-join (tables.py:397-426) of device key columns d_left[nl], d_right[nr]
 * (kind 0: int64 keys; kind 1: float64 keys with -0.0 == 0.0 and NaN never
 * matching). Builds on the smaller side (left when nl <= nr); the pairs come
 * out in the reference's order: probe row ascending, then build row ascending.
 * *out owns the (left row, right row) pair lists; *n_pairs = their length. */
GT_API int gt_join_build(const void* d_left, int64_t nl, const void* d_right, int64_t nr,
                         int kind, gt_join** out, int64_t* n_pairs);
/* Copy the pair lists into device buffers of n_pairs int64 each. */
GT_API int gt_join_export(const gt_join* j, int64_t* d_left_rows, int64_t* d_right_rows);
GT_API void gt_join_free(gt_join* j);

/* ---- synthetic inputs (bench / tests; no reference counterpart) --------- */

/* R-MAT edge table generated on the device, bit-identical to the numpy
 * generator paper_1503_07881_b200.synth.rmat_edges: row e, level l uses
 * splitmix64(key(seed) + e*scale + l); quadrant thresholds a, a+b, a+b+c on
 * 53-bit uniforms; optional keyed Feistel permutation of [0, 2^scale). */
GT_API int gt_rmat_generate(int scale, int64_t rows, double a, double b, double c,
                     uint64_t seed, int permute, int64_t* d_src, int64_t* d_dst);

/* Rows [start, start+rows) of the same R-MAT table (multi-GPU shards). */
GT_API int gt_rmat_generate_range(int scale, int64_t start, int64_t rows, double a, double b,
                                  double c, uint64_t seed, int permute, int64_t* d_src,
                                  int64_t* d_dst);

/* Uniform rows (the stand-in for BASELINE config 4, synth.random_edges
 * semantics: src, dst iid uniform in [0, n_nodes)), bit-identical to the numpy
 * generator paper_1503_07881_b200.synth.uniform_edges: row e uses
 * hi64(splitmix64(key + 2e) * n) for src and key + 2e + 1 for dst,
 * key = splitmix64(seed ^ 0xD1B54A32D192ED03). */
GT_API int gt_uniform_generate_range(int64_t n_nodes, int64_t start, int64_t rows, uint64_t seed,
                                     int64_t* d_src, int64_t* d_dst);

/* ---- multi-GPU primitives ------------------------------------------------
 * One process per GPU; paper_1503_07881_b200/distributed.py runs the
 * collectives (torch.distributed / NCCL) between these calls. They are the
 * pieces of gt_build_csr / gt_pagerank / gt_triangles restricted to one
 * rank's shard; all pointers are device pointers, every call synchronises. */

/* d_out2[0] = min, d_out2[1] = max over the ids of both columns. */
GT_API int gt_id_minmax(const int64_t* d_src, const int64_t* d_dst, int64_t rows,
                        int64_t* d_out2);
/* d_flags[x - lo] = 1 for every id x of both columns (flags zeroed first). */
GT_API int gt_id_presence(const int64_t* d_src, const int64_t* d_dst, int64_t rows, int64_t lo,
                          int64_t span, uint8_t* d_flags);
/* Presence flags (OR over ranks) -> rank map words (uint2[ceil(span/32)]:
 * 32 presence bits + popcount prefix) and the node count. */
GT_API int gt_id_rankmap(const uint8_t* d_flags, int64_t span, void* d_words, int64_t* n_nodes);
/* Sorted distinct ids (N) from the rank map words. */
GT_API int gt_id_list(const void* d_words, int64_t span, int64_t lo, int64_t* d_ids);
/* keys[i] = rank(src[i]) << kbits | rank(dst[i]) through the rank map. */
GT_API int gt_pack_keys(const int64_t* d_src, const int64_t* d_dst, int64_t rows, int64_t lo,
                        const void* d_words, int kbits, uint64_t* d_keys);
/* LSD radix sort of n keys on bits [lo_bit, hi_bit); the result is in d_keys
 * (*result_in_tmp = 0) or d_tmp (1). Stable. */
GT_API int gt_sort_keys(uint64_t* d_keys, uint64_t* d_tmp, int64_t n, int lo_bit, int hi_bit,
                        int* result_in_tmp);
/* Merge nruns sorted runs [h_run_off[r], h_run_off[r+1]) of d_keys into one
 * ascending sequence (earlier run first on ties); h_run_off is a HOST array of
 * nruns+1 offsets from 0 to n. The result is in d_keys (*result_in_tmp = 0) or
 * d_tmp (1). Replaces the re-sort of the received sample-sort buckets
 * (parallel.py:52-93) on the receive side of the sharded build. */
GT_API int gt_merge_runs(uint64_t* d_keys, uint64_t* d_tmp, int64_t n, const int64_t* h_run_off,
                         int nruns, int* result_in_tmp);
/* Drop adjacent duplicates of sorted keys (convert.py:76-80); *m = kept. */
GT_API int gt_unique_keys(const uint64_t* d_in, int64_t n, uint64_t* d_out, int64_t* m);
/* d_counts[b] = #{i : min(keys[i] >> shift, nbuckets-1) == b}, nbuckets <= 4096. */
GT_API int gt_key_bucket_counts(const uint64_t* d_keys, int64_t n, int shift, int nbuckets,
                                int64_t* d_counts);
/* h_out[j] = lower bound of h_bounds[j] in sorted keys (nb <= 4096). */
GT_API int gt_key_lower_bounds(const uint64_t* d_sorted, int64_t n, const uint64_t* h_bounds,
                               int nb, int64_t* h_out);
/* (a << kbits | b) -> (b << kbits | a). */
GT_API int gt_swap_key_halves(const uint64_t* d_in, int64_t n, int kbits, uint64_t* d_out);
/* Sorted keys of rows [row_lo, row_lo+rows) -> d_off[rows+1] (local, from 0),
 * d_adj[m] (low kbits). d_tmp: scratch of m keys (used when row_lo != 0). */
GT_API int gt_csr_from_keys(const uint64_t* d_sorted, int64_t m, int kbits, int64_t row_lo,
                            int64_t rows, uint64_t* d_tmp, int64_t* d_off, int32_t* d_adj);
/* A gt_graph from full device CSR arrays (copied), e.g. replicated shards. */
GT_API int gt_graph_from_csr(int64_t n, int64_t e, const int64_t* d_ids, const int64_t* d_out_off,
                             const int32_t* d_out_adj, const int64_t* d_in_off,
                             const int32_t* d_in_adj, gt_graph** out);
/* Multi-GPU PageRank exchange layout: d_out[i] = r*m + (d_in[i] - bounds[r])
 * for the rank r whose dst range [bounds[r], bounds[r+1]) holds d_in[i]
 * (world <= 64, h_bounds host int64[world+1]): positions in the padded
 * buffer that all_gather_into_tensor fills with one m-sized chunk per rank. */
GT_API int gt_remap_padded(const int32_t* d_in, int64_t e, const int64_t* h_bounds, int world,
                           int64_t m, int32_t* d_out);
/* d_inv[v] = 1/(off[v+1]-off[v]), 0 for an empty row. */
GT_API int gt_inv_degree(const int64_t* d_off, int64_t rows, double* d_inv);
/* PageRank start from the full 1/outdeg vector: contrib = inv/N and the
 * dangling mass (algorithms.py:67-75). */
GT_API int gt_pagerank_init(const double* d_inv, int64_t n, double* d_contrib,
                            double* d_dangling);
/* One PageRank iteration over a dst-row range of the in-CSR (local offsets,
 * global source indices into the replicated contrib vector): scores of the
 * rows (last = 1) or their next contributions (last = 0), and the local
 * dangling partial (algorithms.py:72-85). */
GT_API int gt_pagerank_step(const int64_t* d_in_off, const int32_t* d_in_adj, int64_t rows,
                            int64_t e_local, int64_t n_total, const double* d_contrib,
                            const double* d_inv_rows, const double* d_dangling_prev,
                            double damping, int last, double* d_score_rows,
                            double* d_contrib_rows, double* d_dangling_out);
/* Triangle count restricted to the middle vertices v = part (mod nparts) of
 * the rank-space orientation: the parts of all ranks sum to gt_triangles
 * (the all-reduce is the caller's). */
GT_API int gt_triangles_part(const gt_graph* g, int part, int nparts, int64_t* count);
/* Sharded orientation (distributed.triangle_count): a rank holds the
 * undirected rows of the ids [row_lo, row_lo + rows) (local offsets d_off,
 * global neighbour ids d_adj).
 * gt_tc_undirected_keys: both directions of every edge, self-loops dropped,
 * as (u << kbits | v) keys (d_keys: capacity 2 * d_off[rows]); *n_keys is the
 * count written (replaces Graph.undirected_neighbors, graphs.py:163-167, once
 * sorted, deduped and shuffled by row).
 * gt_tc_degree_rank: d_rank[id] = position of id in (degree, id) order of the
 * n degrees (algorithms.py:103-106).
 * gt_tc_orient_keys: the arcs to higher-ranked neighbours as
 * (rank(u) << kbits | rank(v)) (algorithms.py:108; capacity d_off[rows]).
 * gt_triangles_oriented_part: gt_triangles_part over a caller-built
 * rank-space orientation (d_off_p int64[n+1], d_adj_p int32[m], rows sorted). */
GT_API int gt_tc_undirected_keys(const int64_t* d_off, const int32_t* d_adj, int64_t rows,
                                 int64_t row_lo, int kbits, uint64_t* d_keys, int64_t* n_keys);
GT_API int gt_tc_degree_rank(const int64_t* d_deg, int64_t n, int32_t* d_rank);
GT_API int gt_tc_orient_keys(const int64_t* d_off, const int32_t* d_adj, int64_t rows,
                             int64_t row_lo, const int32_t* d_rank, int kbits, uint64_t* d_keys,
                             int64_t* m_keys);
GT_API int gt_triangles_oriented_part(const int64_t* d_off_p, const int32_t* d_adj_p, int64_t n,
                                      int64_t m, int part, int nparts, int64_t* count);
/* Undirected simple-edge count m of the graph (self-loops dropped, reciprocal
 * pairs merged: the size of the orientation the triangle count builds), or -1
 * when no triangle count has run on g yet (bench unit: undirected edges/s). */
GT_API int gt_graph_undirected_edges(const gt_graph* g, int64_t* m);

/* ---- instrumentation ---------------------------------------------------- */

/* Number of kernels this library has launched since load. */
GT_API int64_t gt_launch_count(void);

/* Per-phase device time accounting (CUDA events on gt_stream()).
 * gt_profile_enable(1) starts recording; gt_profile_read fills up to `cap`
 * entries of (name, total_ms, launches, algorithmic_bytes) and returns the
 * number of phases; gt_profile_reset clears the totals. */
GT_API int gt_profile_enable(int on);
GT_API int gt_profile_reset(void);
GT_API int gt_profile_read(int cap, const char** names, double* total_ms,
                    int64_t* launches, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* GTB200_H */
