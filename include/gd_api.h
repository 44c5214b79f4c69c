/*
 * gd_api.h -- C ABI of libgdgpu.so, the B200 (sm_100a) edge-centric graphlet
 * census.  This is the drop-in boundary for the reference's counting entry
 * points; every function below names the reference interface it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host pointers unless a GD_*_DEVICE flag
 *     says the buffer is device memory.
 *   - Every call is synchronous: the library's stream is synchronised before
 *     return and no caller pointer is retained.
 *   - Return value: GD_OK (0) or a negative status; gd_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - Wide sums are returned as 13 (lo, hi) uint64 pairs per graph in the
 *     reference's CensusSums.FIELDS order (census.py:377-378):
 *       tri, star, indep3, clique4, cycle4, n_tt, n_susv, n_ts, n_ss_same,
 *       n_ti, n_si, n_ii, outside
 *     value = lo + 2**64 * hi (the reference keeps Python ints; SPEC.md:211
 *     mandates 128-bit accumulators).
 *   - Per-edge rows are int64 [m][10] in canonical edge order with columns
 *     RAW_MICRO_FIELDS (census.py:95-97):
 *       tri, star_u, star_v, clique4, cycle4, uu1, vv1, ts1, ti1, si1
 */
#ifndef GD_API_H
#define GD_API_H

#include <stdint.h>

#if defined(__GNUC__)
#define GD_API __attribute__((visibility("default")))
#else
#define GD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped to the reference error hierarchy by the host layer) */
#define GD_OK             0
#define GD_EINVAL        -1  /* bad argument or invalid sanitized graph   -> ValueError          */
#define GD_EPARSE        -2  /* vertex id out of declared range / <0      -> EdgeListParseError  */
#define GD_ECAPACITY     -3  /* size beyond device-path limits            -> GraphSizeError      */
#define GD_ECUDA         -4  /* CUDA runtime / launch failure             -> DeviceError         */
#define GD_ECONSISTENCY  -5  /* on-device identity failed (seen != m ...) -> ConsistencyError    */

/* id conventions of gd_graph_create (graph.py:118-157 and 68-114) */
#define GD_IDS_REMAP      0  /* Graph.from_edges default: dense remap by ascending original id      */
#define GD_IDS_DECLARED   1  /* ParseOptions.num_vertices / _declared_n: ids must lie in [0, n)     */
#define GD_IDS_MAX_ID     2  /* ParseOptions.use_max_id: n = max id + 1                              */
#define GD_IDS_SANITIZED  3  /* Graph(n, edges): no loops/duplicates allowed (ValueError otherwise) */

/* flags */
#define GD_INPUT_DEVICE   1  /* input pairs / table pointer is device memory   */
#define GD_OUTPUT_DEVICE  2  /* per-edge table pointer is device memory        */

#define GD_NUM_SUMS       13
#define GD_NUM_MICRO      10

typedef struct gd_graph gd_graph;  /* opaque, device-resident graph */

GD_API const char* gd_last_error(void);
GD_API int gd_version(void);
GD_API int gd_device_ok(void);              /* 1 if a CUDA device is usable, else 0 */

/*
 * Graph construction on the device.  Replaces Graph.from_edges
 * (graph.py:118-157) + Graph.__init__ (graph.py:68-114): drop self-loops,
 * canonicalise (min, max), dedupe, dense remap by ascending original id (or
 * the declared-n / max-id conventions), degrees, and the degree-ordered
 * relabelled CSR the counting kernels use.  `pairs` is int64 [k][2].
 * `n` is the declared vertex count for GD_IDS_DECLARED / GD_IDS_SANITIZED
 * and ignored otherwise.
 */
GD_API int gd_graph_create(const int64_t* pairs, int64_t k, int64_t n, int ids_mode,
                    int flags, gd_graph** out);

/*
 * Batched construction for many independent small graphs in one device
 * graph (disjoint union).  Replaces the per-graph loop of feature_matrix
 * (analytics.py:111-128).  Graph g owns pairs [pair_offsets[g],
 * pair_offsets[g+1]) with ids in [0, n_per_graph[g]) (declared-n semantics).
 */
GD_API int gd_graph_create_batch(const int64_t* pairs, const int64_t* pair_offsets,
                          const int64_t* n_per_graph, int64_t num_graphs,
                          int flags, gd_graph** out);
/*
 * The same from one int64 [k_g][2] array per graph (pair_lists[g], k_g =
 * pair_offsets[g+1] - pair_offsets[g]): the library gathers them into
 * page-locked staging with all host cores, so callers holding a list of
 * per-graph arrays (feature_matrix's `graphs`) need no packing pass.
 */
GD_API int gd_graph_create_batch_list(const int64_t* const* pair_lists,
                                      const int64_t* pair_offsets, const int64_t* n_per_graph,
                                      int64_t num_graphs, int flags, gd_graph** out);

/* n, m and number of graphs of a device graph (batched: totals) */
GD_API int gd_graph_info(const gd_graph* g, int64_t* n, int64_t* m, int64_t* num_graphs);

/* per-graph n and m (arrays of length num_graphs); either may be NULL */
GD_API int gd_graph_sizes(const gd_graph* g, int64_t* n_per_graph, int64_t* m_per_graph);

/*
 * Export the reference Graph arrays (graph.py:83-114) to host memory; any
 * pointer may be NULL.  edges int64[m][2] canonical (u<v, lexicographic);
 * orig_ids int64[n]; indptr int64[n+1]; indices int64[2m] (rows strictly
 * sorted); edge_slot_ids int64[2m]; degrees int64[n].
 */
GD_API int gd_graph_export(const gd_graph* g, int64_t* edges, int64_t* orig_ids,
                    int64_t* indptr, int64_t* indices, int64_t* edge_slot_ids,
                    int64_t* degrees);

GD_API void gd_graph_free(gd_graph* g);

/*
 * Global census.  Replaces graphlet_census (census.py:478-491) ->
 * run_batches/_census_batch/_count_edge (census.py:437-466, 259-303).
 * sums: uint64 [num_graphs][13][2]; edges_seen: int64 [num_graphs] (the
 * reference's `seen == m` check, census.py:489-490, counted on device).
 */
GD_API int gd_census_global(gd_graph* g, uint64_t* sums, int64_t* edges_seen);

/*
 * Per-edge census.  Replaces micro_table (census.py:503-518) ->
 * _micro_batch/_micro_edge (census.py:469-475, 190-256).  table: int64
 * [m][10] canonical order (host, or device with GD_OUTPUT_DEVICE); sums and
 * edges_seen as for gd_census_global (may be NULL).  A page-locked host table
 * (gd_host_alloc) is filled chunk by chunk on a copy stream while the last
 * rows are still being finalized; a pageable one is staged through
 * page-locked blocks by the host cores.
 */
GD_API int gd_census_per_edge(gd_graph* g, int64_t* table, int flags, uint64_t* sums,
                       int64_t* edges_seen);

/*
 * Dual route.  Replaces frequencies_from_micro (census.py:521-544): the 13
 * wide sums of a per-edge table of one graph with n vertices.
 */
GD_API int gd_sums_from_table(const int64_t* table, int64_t m, int64_t n, int flags,
                       uint64_t* sums);

/*
 * Host closures for many graphs (census.py:388-430, Eqs. 1-4, Lemmas 2-8,
 * Eqs. 18-19) in exact 128-bit integers: sums uint64 [G][13][2] ->
 * counts int64 [G][17][2] (lo, hi of each signed 128-bit count, CLASS_IDS
 * order); status[g] = 0 or 1 + the index of the first failing identity.
 */
GD_API int gd_close_counts(const uint64_t* sums, const int64_t* n_per_graph,
                           const int64_t* m_per_graph, int64_t num_graphs, int64_t* counts,
                           int* status);

/*
 * One-shot convenience entries with the signatures a ctypes/cffi binding of
 * graphlet_census / micro_table binds (sanitized canonical edges of a
 * reference Graph: g.edges, g.m, g.n).
 */
GD_API int gd_census_global_edges(const int64_t* edges, int64_t m, int64_t n, int flags,
                           uint64_t* sums, int64_t* edges_seen);
GD_API int gd_census_per_edge_edges(const int64_t* edges, int64_t m, int64_t n, int flags,
                             int64_t* table, uint64_t* sums, int64_t* edges_seen);

/*
 * Multi-GPU (one process per GPU; replaces the worker pool of run_batches,
 * parallel.py:85-149).  gd_comm_unique_id on rank 0 (128 bytes, broadcast by
 * the caller), gd_comm_init on every rank (NCCL is loaded at this point).
 * gd_census_sharded deals the frames of the counting passes round-robin to
 * the ranks; each rank owns the contiguous canonical edge range
 * gd_shard_rows(m, rank, world).  Between the passes the
 * per-edge triangle counters are all-reduced and the per-edge partial sums
 * reduce-scattered onto their owners; each rank finalizes -- and writes to
 * `table` -- only its own rows (e1 - e0 rows), and every rank returns the
 * global 13 sums (128-bit, all-gathered and added exactly; the reference's
 * fixed-order merge of worker accumulators, parallel.py:138-143).
 * comm == NULL with virtual_ranks = K emulates K shards on this GPU (their
 * ranges together: the full table).
 */
typedef struct gd_comm gd_comm;
GD_API int gd_comm_unique_id(unsigned char* id_out);
GD_API int gd_comm_init(const unsigned char* id, int rank, int world, gd_comm** out);
GD_API void gd_comm_free(gd_comm* comm);
GD_API int gd_census_sharded(gd_graph* g, gd_comm* comm, int virtual_ranks, int per_edge,
                             int64_t* table, int flags, uint64_t* sums, int64_t* edges_seen);
GD_API int gd_shard_rows(int64_t m, int rank, int world, int64_t* e0, int64_t* e1);

/*
 * Device timings (CUDA events on the library stream) of the phases of the
 * last census call on `g`, in milliseconds.  names receives a static,
 * '\n'-separated list of phase names.  Returns the number of phases written.
 */
GD_API int gd_graph_timings(const gd_graph* g, float* ms, int capacity, const char** names);

/* work statistics of the last census call (wedges, triangles, ...) */
GD_API int gd_graph_stats(const gd_graph* g, int64_t* values, int capacity, const char** names);

/* Select the CUDA device of the calling thread (one process per GPU). */
GD_API int gd_set_device(int device);

/* Device memory for GD_OUTPUT_DEVICE tables (device-resident runs). */
GD_API void* gd_device_alloc(int64_t bytes);
GD_API void  gd_device_free(void* p);

/* Pinned host memory helpers (for end-to-end runs without torch). */
GD_API void* gd_host_alloc(int64_t bytes);
GD_API void  gd_host_free(void* p);

/*
 * Edge-list text on the device.  Replaces load_edge_list (graph.py:223-285)
 * for ASCII text: the bytes are copied to the GPU once, lines are tokenised
 * there and the integer pairs stay in device memory, ready for
 * gd_graph_create(..., GD_INPUT_DEVICE).  `prefixes` are the comment
 * prefixes (ParseOptions.comment_prefixes, graph.py:44).  Flags:
 * GD_PARSE_CR_NEWLINE marks text read from a file in universal-newline mode
 * (a lone '\r' is a line break there); GD_PARSE_MM_SHIFT shifts the ids of a
 * MatrixMarket file with a size header to 0-based (graph.py:277-283).
 * gd_parsed_info fills int64 info[12]:
 *   [0] pairs  [1] MatrixMarket rows or -1
 *   [2] error kind: 0 none, 1 "expected at least 2 integer tokens",
 *       2 "non-integer vertex id", 3 "malformed MatrixMarket size header",
 *       4 "no data lines" (EdgeListParseError, graph.py:257-271)
 *   [3] error line (1-based)  [4] byte offset  [5] byte length of that line
 *   [6] nonzero: input outside the ASCII rules (non-ASCII bytes, a lone '\r'
 *       under GD_PARSE_CR_NEWLINE, ids beyond int64) -- nothing parsed; the
 *       caller must decide such input with CPython's rules
 *   [7] min id  [8] max id  [9] shift applied  [10] lines
 */
#define GD_PARSE_CR_NEWLINE 1
#define GD_PARSE_MM_SHIFT   2
typedef struct gd_parsed gd_parsed;
GD_API int gd_parse_edge_list(const char* text, int64_t len, const char* const* prefixes,
                              int nprefixes, int flags, gd_parsed** out);
GD_API int gd_parsed_info(const gd_parsed* p, int64_t* info);
/* Device pointer of the parsed int64 [pairs][2] array (valid until freed). */
GD_API const int64_t* gd_parsed_pairs(const gd_parsed* p);
GD_API void gd_parsed_free(gd_parsed* p);

/*
 * Derived per-edge outputs on the device.  `table` is
 * the [m][10] micro table of `g` (device memory with GD_INPUT_DEVICE),
 * `orig_ids` the host int64 [n] original vertex ids.
 * gd_micro_roles replaces _derive_micro over all edges (census.py:574-596):
 * roles = int64 [m][15] in the order tt1 tt0 susv1 susv0 ts1 ts0 ss1 ss0
 * ti1 ti0 si1 si0 ii1 ii0 indep3.
 * gd_micro_csv replaces micro_csv (census.py:603-623): the CSV text
 * (header + one row per edge, original ids) in a device buffer, read with
 * gd_text_size / gd_text_copy.
 * A negative derived count returns GD_ECONSISTENCY and sets *bad to
 * (edge << 4 | k), k indexing tt0 susv0 ts0 ss0 ti0 ti1 si0 si1 ii0 ii1 (the
 * reference's check order); *bad = -1 otherwise.
 */
typedef struct gd_text gd_text;
GD_API int gd_micro_roles(const gd_graph* g, const int64_t* table, int flags,
                          const int64_t* orig_ids, int64_t* roles, int64_t* bad);
GD_API int gd_micro_csv(const gd_graph* g, const int64_t* table, int flags,
                        const int64_t* orig_ids, gd_text** out, int64_t* bad);
GD_API int64_t gd_text_size(const gd_text* t);
GD_API int gd_text_copy(const gd_text* t, int64_t offset, int64_t len, char* host);
GD_API void gd_text_free(gd_text* t);

/*
 * Edge analytics over the per-edge table (analytics.py:
 * 142-194).  Patterns: GD_PATTERN_* (weights: triangle = t, clique4 = cl,
 * cycle4 = cy, star4 = C(su,2) + C(sv,2) - uu - vv).  `table` is the [m][10]
 * micro table (device memory with GD_INPUT_DEVICE); outputs are host arrays.
 * gd_rank_edges writes the top `k` edges (k < 0: all) by descending weight,
 * canonical index breaking ties: index, dense endpoints u < v, weight.
 */
#define GD_PATTERN_TRIANGLE 0
#define GD_PATTERN_CLIQUE4  1
#define GD_PATTERN_CYCLE4   2
#define GD_PATTERN_STAR4    3
GD_API int gd_edge_weights(const gd_graph* g, const int64_t* table, int flags, int pattern,
                           int64_t* weights);
GD_API int gd_rank_edges(const gd_graph* g, const int64_t* table, int flags, int pattern,
                         int64_t k, int64_t* index, int64_t* u, int64_t* v, int64_t* weight);
GD_API int gd_vertex_triangles(const gd_graph* g, const int64_t* table, int flags,
                               int64_t* per_vertex);

/*
 * Incremental induced-subgraph selections (replaces
 * SelectionState._refresh_region / _local_tuple / _close, selection.py:
 * 120-205).  Actions: GD_SEL_ADD_VERTEX / GD_SEL_REMOVE_VERTEX (a = dense
 * vertex id), GD_SEL_READMIT_EDGE / GD_SEL_EXCLUDE_EDGE (a = canonical edge
 * id).  The caller applies the reference's validation and no-op rules first.
 * `moments` receives 11 (lo, hi) two's complement 128-bit running sums over
 * the selected edges: m_sel, S t, S s, S cl, S cy, S C(t,2), S su*sv, S t*s,
 * S C(su,2)+C(sv,2), S t^2, S s^2 (s = su + sv), from which the closure of
 * the selection's census is evaluated (CensusSums with n_sel, m_sel).
 */
#define GD_SEL_ADD_VERTEX    0
#define GD_SEL_REMOVE_VERTEX 1
#define GD_SEL_READMIT_EDGE  2
#define GD_SEL_EXCLUDE_EDGE  3
typedef struct gd_selection gd_selection;
GD_API int gd_selection_create(const gd_graph* g, gd_selection** out);
GD_API int gd_selection_apply(gd_selection* s, int action, int64_t a, uint64_t* moments);
GD_API void gd_selection_free(gd_selection* s);

/* Write a buffer larger than L2 on the library stream (timing hygiene). */
GD_API int gd_flush_l2(void);

/* Release the calling thread's cached census workspace (slot accumulators,
 * hit buffer, counter slabs).  It is kept between calls so that censuses of
 * fresh graphs of similar size do not re-allocate; no reference counterpart
 * (the reference allocates per call, census.py:190-303). */
GD_API int gd_trim_workspace(void);

/* (new) Diagnostics of the stream-ordered device pool the library allocates
 * from: out[0] reserved bytes, out[1] reserved high-water mark, out[2] used
 * bytes, out[3] used high-water mark. */
GD_API int gd_pool_stats(uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* GD_API_H */
