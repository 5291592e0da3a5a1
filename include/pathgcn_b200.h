/* pathgcn_b200 — C ABI of the B200-native backward-aggregation path.
 *
 * Drop-in for the four operator groups of the reference's C++ API
 * (namespace pathgcn, /root/reference/proj/core/include/pathgcn/*.hpp):
 * graph load, execution-path build, group partition, backward aggregate.
 * Each entry point names the reference interface it replaces. Plain
 * pointers and sizes only; device memory is owned by the opaque handles.
 *
 * Status codes (every function returns int): 0 ok; 2 config/shape/staleness
 * (ConfigError, ShapeError, StalenessError — error.hpp:10-31); 3 io
 * (IoError, error.hpp:33-35); 4 numeric (NumericError, error.hpp:37-47);
 * 5 CUDA device/runtime failure. pg_last_error() returns the message of the
 * calling thread's last failure.
 *
 * Threading (mirrors the reference's "synchronous, internally parallel"
 * contract): build calls are synchronous; pg_backward_aggregate /
 * pg_aggregate_pull / dense ops are asynchronous on the caller's stream and
 * ACCUMULATE into the output like aggregate_pull (aggregate.hpp:50-55)
 * unless PG_AGG_OVERWRITE is set (equivalent for a zeroed output). A handle
 * is not thread-safe; distinct handles may be used concurrently. Multi-GPU:
 * one handle set and one NCCL rank per device.
 *
 * There is no CPU fallback: without a CUDA device every call returns 5.
 */
#ifndef PATHGCN_B200_H
#define PATHGCN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_OK 0
#define PG_ERR_CONFIG 2
#define PG_ERR_IO 3
#define PG_ERR_NUMERIC 4
#define PG_ERR_DEVICE 5

/* WeightMode (csr_graph.hpp:13) */
#define PG_WEIGHTS_UNIT 0
#define PG_WEIGHTS_SYMNORM 1

/* aggregation flags. CommitMode (aggregate.hpp:21): Deterministic is the
 * default; PG_AGG_FAST selects Fast, which on the device runs the same
 * atomic-free kernel (a valid Fast result, bit-equal to Deterministic) and
 * reports the reference's Fast counters. */
#define PG_AGG_FAST 1u
#define PG_AGG_OVERWRITE 2u
/* PG_AGG_GROUPED (implies Fast): the group-partitioned kernel of
 * aggregate.hpp:84-115 — one (sub-)warp per neighbour group, plain commit
 * for single-group destinations, fp32 atomics for the rest, so gs sets the
 * GPU's unit of work. Within fp32 tolerance of Deterministic, not bit-exact.
 * Whole groupings only (no row ranges / segments / host buffers). */
#define PG_AGG_GROUPED 4u

typedef struct pg_graph_s* pg_graph;         /* CsrGraph      csr_graph.hpp:19-38   */
typedef struct pg_frontiers_s* pg_frontiers; /* FrontierSets  frontier.hpp:14-18    */
typedef struct pg_path_s* pg_path;           /* ExecutionPath execution_path.hpp:16-33 */
typedef struct pg_groups_s* pg_groups;       /* GroupedCsr    grouping.hpp:14-28    */
typedef struct pg_edge_list_s* pg_edge_list; /* EdgeList      edge_list.hpp:14-18   */

int pg_last_error(char* buf, size_t cap);
/* The reference exception type of the calling thread's last failure
 * (error.hpp:10-47), so wrappers rethrow the exact subtype: PG_KIND_* below;
 * *line (nullable) = ParseError::line_number for PG_KIND_PARSE, else 0. */
#define PG_KIND_NONE 0
#define PG_KIND_CONFIG 1      /* ConfigError    -> status 2 */
#define PG_KIND_SHAPE 2       /* ShapeError     -> status 2 */
#define PG_KIND_STALENESS 3   /* StalenessError -> status 2 */
#define PG_KIND_PARSE 4       /* ParseError     -> status 2 */
#define PG_KIND_IO 5          /* IoError        -> status 3 */
#define PG_KIND_NUMERIC 6     /* NumericError   -> status 4 */
#define PG_KIND_DEVICE 7      /* (new) CUDA failure -> status 5 */
int pg_last_error_kind(uint64_t* line);
int pg_version(void);
int pg_device_count(int* count);
/* Scheduling knob (never changes results): destinations with at least this
 * many path edges run on the heavy-destination kernel (cooperative staged,
 * or the TMA bulk ring with tuning "heavy_tma"). 0 disables; UINT64_MAX
 * (default, or $PG_HEAVY_MIN_DEG) = width dependent: 4096 for rows of <= 32
 * floats, off for wider rows. */
int pg_set_heavy_min_degree(uint64_t min_degree);
/* Other SpMM scheduling knobs (never change results), by name: "vec_u"
 * (edges per gather batch: 4, 8, 16), "chunk_major" (0/1: column-chunk-major
 * item order for rows wider than 128 floats), "heavy_tma" (1: heavy narrow
 * destinations on the TMA cp.async.bulk + mbarrier ring), "heavy_narrow",
 * "heavy_wide_pipe", "wide_lpd", "src_segs" (0 = automatic L2-sized source
 * segments, K = forced), "ld_cg", "grouped_seg"; for the host-buffer
 * calls "host_segs" (source-row segments uploaded and reduced in turn, 1..8),
 * "host_chunks" (destination-row chunks of the last pass whose D2H overlaps
 * the next chunk, 1..16), "host_final_segs" (trailing source segments the
 * chunked last pass spans, 1..host_segs), "host_seg_balance" (1: segments of
 * equal edge counts, 0: equal rows), "host_last_seg_pct" (% of the edges in
 * the last, chunked segment; 0 = 1/K), "host_chunk_balance" (chunk cuts: %
 * weight of edges vs rows), "host_copy_prio" (copy/repack streams at the
 * highest priority), "host_pitch2d" (measured slower,
 * off) and "host_trace" (1: phase times on stderr). Round-2 knobs (each
 * measured; DESIGN.md §4 gives the numbers): "hub_inline" (1, default: wide-
 * row hubs as the main SpMM's destination-major front; 0: side kernel),
 * "hub_front_min", "rec_window" (0 / 1 shuffles / 2 REDUX), "row_kernel" +
 * "row_u" + "row_seg_mb" + "row_heavy" (whole-row warps), "vec_block" (256 /
 * 512 / 1024), "vec_window" (source-window lockstep CTAs), "narrow_u",
 * "grouped_src_segs" (grouped Fast over L2-sized segments), "gemm_packed"
 * (2, default: register-tiled k_gemm3; 1: k_gemm2; 0: k_gemm), "gemm3_rows",
 * "gemm_beside_wgrad", "atb_depth", "host_hub_chunk_side" + "host_hub_min",
 * "host_first_chunk_pct", "host_seq", "atb_quad", "host_small_chunks",
 * "vec8" (2, default: 256-bit row gathers for rows wider than 64 columns
 * from 2^21 edges per call; 1: every width; 0: off).
 * A negative value restores the default ($PG_<KEY> at load, else built-in).
 * Unknown key -> PG_ERR_CONFIG. */
int pg_set_tuning(const char* key, int64_t value);

/* ---------------- graph load ---------------- */

/* rmat.cpp:10-44 gen_rmat (host, same libstdc++ mt19937_64 stream):
 * writes 2*m ids to pairs, *n_pad = padded vertex count. */
int pg_gen_rmat(uint32_t n, uint64_t m, double a, double b, double c, double d, uint64_t seed,
                uint32_t* pairs, uint32_t* n_pad);
/* training_set.cpp:28-49 sample_training_set (host). *k = max(1, llround(ratio*n)). */
int pg_training_set_size(uint32_t n, double ratio, uint64_t* k);
int pg_sample_training_set(uint32_t n, double ratio, uint64_t seed, uint32_t* out);

/* edge_list.cpp:34-62 load_edge_list_file: "src dst" lines, '#' comments and
 * blank lines skipped, tokens trimmed, ids strict non-negative u32; self
 * loops dropped and counted. Malformed line -> PG_ERR_CONFIG (ParseError,
 * the message ends "(line N)"); unreadable file -> PG_ERR_IO. */
int pg_edge_list_load(const char* path, pg_edge_list* out);
int pg_edge_list_info(pg_edge_list el, uint64_t* npairs, uint64_t* self_loops_dropped);
int pg_edge_list_export(pg_edge_list el, uint32_t* pairs);  /* 2*npairs ids */
int pg_edge_list_destroy(pg_edge_list el);
/* edge_list.cpp:70-73 write_edge_list ("u v" per line) */
int pg_edge_list_write(const char* path, const uint32_t* pairs, uint64_t npairs);
/* load_edge_list_file + build_undirected_csr + assign_edge_weights
 * (no n_hint: n = 1 + max id), the graph built on `device` */
int pg_graph_load_file(int device, const char* path, int weight_mode, pg_graph* out);
/* training_set.cpp:51-73 load_training_set: one id per line (std::stoll),
 * '#' comments and blank lines skipped; ids >= n or negative ->
 * PG_ERR_CONFIG; sorted, de-duplicated; empty -> PG_ERR_CONFIG. out NULL:
 * only *k. Otherwise cap must be >= *k. */
int pg_training_set_load(const char* path, uint32_t n, uint32_t* out, uint64_t cap, uint64_t* k);
/* training_set.cpp:81-83 write_training_set (one id per line) */
int pg_training_set_write(const char* path, const uint32_t* vt, uint64_t k);

/* csr_graph.cpp:33-63 build_undirected_csr + :65-77 assign_edge_weights, on
 * device. n_hint < 0: none. pairs: 2*npairs host ids. */
int pg_graph_build(int device, int64_t n_hint, const uint32_t* pairs, uint64_t npairs,
                   int weight_mode, pg_graph* out);
/* Upload an existing host CsrGraph (offsets u64[n+1], neighbors u32[m],
 * weights f64[m]); validates the CsrGraph invariants (sorted, unique,
 * symmetric, symmetric weights) when validate != 0. */
int pg_graph_create(int device, uint32_t n, const uint64_t* offsets, const uint32_t* neighbors,
                    const double* weights, int validate, pg_graph* out);
/* csr_graph.cpp:65-77 assign_edge_weights */
int pg_graph_assign_weights(pg_graph g, int weight_mode);
/* n, m, max_degree (csr_graph.cpp:13-17), FNV fingerprint (csr_graph.cpp:19-31) */
int pg_graph_info(pg_graph g, uint32_t* n, uint64_t* m, uint32_t* max_degree, uint64_t* fingerprint);
/* copy to host (any pointer may be NULL) */
int pg_graph_export(pg_graph g, uint64_t* offsets, uint32_t* neighbors, double* weights);
int pg_graph_destroy(pg_graph g);
/* execution_path.cpp:17-22 path_fingerprint(g, V_t, L) */
int pg_path_fingerprint(pg_graph g, const uint32_t* vt, uint64_t k, uint64_t layers, uint64_t* fp);

/* ---------------- execution-path build ---------------- */

/* frontier.cpp:7-26 compute_frontiers. vt: sorted unique host ids. */
int pg_frontiers_compute(pg_graph g, const uint32_t* vt, uint64_t k, uint64_t layers, pg_frontiers* out);
int pg_frontiers_size(pg_frontiers f, uint64_t level, uint64_t* size);
int pg_frontiers_export(pg_frontiers f, uint64_t level, uint32_t* out);
int pg_frontiers_destroy(pg_frontiers f);

/* execution_path.cpp:24-88 extract_execution_path (layer l: dests N^{L-l},
 * sources N^{L-l-1}). prepare_all_paths (:90-96) = layers L-1 .. 0. */
int pg_path_extract(pg_graph g, pg_frontiers f, uint64_t layer, pg_path* out);
int pg_path_info(pg_path p, uint64_t* layer, uint32_t* dests, uint32_t* srcs, uint64_t* edges,
                 uint32_t* parent_rows, uint32_t* max_degree);
/* copy the ExecutionPath arrays to host (any pointer may be NULL) */
int pg_path_export(pg_path p, uint32_t* dest_local_to_global, uint32_t* src_local_to_global,
                   uint32_t* src_pos_in_parent, uint64_t* offsets, uint32_t* neighbors,
                   double* weights);
/* ExecutionPath::fingerprint stamp (train.hpp:108-112) */
int pg_path_set_fingerprint(pg_path p, uint64_t fp);
int pg_path_get_fingerprint(pg_path p, uint64_t* fp);
int pg_path_destroy(pg_path p);

/* ---------------- group partition ---------------- */

/* gs_model.cpp:68-74 regression_gs over train.hpp:16-24 path_stats
 * (|D|, directed pull-edge count, E/|D|); beta NULL = default_gs_model
 * (gs_model.cpp:64-66). */
int pg_gs_regression(pg_path p, const double* beta, uint32_t* gs);
/* gs_model.cpp:68-74 on explicit GraphStats */
int pg_gs_regression_stats(uint32_t n_vertices, uint64_t n_edges, double avg_degree,
                           const double* beta, uint32_t* gs);
/* group_cost.cpp:30-34 default_gs_candidates; *count <= 33 */
int pg_gs_default_candidates(uint32_t max_degree, uint32_t* out, uint64_t* count);
/* group_cost.cpp:36-53 oracle_gs with cost_model_evaluator(dim, {workers,
 * lambda}) (:9-28), evaluated on device. cands NULL: default candidates of
 * the path's max degree; table gets one cost per candidate (capacity 33 when
 * cands is NULL); *ncand_out = candidates evaluated. */
int pg_gs_oracle_cost(pg_path p, uint64_t dim, int workers, double lambda, const uint32_t* cands,
                      uint64_t ncand, uint32_t* best, double* table, uint64_t* ncand_out);
/* group_cost.cpp:9-24 grouping_cost for a built grouping */
int pg_grouping_cost(pg_groups G, uint64_t dim, int workers, double lambda, double* cost);
/* train.hpp:35-54 measured_evaluator + group_cost.cpp:36-53 oracle_gs on
 * the device ("oracle:measured"): per candidate gs, the path is grouped and
 * the PG_AGG_GROUPED aggregation of a U(0,1) input (mt19937_64(derive_seed(
 * seed, 17)), parent-frontier rows x dim) is timed with CUDA events, median
 * of `repeats`; argmin, ties -> smaller gs. table[i] = seconds. cands NULL:
 * default_gs_candidates(max degree). Timing based: not bit-reproducible. */
int pg_gs_oracle_measured(pg_path p, uint64_t dim, int repeats, uint64_t seed, const uint32_t* cands,
                          uint64_t ncand, uint32_t* best, double* table, uint64_t* ncand_out);

/* grouping.cpp:7-27 group_neighbors over a path (or the whole graph). The
 * grouping borrows its base, which must outlive it (grouping.hpp:10-13). */
int pg_group(pg_path p, uint32_t gs, pg_groups* out);
int pg_group_graph(pg_graph g, uint32_t gs, pg_groups* out);
int pg_groups_info(pg_groups G, uint32_t* gs, uint64_t* count, uint32_t* dests);
int pg_groups_export(pg_groups G, uint32_t* dest, uint64_t* edge_begin, uint64_t* edge_end,
                     uint64_t* dest_groups);
int pg_groups_destroy(pg_groups G);

/* ---------------- backward aggregate ---------------- */

/* aggregate.hpp:56-122 aggregate_pull<float>: out[D x dim] (+)=
 * A_path * in, where in rows are the path's LOCAL source ids
 * (in_rows == |S|) — the reference operator on device pointers. */
int pg_aggregate_pull(pg_groups G, const float* in_dev, uint64_t in_rows, uint64_t ld_in,
                      float* out_dev, uint64_t ld_out, uint64_t dim, unsigned flags,
                      void* stream);
/* The reference's timed backward-aggregation stage (engine.hpp:331-338):
 *   y_used = gather_rows(y_grad, path.src_pos_in_parent);
 *   aggregate_pull(groups, y_used, x_grad)
 * with the gather folded into the edge stream. y_dev rows follow the
 * parent frontier (y_rows == parent_rows); x_dev has the path's D rows. */
int pg_backward_aggregate(pg_groups G, const float* y_dev, uint64_t y_rows, uint64_t ld_in,
                          float* x_dev, uint64_t ld_out, uint64_t dim, unsigned flags,
                          void* stream);
/* Same stage on destination rows [row_begin, row_end) of the path (dest
 * local order), for destination-row sharding (pg_path_shard_bounds):
 * x_dev holds row_end - row_begin rows, row r = destination row_begin + r. */
int pg_backward_aggregate_rows(pg_groups G, uint32_t row_begin, uint32_t row_end,
                               const float* y_dev, uint64_t y_rows, uint64_t ld_in, float* x_dev,
                               uint64_t ld_out, uint64_t dim, unsigned flags, void* stream);
/* Host-buffer drop-ins for DenseMatrix<float> callers (row-major, ld = cols):
 * copy in, run, copy out, synchronise. Pinned (cudaHostAlloc /
 * cudaHostRegister) buffers are DMA'd directly; pageable ones (a
 * std::vector) are staged through library-owned pinned slots by host
 * threads (all cores up to 16, $PG_STAGE_THREADS), overlapped with the
 * copies (Reddit layer 0: ~26.5 ms pinned, ~31 ms pageable, vs ~105 ms for
 * driver-staged pageable copies). */
int pg_aggregate_pull_host(pg_groups G, const float* in_host, uint64_t in_rows, uint64_t dim,
                           float* out_host, unsigned flags, uint64_t* counters);
int pg_backward_aggregate_host(pg_groups G, const float* y_host, uint64_t y_rows, uint64_t dim,
                               float* x_host, unsigned flags, uint64_t* counters);
/* aggregate_pull<double> — the reference's default precision
 * (run_config.hpp:53 Precision::F64): the same operators on f64 rows with the
 * f64 path weights, Deterministic order (bit-exact with the reference's
 * f64 build; PG_AGG_FAST gives the same result; PG_AGG_GROUPED is fp32-only).
 * Device rows need an even ld and a 16-byte aligned base; the host variants
 * take DenseMatrix<double> rows (ld = cols) and are synchronous. */
int pg_aggregate_pull_f64(pg_groups G, const double* in_dev, uint64_t in_rows, uint64_t ld_in, double* out_dev,
                          uint64_t ld_out, uint64_t dim, unsigned flags, void* stream);
int pg_backward_aggregate_f64(pg_groups G, const double* y_dev, uint64_t y_rows, uint64_t ld_in, double* x_dev,
                              uint64_t ld_out, uint64_t dim, unsigned flags, void* stream);
int pg_aggregate_pull_host_f64(pg_groups G, const double* in_host, uint64_t in_rows, uint64_t dim,
                               double* out_host, unsigned flags, uint64_t* counters);
int pg_backward_aggregate_host_f64(pg_groups G, const double* y_host, uint64_t y_rows, uint64_t dim,
                                   double* x_host, unsigned flags, uint64_t* counters);
/* StageCounters (aggregate.hpp:23-39) of one call, analytically:
 * {edges_traversed, groups_executed, atomic_commits}. */
int pg_stage_counters(pg_groups G, uint64_t dim, unsigned flags, uint64_t* counters);
/* Edge-balanced destination-row split for multi-GPU: bounds
 * [world+1] in dest-local row order, cut at E*r/world. */
int pg_path_shard_bounds(pg_path p, uint32_t world, uint32_t* bounds);

/* Multi-GPU: after a padded allgather of y_grad row shards, parent row p
 * lives at row map[p] of a new_rows-row buffer. Installs the remapped edge
 * stream on this grouping (pg_backward_aggregate* then expect
 * y_rows == new_rows); map NULL removes it. map: host u32[parent_rows]. */
int pg_groups_remap_sources(pg_groups G, const uint32_t* map, uint64_t map_len, uint64_t new_rows);

/* Source-row segments: cuts[0..nseg] (cuts[0] = 0, cuts[nseg] = input rows)
 * split every destination's edge list by source row. Edges are sorted by
 * source within a destination, so running segments 0..nseg-1 in order —
 * the first with PG_AGG_OVERWRITE (or onto the caller's initial output),
 * the rest accumulating — reproduces the serial fp32 order bit for bit.
 * This lets compute on rows that have arrived overlap the transfer of the
 * rest (H2D, or per-rank broadcasts in the multi-GPU exchange).
 * cuts NULL / nseg 0 clears. */
int pg_groups_set_segments(pg_groups G, const uint64_t* cuts, uint32_t nseg);
int pg_backward_aggregate_segment(pg_groups G, uint32_t seg, uint32_t row_begin, uint32_t row_end,
                                  const float* y_dev, uint64_t y_rows, uint64_t ld_in, float* x_dev,
                                  uint64_t ld_out, uint64_t dim, unsigned flags, void* stream);

/* ---------------- multi-GPU ----------------
 * One NCCL rank per device (NCCL is dlopen'ed at first use: the copy already
 * in the process, else libnccl.so.2). The destinations of each execution
 * path are sharded by edge count (pg_path_shard_bounds; the parent frontier
 * of path i is cut where path i-1's destinations are). Rank 0 makes the id
 * (pg_comm_unique_id) and the caller ships its 128 bytes to every rank over
 * its own bootstrap channel (MPI, torch.distributed, a file). */
typedef struct pg_comm_s* pg_comm;
#define PG_COMM_ID_BYTES 128
int pg_comm_unique_id(uint8_t* id);
int pg_comm_init_rank(int device, const uint8_t* id, int world, int rank, pg_comm* out);
int pg_comm_info(pg_comm c, int* world, int* rank, int* nccl_version);
int pg_comm_destroy(pg_comm c);
/* In-place all-gather-v of a pitched row matrix over the communicator: rank
 * s owns rows [bounds[s], bounds[s+1]) (world+1 cuts); whole ld-float rows
 * are broadcast in rank order on the library's communication stream,
 * ordered after and before `stream`. */
int pg_comm_allgather_rows(pg_comm c, float* rows, uint64_t ld, const uint32_t* bounds, void* stream);
/* The timed stage (engine.hpp:331-338) row-sharded: this rank holds its
 * parent rows [parent_bounds[rank], parent_bounds[rank+1]) of y_dev (the
 * full P x ld frontier-order matrix); the call completes y_dev from the
 * other ranks (per-owner broadcasts on the communication stream) and
 * aggregates destination rows [dest_bounds[rank], dest_bounds[rank+1]) into
 * x_dev. Default: source-segment pass k runs as soon as owner k's rows have
 * landed (the exchange overlaps the SpMM; passes in owner order are the
 * serial fp32 order, so every row is bit-identical to one GPU);
 * PG_SHARD_SINGLE_PASS waits for the whole exchange, then one pass.
 * Sets the grouping's source segments (pg_groups_set_segments) to the
 * owner cuts. Asynchronous on `stream`. */
#define PG_SHARD_SINGLE_PASS 8u
int pg_backward_aggregate_sharded(pg_comm c, pg_groups G, const uint32_t* parent_bounds,
                                  const uint32_t* dest_bounds, float* y_dev, uint64_t y_rows, uint64_t ld_in,
                                  float* x_dev, uint64_t ld_out, uint64_t dim, unsigned flags, void* stream);

/* ---------------- dense helpers of backward_epp ---------------- */

/* dense_matrix.hpp:78-95 gemm_a_bt: out[n x m] = a[n x k] * b[m x k]^T */
int pg_gemm_a_bt(const float* a, uint64_t lda, const float* b, uint64_t ldb, float* out,
                 uint64_t ldo, uint64_t n, uint64_t m, uint64_t k, void* stream);
/* gemm_a_bt with flags: PG_GEMM_TF32X3 runs it on the tensor cores
 * (tcgen05.mma kind::tf32, operands split hi + lo, 3 MMAs per K step, fp32
 * accumulation in TMEM): within the reference's 1e-5 relative / 1e-6
 * absolute fp32 tolerance of the exact product, NOT bit-exact (the K sum is
 * re-associated). Needs a 16-byte aligned a with lda % 4 == 0. flags 0 =
 * pg_gemm_a_bt (bit-exact). */
#define PG_GEMM_TF32X3 1u
int pg_gemm_a_bt_ex(const float* a, uint64_t lda, const float* b, uint64_t ldb, float* out,
                    uint64_t ldo, uint64_t n, uint64_t m, uint64_t k, unsigned flags, void* stream);
/* dense_matrix.hpp:114-121 relu_backward */
int pg_relu_backward(const float* grad, uint64_t ldg, const float* pre, uint64_t ldp, float* out,
                     uint64_t ldo, uint64_t rows, uint64_t cols, void* stream);
/* engine.hpp:162-169 gather_rows (ids on device) */
int pg_gather_rows(const float* src, uint64_t lds, const uint32_t* ids_dev, uint64_t k, float* out,
                   uint64_t ldo, uint64_t cols, void* stream);
/* device pointers to a path's frontier-order arrays for chained drivers */
int pg_path_device_arrays(pg_path p, const uint32_t** dest, const uint32_t** srcpos,
                          const uint64_t** offsets);

/* Device memory for callers without the CUDA runtime headers (the C++
 * header's DeviceMatrix): stream-less, synchronous. */
int pg_device_alloc(int device, uint64_t bytes, void** out);
int pg_device_free(int device, void* p);
int pg_memcpy_h2d(int device, void* dst, const void* src, uint64_t bytes);
int pg_memcpy_d2h(int device, void* dst, const void* src, uint64_t bytes);
int pg_memset_zero(int device, void* dst, uint64_t bytes);
int pg_device_synchronize(int device);
/* Kernels launched by this library so far in this process (every launch,
 * all devices and threads). */
uint64_t pg_launch_count(void);

/* ---------------- the GCN chain around the aggregation (engine.hpp) ----------------
 * Device-resident and bit-exact with the reference's f32 build. Matrices are
 * device fp32, rows x cols with row pitch ld floats (the reference's
 * DenseMatrix<float> is ld = cols; ld a multiple of 4 with a 16-byte-aligned
 * base lets the SpMM use 128-bit gathers). All calls are asynchronous on
 * `stream` except where a counter is returned. */
typedef struct pg_mat {
    float* data;
    uint64_t rows, cols, ld;
} pg_mat;

/* Whole-matrix copies between a host DenseMatrix<float> (row-major, ld =
 * cols) and a pitched device pg_mat: one flat copy plus an on-device repack
 * when the pitches differ (not one copy per row). Synchronous. */
int pg_mat_upload(int device, pg_mat dst, const float* host);
int pg_mat_download(int device, float* host, pg_mat src);

/* dense_matrix.hpp:40-55 gemm (b_transposed = 0) and :78-95 gemm_a_bt
 * (b_transposed = 1): ascending k, separately rounded, + 0 */
int pg_gemm(pg_mat a, pg_mat b, int b_transposed, pg_mat out, void* stream);
/* dense_matrix.hpp:57-76 gemm_at_b: out = a^T b, or with a_rows (device
 * u32[b.rows]) out = gather_rows(a, a_rows)^T b (engine.hpp:323-324 fused) */
int pg_gemm_at_b(pg_mat a, const uint32_t* a_rows, pg_mat b, pg_mat out, void* stream);
/* the same with flags: PG_GEMM_TF32X3 = on the tensor cores, split-K over the
 * rows (CTA partials added in a fixed order, deterministic), 3xTF32 products:
 * within the fp32 tolerance of the exact W', NOT bit-exact. a and b need
 * 16-byte aligned rows (ld % 4 == 0). Tuning "gemm_tc" = 1 routes the
 * chains' W' and y_grad GEMMs here (when aligned). */
int pg_gemm_at_b_ex(pg_mat a, const uint32_t* a_rows, pg_mat b, pg_mat out, unsigned flags, void* stream);
/* dense_matrix.hpp:98-104 relu and :116-135 row_softmax (expf bit-exact
 * with glibc 2.39 on FMA x86-64) */
int pg_relu(pg_mat x, pg_mat out, void* stream);
int pg_row_softmax(pg_mat x, pg_mat out, void* stream);
/* engine.hpp:146-156 top_grad_from_probs: out = 0; out[v] = (probs[v] -
 * ref[v]) / |V_t| for v in vt (device u32[k]) */
int pg_top_grad_from_probs(pg_mat probs, pg_mat ref, const uint32_t* vt_dev, uint64_t k, pg_mat out,
                           void* stream);
/* aggregate.hpp:127-210 aggregate_pull_filtered (Deterministic) over a
 * full-graph grouping: destinations outside frontier level dest_level keep
 * their rows, sources outside src_level are skipped. counters (nullable,
 * synchronising): {edges_traversed, groups_executed, edges_skipped,
 * groups_skipped}. */
int pg_aggregate_pull_filtered(pg_groups G, pg_frontiers F, uint64_t dest_level, uint64_t src_level,
                               const float* in_dev, uint64_t in_rows, uint64_t ld_in, float* out_dev,
                               uint64_t ld_out, uint64_t dim, unsigned flags, uint64_t* counters,
                               void* stream);
/* engine.hpp:114-140 forward over a full-graph grouping: per layer
 * y[l] = pull(x_l), pre[l] = y[l] W[l], x[l] = relu(pre[l]) (softmax at the
 * last layer); x_0 = x0 and x[l] holds X^(l+1). Arrays of `layers`. */
int pg_forward(pg_groups graph_groups, pg_mat x0, const pg_mat* w, uint64_t layers, pg_mat* y, pg_mat* pre,
               pg_mat* x, void* stream);
/* engine.hpp:267-349 backward_epp: path_groups[i] groups the execution
 * path of layer L-1-i; y/pre/w are the forward artefacts (n rows);
 * top_grad n x dims[L-1]; w_grads[l] receives W^(l)'. gather_mode 0 = Local
 * (compact frontier-order matrices, relu_backward fused into the SpMM
 * epilogue unless x_grads is given), 1 = Global. x_grads (nullable, Local
 * only): |levels[i+1]| x in_dim rows per path i. edges_per_layer (nullable):
 * backward_edges_per_layer. Stale fingerprints / depth -> PG_ERR_CONFIG. */
int pg_backward_epp(const pg_groups* path_groups, pg_frontiers F, uint64_t layers, const pg_mat* y,
                    const pg_mat* pre, pg_mat top_grad, const pg_mat* w, uint64_t expected_fingerprint,
                    int gather_mode, pg_mat* w_grads, pg_mat* x_grads, uint64_t* edges_per_layer, void* stream);
/* engine.hpp:177-214 backward_all_active (Alg. 1) over a full-graph
 * grouping; x_grads (nullable) n x in_dim, layer L-1 first. */
int pg_backward_all_active(pg_groups graph_groups, uint64_t layers, const pg_mat* y, const pg_mat* pre,
                           pg_mat top_grad, const pg_mat* w, pg_mat* w_grads, pg_mat* x_grads,
                           uint64_t* edges_per_layer, void* stream);
/* engine.hpp:218-257 backward_ifelse: the full-graph traversal with the
 * frontier activity filters; edges_per_layer (nullable, synchronising). */
int pg_backward_ifelse(pg_groups graph_groups, pg_frontiers F, uint64_t layers, const pg_mat* y,
                       const pg_mat* pre, pg_mat top_grad, const pg_mat* w, pg_mat* w_grads, pg_mat* x_grads,
                       uint64_t* edges_per_layer, void* stream);

#ifdef __cplusplus
}
#endif
#endif
