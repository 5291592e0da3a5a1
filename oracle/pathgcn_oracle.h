/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference (pathgcn, /root/reference/proj/core)
 * algorithms on the backward-aggregation hot path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * Pinned against the reference's own golden vectors (tests/test_oracle_golden.py)
 * and against the reference itself compiled from source into
 * oracle/_ref/libpathgcn_ref.so (tests/test_oracle_vs_ref.py).
 *
 * Conventions mirror the reference types (types.hpp:9-25): vertex ids u32,
 * edge offsets u64, weights f64, row-major matrices with ld = cols.
 */
#ifndef PATHGCN_ORACLE_H
#define PATHGCN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- libstdc++ <random> restatement (inputs only) ---- */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void orc_mt64_seed(orc_mt64* r, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* r);
double orc_canonical(orc_mt64* r);
uint64_t orc_uniform_int(orc_mt64* r, uint64_t a, uint64_t b);
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream);

uint32_t orc_gen_rmat(uint32_t n, uint64_t m, double a, double b, double c, double d,
                      uint64_t seed, uint32_t* pairs_out);
uint64_t orc_training_set_size(uint32_t n, double ratio);
int orc_sample_training_set(uint32_t n, double ratio, uint64_t seed, uint32_t* out);
void orc_random_matrix_f32(uint64_t rows, uint64_t cols, uint64_t seed, double lo, double hi,
                           float* out);

/* ---- graph load ---- */
int orc_build_undirected_csr(int64_t n_hint, const uint32_t* pairs, uint64_t npairs,
                             uint32_t* n_out, uint64_t* m_out, uint64_t** offsets_out,
                             uint32_t** nbrs_out);
void orc_assign_edge_weights(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                             int symnorm, double* w);
void orc_free(void* p);
uint64_t orc_graph_fingerprint(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs);
uint64_t orc_training_fingerprint(const uint32_t* vt, uint64_t k);
uint64_t orc_path_fingerprint(uint64_t graph_fp, uint64_t train_fp, uint64_t layers);

/* ---- execution-path build ---- */
int orc_compute_frontiers(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                          const uint32_t* vt, uint64_t k, uint64_t L, uint32_t* levels,
                          uint64_t* sizes);
int orc_extract_path(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs, const double* w,
                     const uint32_t* dests, uint32_t D, const uint32_t* parent, uint32_t P,
                     uint64_t* p_offsets, uint32_t* p_nbrs, double* p_w, uint32_t* src,
                     uint32_t* srcpos, uint64_t* E_out, uint32_t* S_out);

/* ---- group partition + gs selection ---- */
uint64_t orc_group_count(uint32_t D, const uint64_t* offsets, uint32_t gs);
int orc_group_neighbors(uint32_t D, const uint64_t* offsets, uint32_t gs, uint32_t* g_dest,
                        uint64_t* g_begin, uint64_t* g_end, uint64_t* dest_groups);
uint32_t orc_regression_gs(uint32_t n_vertices, uint64_t n_edges, double avg_degree,
                           const double* beta);
uint32_t orc_path_regression_gs(uint32_t D, uint64_t E);
double orc_grouping_cost(uint32_t D, const uint64_t* offsets, uint32_t gs, uint64_t dim,
                         int workers, double lambda);
uint64_t orc_default_candidates(uint32_t max_degree, uint32_t* out);
int orc_oracle_gs_cost(uint32_t D, const uint64_t* offsets, const uint32_t* cands,
                       uint64_t ncand, uint64_t dim, int workers, double lambda, uint32_t* best,
                       double* table);
uint64_t orc_fast_atomic_commits(uint32_t D, const uint64_t* offsets, uint32_t gs, uint64_t dim);

/* ---- backward aggregation + dense helpers ---- */
void orc_aggregate_pull_f32(uint32_t D, const uint64_t* offsets, const uint32_t* nbrs,
                            const double* w, const float* in, uint64_t dim, float* out);
void orc_aggregate_pull_f64(uint32_t D, const uint64_t* offsets, const uint32_t* nbrs,
                            const double* w, const double* in, uint64_t dim, double* out);
void orc_gather_rows_f32(const float* src, uint64_t cols, const uint32_t* ids, uint64_t k,
                         float* out);
void orc_gemm_a_bt_f32(const float* a, uint64_t n, uint64_t k, const float* b, uint64_t m,
                       float* out);
void orc_gemm_a_bt_f64(const double* a, uint64_t n, uint64_t k, const double* b, uint64_t m,
                       double* out);
void orc_relu_backward_f32(const float* grad, const float* pre, uint64_t count, float* out);

/* ---- the GCN chain around the aggregation (engine.hpp), f32 ---- */
void orc_gemm_f32(const float* a, uint64_t n, uint64_t k, const float* b, uint64_t m, float* out);
void orc_gemm_at_b_f32(const float* a, uint64_t n, uint64_t r, const float* b, uint64_t c, float* out);
void orc_relu_f32(const float* x, uint64_t count, float* out);
void orc_row_softmax_f32(const float* x, uint64_t rows, uint64_t cols, float* out);
void orc_top_grad_f32(const float* probs, const float* ref, uint64_t n, uint64_t c, const uint32_t* vt,
                      uint64_t k, float* out);
void orc_aggregate_pull_filtered_f32(uint32_t D, const uint64_t* offsets, const uint32_t* nbrs,
                                     const double* w, const float* in, uint64_t dim,
                                     const uint8_t* dest_active, const uint8_t* src_active, uint32_t gs,
                                     float* out, uint64_t* counters);

#ifdef __cplusplus
}
#endif
#endif
