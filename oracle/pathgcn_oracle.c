/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product path.
 *
 * Plain-C restatement of the reference algorithms on the backward-aggregation
 * hot path of arXiv 2204.02662's pathgcn (/root/reference/proj/core). Each
 * function cites the reference file:line it restates. Build: oracle/Makefile
 * (-ffp-contract=off: mul and add stay separately rounded, like the reference's
 * default-flag x86-64 build).
 *
 * Pinned by tests/test_oracle_golden.py (the reference's own known-answer
 * tests) and tests/test_oracle_vs_ref.py (the reference compiled from source,
 * oracle/_ref/libpathgcn_ref.so).
 */
#include "pathgcn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* libstdc++ <random> (GCC 13): std::mt19937_64, generate_canonical<double,53>,
 * uniform_int_distribution<size_t> (Lemire nearly-divisionless, 128-bit
 * product). Only used to synthesise the same inputs the reference draws in
 * rmat.cpp:20-43, training_set.cpp:36-42 and fixtures.hpp:96-104.        */

void orc_mt64_seed(orc_mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* r) {
    static const uint64_t UPPER = 0xFFFFFFFF80000000ull, LOWER = 0x7FFFFFFFull;
    static const uint64_t MATRIX = 0xB5026F5AA96619E9ull;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & UPPER) | (r->mt[(i + 1) % 312] & LOWER);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= MATRIX;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* generate_canonical<double, 53>(mt19937_64): one draw, divided by 2^64,
 * clamped below 1. */
double orc_canonical(orc_mt64* r) {
    double sum = (double)orc_mt64_next(r);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* uniform_int_distribution<size_t>(a, b) over a 64-bit engine. */
uint64_t orc_uniform_int(orc_mt64* r, uint64_t a, uint64_t b) {
    uint64_t urange = b - a;
    if (urange == UINT64_MAX) return orc_mt64_next(r) + a;
    uint64_t range = urange + 1;
    unsigned __int128 product = (unsigned __int128)orc_mt64_next(r) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)orc_mt64_next(r) * range;
            low = (uint64_t)product;
        }
    }
    return (uint64_t)(product >> 64) + a;
}

/* engine.hpp:60-68 */
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
    uint64_t h = seed ^ (0x9e3779b97f4a7c15ull + stream);
    h ^= h >> 30;
    h *= 0xbf58476d1ce4e5b9ull;
    h ^= h >> 27;
    h *= 0x94d049bb133111ebull;
    h ^= h >> 31;
    return h;
}

/* rmat.cpp:10-44 — pads n to 2^levels, draws m raw pairs. Returns n_pad. */
uint32_t orc_gen_rmat(uint32_t n, uint64_t m, double a, double b, double c, double d,
                      uint64_t seed, uint32_t* pairs_out) {
    (void)d;
    if (n == 0) return 0;
    int levels = 0;
    while (((uint32_t)1 << levels) < n) ++levels;
    orc_mt64 rng;
    orc_mt64_seed(&rng, seed);
    for (uint64_t i = 0; i < m; ++i) {
        uint32_t src = 0, dst = 0;
        for (int lvl = levels - 1; lvl >= 0; --lvl) {
            double r = orc_canonical(&rng) * (1.0 - 0.0) + 0.0;
            if (r < a) {
            } else if (r < a + b) {
                dst |= (uint32_t)1 << lvl;
            } else if (r < a + b + c) {
                src |= (uint32_t)1 << lvl;
            } else {
                src |= (uint32_t)1 << lvl;
                dst |= (uint32_t)1 << lvl;
            }
        }
        pairs_out[2 * i] = src;
        pairs_out[2 * i + 1] = dst;
    }
    return (uint32_t)1 << levels;
}

/* training_set.cpp:32-35 */
uint64_t orc_training_set_size(uint32_t n, double ratio) {
    long long k = llround(ratio * (double)n);
    return k < 1 ? 1 : (uint64_t)k;
}

static int cmp_u32(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    return a < b ? -1 : a > b;
}

/* training_set.cpp:28-49 — partial Fisher-Yates, then sorted. */
int orc_sample_training_set(uint32_t n, double ratio, uint64_t seed, uint32_t* out) {
    if (n == 0 || !(ratio > 0.0) || ratio > 1.0) return 2;
    uint64_t k = orc_training_set_size(n, ratio);
    uint32_t* ids = (uint32_t*)malloc((size_t)n * 4);
    for (uint32_t i = 0; i < n; ++i) ids[i] = i;
    orc_mt64 rng;
    orc_mt64_seed(&rng, seed);
    for (uint64_t i = 0; i < k; ++i) {
        uint64_t j = orc_uniform_int(&rng, i, (uint64_t)n - 1);
        uint32_t t = ids[i];
        ids[i] = ids[j];
        ids[j] = t;
    }
    memcpy(out, ids, k * 4);
    free(ids);
    qsort(out, k, 4, cmp_u32);
    return 0;
}

/* fixtures.hpp:96-104 — U(lo, hi) doubles cast to float. */
void orc_random_matrix_f32(uint64_t rows, uint64_t cols, uint64_t seed, double lo, double hi,
                           float* out) {
    orc_mt64 rng;
    orc_mt64_seed(&rng, seed);
    for (uint64_t i = 0; i < rows * cols; ++i)
        out[i] = (float)(orc_canonical(&rng) * (hi - lo) + lo);
}

/* ------------------------------------------------------------------------ */
/* graph load                                                              */

static void radix_sort_u64(uint64_t* keys, uint64_t n, int key_bits) {
    uint64_t* tmp = (uint64_t*)malloc((size_t)(n ? n : 1) * 8);
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    for (int shift = 0; shift < key_bits; shift += 16) {
        uint64_t count[65537];
        memset(count, 0, sizeof(count));
        for (uint64_t i = 0; i < n; ++i) count[((src[i] >> shift) & 0xFFFF) + 1]++;
        for (int d = 0; d < 65536; ++d) count[d + 1] += count[d];
        for (uint64_t i = 0; i < n; ++i) dst[count[(src[i] >> shift) & 0xFFFF]++] = src[i];
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) memcpy(keys, src, (size_t)n * 8);
    free(tmp);
}

/* csr_graph.cpp:33-63 — drop self loops, symmetrise, sort (u, v)
 * lexicographically (== sorting u<<32|v), unique, count offsets.
 * n = max(n_hint, 1 + max id). Returns 2 (ConfigError) for an empty list
 * without a hint. */
int orc_build_undirected_csr(int64_t n_hint, const uint32_t* pairs, uint64_t npairs,
                             uint32_t* n_out, uint64_t* m_out, uint64_t** offsets_out,
                             uint32_t** nbrs_out) {
    uint32_t n = n_hint >= 0 ? (uint32_t)n_hint : 0;
    int any = 0;
    for (uint64_t i = 0; i < npairs; ++i) {
        uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
        if (u == v) continue;
        any = 1;
        uint32_t mx = (u > v ? u : v) + 1;
        if (mx > n) n = mx;
    }
    if (!any && n_hint < 0) return 2;
    uint64_t* dir = (uint64_t*)malloc((size_t)(2 * npairs + 1) * 8);
    uint64_t nd = 0;
    for (uint64_t i = 0; i < npairs; ++i) {
        uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
        if (u == v) continue;
        dir[nd++] = ((uint64_t)u << 32) | v;
        dir[nd++] = ((uint64_t)v << 32) | u;
    }
    radix_sort_u64(dir, nd, 64);
    uint64_t m = 0;
    for (uint64_t i = 0; i < nd; ++i)
        if (i == 0 || dir[i] != dir[i - 1]) dir[m++] = dir[i];
    uint64_t* offsets = (uint64_t*)calloc((size_t)n + 1, 8);
    uint32_t* nbrs = (uint32_t*)malloc((size_t)(m ? m : 1) * 4);
    for (uint64_t i = 0; i < m; ++i) offsets[(dir[i] >> 32) + 1]++;
    for (uint32_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
    for (uint64_t i = 0; i < m; ++i) nbrs[i] = (uint32_t)dir[i];
    free(dir);
    *n_out = n;
    *m_out = m;
    *offsets_out = offsets;
    *nbrs_out = nbrs;
    return 0;
}

/* csr_graph.cpp:65-77 — unit: 1.0; sym-norm: 1/sqrt(deg u * deg v) in f64. */
void orc_assign_edge_weights(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                             int symnorm, double* w) {
    for (uint32_t u = 0; u < n; ++u) {
        const double du = (double)(offsets[u + 1] - offsets[u]);
        for (uint64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
            if (!symnorm) {
                w[e] = 1.0;
                continue;
            }
            const uint32_t v = nbrs[e];
            const double dv = (double)(offsets[v + 1] - offsets[v]);
            w[e] = 1.0 / sqrt(du * dv);
        }
    }
}

void orc_free(void* p) { free(p); }

static void fnv_mix(uint64_t* h, uint64_t x) {
    for (int i = 0; i < 8; ++i) {
        *h ^= (x >> (8 * i)) & 0xFF;
        *h *= 1099511628211ull;
    }
}

/* csr_graph.cpp:19-31 */
uint64_t orc_graph_fingerprint(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs) {
    uint64_t h = 1469598103934665603ull;
    fnv_mix(&h, n);
    for (uint64_t i = 0; i <= n; ++i) fnv_mix(&h, offsets[i]);
    for (uint64_t e = 0; e < offsets[n]; ++e) fnv_mix(&h, nbrs[e]);
    return h;
}

/* training_set.cpp:15-26 */
uint64_t orc_training_fingerprint(const uint32_t* vt, uint64_t k) {
    uint64_t h = 1469598103934665603ull;
    fnv_mix(&h, k);
    for (uint64_t i = 0; i < k; ++i) fnv_mix(&h, vt[i]);
    return h;
}

/* execution_path.cpp:17-22 */
uint64_t orc_path_fingerprint(uint64_t graph_fp, uint64_t train_fp, uint64_t layers) {
    uint64_t h = graph_fp;
    h ^= train_fp + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= layers + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

/* ------------------------------------------------------------------------ */
/* execution-path build                                                    */

/* frontier.cpp:7-26 — levels[0] = V_t; levels[k+1] = ascending scan of the
 * mark array set over N(levels[k]) (walk semantics). `levels` holds L+1
 * slices of n entries; sizes[k] = |levels[k]|. 2 = ConfigError. */
int orc_compute_frontiers(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                          const uint32_t* vt, uint64_t k, uint64_t L, uint32_t* levels,
                          uint64_t* sizes) {
    if (L < 1 || k == 0) return 2;
    memcpy(levels, vt, k * 4);
    sizes[0] = k;
    unsigned char* mark = (unsigned char*)malloc((size_t)n + 1);
    for (uint64_t lv = 0; lv < L; ++lv) {
        memset(mark, 0, (size_t)n + 1);
        const uint32_t* cur = levels + lv * (uint64_t)n;
        for (uint64_t i = 0; i < sizes[lv]; ++i) {
            uint32_t v = cur[i];
            for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) mark[nbrs[e]] = 1;
        }
        uint32_t* next = levels + (lv + 1) * (uint64_t)n;
        uint64_t cnt = 0;
        for (uint32_t v = 0; v < n; ++v)
            if (mark[v]) next[cnt++] = v;
        sizes[lv + 1] = cnt;
    }
    free(mark);
    return 0;
}

/* execution_path.cpp:24-88 for one layer: dests = levels[L-l],
 * parent = levels[L-l-1]. Keeps u in N(v) ∩ parent in parent-CSR order with
 * bitwise-copied weights. src = sorted unique kept sources (the reference's
 * sort+unique, :66-70, here as an ascending scan of a mark array — the same
 * set in the same order); neighbors = rank of the global source in src
 * (:72-79); srcpos = index of src[s] in the parent array (:81-86).
 * Output capacities: p_nbrs/p_w >= sum of deg(dests), src/srcpos >= P. */
int orc_extract_path(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs, const double* w,
                     const uint32_t* dests, uint32_t D, const uint32_t* parent, uint32_t P,
                     uint64_t* p_offsets, uint32_t* p_nbrs, double* p_w, uint32_t* src,
                     uint32_t* srcpos, uint64_t* E_out, uint32_t* S_out) {
    unsigned char* in_parent = (unsigned char*)calloc((size_t)n + 1, 1);
    unsigned char* used = (unsigned char*)calloc((size_t)n + 1, 1);
    uint32_t* rank = (uint32_t*)malloc((size_t)(n + 1) * 4);
    uint32_t* ppos = (uint32_t*)malloc((size_t)(n + 1) * 4);
    for (uint32_t i = 0; i < P; ++i) {
        in_parent[parent[i]] = 1;
        ppos[parent[i]] = i;
    }
    p_offsets[0] = 0;
    uint64_t wpos = 0;
    for (uint32_t i = 0; i < D; ++i) {
        const uint32_t v = dests[i];
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const uint32_t u = nbrs[e];
            if (!in_parent[u]) continue;
            p_nbrs[wpos] = u; /* global id for now */
            p_w[wpos] = w[e];
            used[u] = 1;
            ++wpos;
        }
        p_offsets[i + 1] = wpos;
    }
    uint32_t S = 0;
    for (uint32_t u = 0; u < n; ++u)
        if (used[u]) {
            rank[u] = S;
            src[S] = u;
            srcpos[S] = ppos[u];
            ++S;
        }
    for (uint64_t e = 0; e < wpos; ++e) p_nbrs[e] = rank[p_nbrs[e]];
    *E_out = wpos;
    *S_out = S;
    free(in_parent);
    free(used);
    free(rank);
    free(ppos);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* group partition + group-size selection                                  */

/* grouping.cpp:15-20 */
uint64_t orc_group_count(uint32_t D, const uint64_t* offsets, uint32_t gs) {
    uint64_t total = 0;
    for (uint32_t v = 0; v < D; ++v) {
        uint32_t deg = (uint32_t)(offsets[v + 1] - offsets[v]);
        total += (deg + gs - 1) / gs;
    }
    return total;
}

/* grouping.cpp:7-27 — 2 = ConfigError (gs == 0). */
int orc_group_neighbors(uint32_t D, const uint64_t* offsets, uint32_t gs, uint32_t* g_dest,
                        uint64_t* g_begin, uint64_t* g_end, uint64_t* dest_groups) {
    if (gs == 0) return 2;
    uint64_t total = 0;
    dest_groups[0] = 0;
    for (uint32_t v = 0; v < D; ++v) {
        uint32_t deg = (uint32_t)(offsets[v + 1] - offsets[v]);
        total += (deg + gs - 1) / gs;
        dest_groups[v + 1] = total;
    }
    uint64_t i = 0;
    for (uint32_t v = 0; v < D; ++v)
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; e += gs) {
            g_dest[i] = v;
            g_begin[i] = e;
            g_end[i] = e + gs < offsets[v + 1] ? e + gs : offsets[v + 1];
            ++i;
        }
    return 0;
}

/* gs_model.cpp:64-74 (beta NULL = default_gs_model). */
uint32_t orc_regression_gs(uint32_t n_vertices, uint64_t n_edges, double avg_degree,
                           const double* beta) {
    static const double def[4] = {0.65538, 1.67431e-5, -2.24342e-6, 0.63641};
    const double* b = beta ? beta : def;
    const double raw = b[0] + b[1] * (double)n_vertices + b[2] * (double)n_edges + b[3] * avg_degree;
    const long long rounded = llround(raw);
    return rounded < 1 ? 1 : (uint32_t)rounded;
}

/* train.hpp:16-24 path_stats: |D|, directed pull-edge count, E/|D|. */
uint32_t orc_path_regression_gs(uint32_t D, uint64_t E) {
    const double avg = D == 0 ? 0.0 : (double)E / (double)D;
    return orc_regression_gs(D, E, avg, NULL);
}

/* group_cost.cpp:9-24 — round-robin loads over groups in order, atomic
 * writes (k-1)*dim per multi-group destination. -1.0 on W < 1. */
double orc_grouping_cost(uint32_t D, const uint64_t* offsets, uint32_t gs, uint64_t dim,
                         int workers, double lambda) {
    if (workers < 1 || gs == 0) return -1.0;
    uint64_t* load = (uint64_t*)calloc((size_t)workers, 8);
    uint64_t i = 0, atomic_writes = 0;
    for (uint32_t v = 0; v < D; ++v) {
        uint64_t k = 0;
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; e += gs) {
            uint64_t end = e + gs < offsets[v + 1] ? e + gs : offsets[v + 1];
            load[i % (uint64_t)workers] += (end - e) * dim;
            ++i;
            ++k;
        }
        if (k > 1) atomic_writes += (k - 1) * dim;
    }
    uint64_t max_load = 0;
    for (int w = 0; w < workers; ++w)
        if (load[w] > max_load) max_load = load[w];
    free(load);
    return (double)max_load + lambda * (double)atomic_writes;
}

/* group_cost.cpp:30-34 */
uint64_t orc_default_candidates(uint32_t max_degree, uint32_t* out) {
    uint64_t cnt = 0;
    uint32_t target = max_degree > 1 ? max_degree : 1;
    out[cnt++] = 1;
    while (out[cnt - 1] < target) {
        out[cnt] = out[cnt - 1] * 2;
        ++cnt;
    }
    return cnt;
}

/* group_cost.cpp:36-53 with cost_model_evaluator (:26-28): argmin, ties to
 * the smaller gs. 2 = ConfigError (empty candidate list / bad workers). */
int orc_oracle_gs_cost(uint32_t D, const uint64_t* offsets, const uint32_t* cands,
                       uint64_t ncand, uint64_t dim, int workers, double lambda, uint32_t* best,
                       double* table) {
    if (ncand == 0 || workers < 1) return 2;
    double best_cost = 0.0;
    uint32_t best_gs = 1;
    int first = 1;
    for (uint64_t i = 0; i < ncand; ++i) {
        if (cands[i] == 0) return 2;
        double c = orc_grouping_cost(D, offsets, cands[i], dim, workers, lambda);
        table[i] = c;
        if (first || c < best_cost || (c == best_cost && cands[i] < best_gs)) {
            first = 0;
            best_cost = c;
            best_gs = cands[i];
        }
    }
    *best = best_gs;
    return 0;
}

/* aggregate.hpp:107-111 + :119-120: Fast mode commits `width` atomics for
 * every group of a destination that owns more than one group. */
uint64_t orc_fast_atomic_commits(uint32_t D, const uint64_t* offsets, uint32_t gs, uint64_t dim) {
    uint64_t total = 0;
    for (uint32_t v = 0; v < D; ++v) {
        uint64_t deg = offsets[v + 1] - offsets[v];
        uint64_t k = (deg + gs - 1) / gs;
        if (k > 1) total += k * dim;
    }
    return total;
}

/* ------------------------------------------------------------------------ */
/* backward aggregation                                                    */

/* aggregate.hpp:69-83 (Deterministic): per destination and column, ascending
 * edge order, out += (T)w * in, then out += T(0). Accumulates into `out`. */
void orc_aggregate_pull_f32(uint32_t D, const uint64_t* offsets, const uint32_t* nbrs,
                            const double* w, const float* in, uint64_t dim, float* out) {
    for (uint32_t v = 0; v < D; ++v) {
        float* o = out + (uint64_t)v * dim;
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const float we = (float)w[e];
            const float* x = in + (uint64_t)nbrs[e] * dim;
            for (uint64_t j = 0; j < dim; ++j) o[j] += we * x[j];
        }
        for (uint64_t j = 0; j < dim; ++j) o[j] += 0.0f;
    }
}

void orc_aggregate_pull_f64(uint32_t D, const uint64_t* offsets, const uint32_t* nbrs,
                            const double* w, const double* in, uint64_t dim, double* out) {
    for (uint32_t v = 0; v < D; ++v) {
        double* o = out + (uint64_t)v * dim;
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const double we = w[e];
            const double* x = in + (uint64_t)nbrs[e] * dim;
            for (uint64_t j = 0; j < dim; ++j) o[j] += we * x[j];
        }
        for (uint64_t j = 0; j < dim; ++j) o[j] += 0.0;
    }
}

/* engine.hpp:162-169 */
void orc_gather_rows_f32(const float* src, uint64_t cols, const uint32_t* ids, uint64_t k,
                         float* out) {
    for (uint64_t i = 0; i < k; ++i) memcpy(out + i * cols, src + (uint64_t)ids[i] * cols, cols * 4);
}

/* dense_matrix.hpp:78-95 — ascending-k dot products, then + T(0). */
void orc_gemm_a_bt_f32(const float* a, uint64_t n, uint64_t k, const float* b, uint64_t m,
                       float* out) {
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < m; ++j) {
            float acc = 0.0f;
            for (uint64_t t = 0; t < k; ++t) acc += a[i * k + t] * b[j * k + t];
            out[i * m + j] = acc + 0.0f;
        }
}

void orc_gemm_a_bt_f64(const double* a, uint64_t n, uint64_t k, const double* b, uint64_t m,
                       double* out) {
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < m; ++j) {
            double acc = 0.0;
            for (uint64_t t = 0; t < k; ++t) acc += a[i * k + t] * b[j * k + t];
            out[i * m + j] = acc + 0.0;
        }
}

/* dense_matrix.hpp:114-121 */
void orc_relu_backward_f32(const float* grad, const float* pre, uint64_t count, float* out) {
    for (uint64_t i = 0; i < count; ++i) out[i] = pre[i] > 0.0f ? grad[i] : 0.0f;
}

/* ---- the GCN chain (engine.hpp / dense_matrix.hpp), f32 ---- */

/* dense_matrix.hpp:40-55 gemm: per i, k ascending, orow[j] += a[i][k]*b[k][j]; + 0 */
void orc_gemm_f32(const float* a, uint64_t n, uint64_t k, const float* b, uint64_t m, float* out) {
    memset(out, 0, n * m * 4);
    for (uint64_t i = 0; i < n; ++i) {
        float* o = out + i * m;
        for (uint64_t t = 0; t < k; ++t) {
            const float aik = a[i * k + t];
            const float* br = b + t * m;
            for (uint64_t j = 0; j < m; ++j) o[j] += aik * br[j];
        }
        for (uint64_t j = 0; j < m; ++j) o[j] += 0.0f;
    }
}

/* dense_matrix.hpp:57-76 gemm_at_b: out[i][j] = sum_k a[k][i]*b[k][j], k ascending; + 0 */
void orc_gemm_at_b_f32(const float* a, uint64_t n, uint64_t r, const float* b, uint64_t c, float* out) {
    memset(out, 0, r * c * 4);
    for (uint64_t i = 0; i < r; ++i) {
        float* o = out + i * c;
        for (uint64_t t = 0; t < n; ++t) {
            const float aki = a[t * r + i];
            const float* br = b + t * c;
            for (uint64_t j = 0; j < c; ++j) o[j] += aki * br[j];
        }
        for (uint64_t j = 0; j < c; ++j) o[j] += 0.0f;
    }
}

/* dense_matrix.hpp:98-104 */
void orc_relu_f32(const float* x, uint64_t count, float* out) {
    for (uint64_t i = 0; i < count; ++i) out[i] = x[i] > 0.0f ? x[i] : 0.0f;
}

/* dense_matrix.hpp:116-135 row_softmax: std::max((a < b) ? b : a), expf, serial sum, divide */
void orc_row_softmax_f32(const float* x, uint64_t rows, uint64_t cols, float* out) {
    for (uint64_t i = 0; i < rows; ++i) {
        const float* in = x + i * cols;
        float* o = out + i * cols;
        float mx = in[0];
        for (uint64_t j = 1; j < cols; ++j) mx = (mx < in[j]) ? in[j] : mx;
        float sum = 0.0f;
        for (uint64_t j = 0; j < cols; ++j) {
            o[j] = expf(in[j] - mx);
            sum += o[j];
        }
        for (uint64_t j = 0; j < cols; ++j) o[j] /= sum;
    }
}

/* engine.hpp:146-156 top_grad_from_probs */
void orc_top_grad_f32(const float* probs, const float* ref, uint64_t n, uint64_t c, const uint32_t* vt,
                      uint64_t k, float* out) {
    memset(out, 0, n * c * 4);
    const float inv = 1.0f / (float)k;
    for (uint64_t t = 0; t < k; ++t) {
        const uint64_t v = vt[t];
        for (uint64_t j = 0; j < c; ++j) out[v * c + j] = (probs[v * c + j] - ref[v * c + j]) * inv;
    }
}

/* aggregate.hpp:127-170 aggregate_pull_filtered, Deterministic branch, and
 * its counters {edges, groups, edges_skipped, groups_skipped} (groups of a
 * destination = ceil(deg / gs), grouping.cpp:7-27) */
void orc_aggregate_pull_filtered_f32(uint32_t D, const uint64_t* offsets, const uint32_t* nbrs,
                                     const double* w, const float* in, uint64_t dim,
                                     const uint8_t* dest_active, const uint8_t* src_active, uint32_t gs,
                                     float* out, uint64_t* counters) {
    uint64_t edges = 0, groups = 0, eskip = 0, gskip = 0;
    for (uint32_t v = 0; v < D; ++v) {
        const uint64_t deg = offsets[v + 1] - offsets[v];
        const uint64_t g = (deg + gs - 1) / gs;
        if (!dest_active[v]) {
            gskip += g;
            eskip += deg;
            continue;
        }
        groups += g;
        float* o = out + (uint64_t)v * dim;
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const uint32_t u = nbrs[e];
            if (!src_active[u]) {
                ++eskip;
                continue;
            }
            ++edges;
            const float we = (float)w[e];
            const float* x = in + (uint64_t)u * dim;
            for (uint64_t j = 0; j < dim; ++j) o[j] += we * x[j];
        }
        for (uint64_t j = 0; j < dim; ++j) o[j] += 0.0f;
    }
    if (counters) {
        counters[0] = edges;
        counters[1] = groups;
        counters[2] = eskip;
        counters[3] = gskip;
    }
}
