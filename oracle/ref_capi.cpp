// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference implementation
// (/root/reference/proj/core). Compiled by oracle/Makefile from the
// reference's own sources into oracle/_ref/libpathgcn_ref.so, it is used
//   * by tests/ to pin the C restatement (oracle/pathgcn_oracle.c) and to
//     generate the golden fixtures under tests/golden/;
//   * by bench.py's reference arm / cpu_baseline leg to time the reference's
//     own CPU backward-aggregation stage (engine.hpp:331-338).
// Every entry point forwards to the reference function named in its comment;
// only handle plumbing and the bounded-sample sub-path builder are ours.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "pathgcn/train.hpp"
#include "pathgcn/rmat.hpp"

using namespace pathgcn;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return 2;
    if (dynamic_cast<const IoError*>(&e)) return 3;
    if (dynamic_cast<const NumericError*>(&e)) return 4;
    return 1;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

struct RefGraph { CsrGraph g; };
struct RefFront { FrontierSets f; };
struct RefPath { ExecutionPath p; };
struct RefGroups { GroupedCsr gr; };

TrainingSet make_vt(const uint32_t* vt, uint64_t k) {
    TrainingSet t;
    t.vertices.assign(vt, vt + k);
    return t;
}

}  // namespace

extern "C" {

int ref_last_error(char* buf, uint64_t n) {
    if (n == 0) return static_cast<int>(g_err.size());
    std::snprintf(buf, n, "%s", g_err.c_str());
    return static_cast<int>(g_err.size());
}

int ref_max_threads() { return resolve_workers(0); }

void ref_free_graph(void* h) { delete static_cast<RefGraph*>(h); }
void ref_free_front(void* h) { delete static_cast<RefFront*>(h); }
void ref_free_path(void* h) { delete static_cast<RefPath*>(h); }
void ref_free_groups(void* h) { delete static_cast<RefGroups*>(h); }

// rmat.cpp:10-44
uint32_t ref_gen_rmat(uint32_t n, uint64_t m, double a, double b, double c, double d,
                      uint64_t seed, uint32_t* pairs_out) {
    uint32_t n_pad = 0;
    guard([&] {
        RmatParams p;
        p.n = n; p.m = m; p.a = a; p.b = b; p.c = c; p.d = d; p.seed = seed;
        EdgeList el = gen_rmat(p);
        for (uint64_t i = 0; i < el.pairs.size(); ++i) {
            pairs_out[2 * i] = el.pairs[i].first;
            pairs_out[2 * i + 1] = el.pairs[i].second;
        }
        n_pad = *el.n_hint;
    });
    return n_pad;
}

// csr_graph.cpp:33-63 + :65-77 (graph load). n_hint < 0: no hint.
int ref_graph_build(int64_t n_hint, const uint32_t* pairs, uint64_t npairs, int weight_mode,
                    void** out) {
    return guard([&] {
        EdgeList el;
        if (n_hint >= 0) el.n_hint = static_cast<VertexId>(n_hint);
        el.pairs.resize(npairs);
        for (uint64_t i = 0; i < npairs; ++i) el.pairs[i] = {pairs[2 * i], pairs[2 * i + 1]};
        auto* h = new RefGraph{build_undirected_csr(el)};
        assign_edge_weights(h->g, weight_mode ? WeightMode::SymNorm : WeightMode::Unit);
        *out = h;
    });
}

// edge_list.cpp:34-62 through a file path (load_edge_list_file)
int ref_graph_load_file(const char* path, int weight_mode, void** out) {
    return guard([&] {
        EdgeList el = load_edge_list_file(path);
        auto* h = new RefGraph{build_undirected_csr(el)};
        assign_edge_weights(h->g, weight_mode ? WeightMode::SymNorm : WeightMode::Unit);
        *out = h;
    });
}

int ref_graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                       const double* w, void** out) {
    return guard([&] {
        auto* h = new RefGraph;
        h->g.n = n;
        h->g.offsets.assign(offsets, offsets + n + 1);
        const uint64_t m = offsets[n];
        h->g.neighbors.assign(nbrs, nbrs + m);
        h->g.weights.assign(w, w + m);
        *out = h;
    });
}

void ref_graph_info(void* hg, uint32_t* n, uint64_t* m, uint32_t* maxdeg, uint64_t* fp) {
    const CsrGraph& g = static_cast<RefGraph*>(hg)->g;
    *n = g.n;
    *m = g.m();
    *maxdeg = g.max_degree();
    *fp = g.fingerprint();  // csr_graph.cpp:19-31
}

void ref_graph_export(void* hg, uint64_t* offsets, uint32_t* nbrs, double* w) {
    const CsrGraph& g = static_cast<RefGraph*>(hg)->g;
    std::memcpy(offsets, g.offsets.data(), g.offsets.size() * 8);
    std::memcpy(nbrs, g.neighbors.data(), g.neighbors.size() * 4);
    std::memcpy(w, g.weights.data(), g.weights.size() * 8);
}

// training_set.cpp:28-49
uint64_t ref_training_set_size(uint32_t n, double ratio) {
    return std::max<uint64_t>(1, static_cast<uint64_t>(std::llround(ratio * double(n))));
}

int ref_sample_training_set(uint32_t n, double ratio, uint64_t seed, uint32_t* out) {
    return guard([&] {
        TrainingSet vt = sample_training_set(n, ratio, seed);
        std::memcpy(out, vt.vertices.data(), vt.vertices.size() * 4);
    });
}

// training_set.cpp:15-26, execution_path.cpp:17-22
uint64_t ref_training_fingerprint(const uint32_t* vt, uint64_t k) {
    return make_vt(vt, k).fingerprint();
}

uint64_t ref_path_fingerprint(void* hg, const uint32_t* vt, uint64_t k, uint64_t L) {
    return path_fingerprint(static_cast<RefGraph*>(hg)->g, make_vt(vt, k), L);
}

// frontier.cpp:7-26
int ref_frontiers(void* hg, const uint32_t* vt, uint64_t k, uint64_t L, void** out) {
    return guard([&] {
        *out = new RefFront{compute_frontiers(static_cast<RefGraph*>(hg)->g, make_vt(vt, k), L)};
    });
}

uint64_t ref_frontier_size(void* hf, uint64_t level) {
    return static_cast<RefFront*>(hf)->f.levels.at(level).size();
}

void ref_frontier_export(void* hf, uint64_t level, uint32_t* out) {
    const auto& lv = static_cast<RefFront*>(hf)->f.levels.at(level);
    std::memcpy(out, lv.data(), lv.size() * 4);
}

// execution_path.cpp:24-88
int ref_path(void* hg, void* hf, uint64_t layer, void** out) {
    return guard([&] {
        *out = new RefPath{extract_execution_path(static_cast<RefGraph*>(hg)->g,
                                                  static_cast<RefFront*>(hf)->f, layer)};
    });
}

void ref_path_info(void* hp, uint32_t* D, uint32_t* S, uint64_t* E) {
    const ExecutionPath& p = static_cast<RefPath*>(hp)->p;
    *D = p.dest_count();
    *S = p.src_count();
    *E = p.edge_count();
}

void ref_path_export(void* hp, uint32_t* dest, uint32_t* src, uint32_t* srcpos,
                     uint64_t* offsets, uint32_t* nbrs, double* w) {
    const ExecutionPath& p = static_cast<RefPath*>(hp)->p;
    std::memcpy(dest, p.dest_local_to_global.data(), p.dest_local_to_global.size() * 4);
    std::memcpy(src, p.src_local_to_global.data(), p.src_local_to_global.size() * 4);
    std::memcpy(srcpos, p.src_pos_in_parent.data(), p.src_pos_in_parent.size() * 4);
    std::memcpy(offsets, p.offsets.data(), p.offsets.size() * 8);
    std::memcpy(nbrs, p.neighbors.data(), p.neighbors.size() * 4);
    std::memcpy(w, p.weights.data(), p.weights.size() * 8);
}

// An ExecutionPath from arrays (e.g. exported by the device path, which the
// parity tests prove bit-identical to extract_execution_path's output).
int ref_path_from_arrays(uint64_t layer, uint32_t D, uint32_t S, const uint32_t* dest,
                         const uint32_t* src, const uint32_t* srcpos, const uint64_t* offsets,
                         const uint32_t* nbrs, const double* w, void** out) {
    return guard([&] {
        auto* h = new RefPath;
        ExecutionPath& p = h->p;
        p.layer = layer;
        p.dest_local_to_global.assign(dest, dest + D);
        p.src_local_to_global.assign(src, src + S);
        p.src_pos_in_parent.assign(srcpos, srcpos + S);
        p.offsets.assign(offsets, offsets + D + 1);
        const uint64_t E = offsets[D];
        p.neighbors.assign(nbrs, nbrs + E);
        p.weights.assign(w, w + E);
        *out = h;
    });
}

// Bounded-sample sub-path for the CPU baseline: keeps every `stride`-th
// destination (all of its edges) and re-compacts the referenced sources the
// same way extract_execution_path does, so the sample is itself a valid
// execution path whose gather and aggregation shrink together.
int ref_path_sample(void* hp, uint32_t stride, void** out) {
    return guard([&] {
        const ExecutionPath& p = static_cast<RefPath*>(hp)->p;
        auto* h = new RefPath;
        ExecutionPath& q = h->p;
        q.layer = p.layer;
        q.fingerprint = p.fingerprint;
        q.offsets.push_back(0);
        std::vector<VertexId> gsrc;
        for (VertexId d = 0; d < p.dest_count(); d += stride) {
            q.dest_local_to_global.push_back(p.dest_local_to_global[d]);
            for (EdgeIndex e = p.offsets[d]; e < p.offsets[d + 1]; ++e) {
                gsrc.push_back(p.neighbors[e]);
                q.weights.push_back(p.weights[e]);
            }
            q.offsets.push_back(gsrc.size());
        }
        std::vector<VertexId> used = gsrc;
        std::sort(used.begin(), used.end());
        used.erase(std::unique(used.begin(), used.end()), used.end());
        q.neighbors.resize(gsrc.size());
        for (std::size_t e = 0; e < gsrc.size(); ++e)
            q.neighbors[e] = static_cast<VertexId>(
                std::lower_bound(used.begin(), used.end(), gsrc[e]) - used.begin());
        for (VertexId s : used) {
            q.src_local_to_global.push_back(p.src_local_to_global[s]);
            q.src_pos_in_parent.push_back(p.src_pos_in_parent[s]);
        }
        *out = h;
    });
}

// grouping.cpp:7-27 over a path view (kind=1) or the graph view (kind=0)
int ref_group(void* owner, int kind, uint32_t gs, void** out) {
    return guard([&] {
        CsrView v = kind ? static_cast<RefPath*>(owner)->p.view()
                         : static_cast<RefGraph*>(owner)->g.view();
        *out = new RefGroups{group_neighbors(v, gs)};
    });
}

uint64_t ref_group_count(void* hgr) { return static_cast<RefGroups*>(hgr)->gr.group_count(); }

void ref_group_export(void* hgr, uint32_t* dest, uint64_t* begin, uint64_t* end,
                      uint64_t* dest_groups) {
    const GroupedCsr& gr = static_cast<RefGroups*>(hgr)->gr;
    for (std::size_t i = 0; i < gr.groups.size(); ++i) {
        dest[i] = gr.groups[i].dest;
        begin[i] = gr.groups[i].edge_begin;
        end[i] = gr.groups[i].edge_end;
    }
    std::memcpy(dest_groups, gr.dest_groups.data(), gr.dest_groups.size() * 8);
}

// gs_model.cpp:64-74 (beta = NULL: default_gs_model)
uint32_t ref_regression_gs(uint32_t n_vertices, uint64_t n_edges, double avg_degree,
                           const double* beta) {
    GraphStats s;
    s.n_vertices = n_vertices;
    s.n_undirected_edges = n_edges;
    s.avg_degree = avg_degree;
    GsModel m = default_gs_model();
    if (beta) m = {beta[0], beta[1], beta[2], beta[3]};
    return regression_gs(s, m);
}

// train.hpp:16-24 path_stats feeding regression_gs
uint32_t ref_path_regression_gs(void* hp) {
    return regression_gs(path_stats(static_cast<RefPath*>(hp)->p), default_gs_model());
}

// group_cost.cpp:30-34
uint64_t ref_default_candidates(uint32_t max_degree, uint32_t* out) {
    auto c = default_gs_candidates(max_degree);
    std::memcpy(out, c.data(), c.size() * 4);
    return c.size();
}

// group_cost.cpp:9-24
double ref_grouping_cost(void* hgr, uint64_t dim, int workers, double lambda) {
    double r = -1.0;
    guard([&] {
        r = grouping_cost(static_cast<RefGroups*>(hgr)->gr, dim, GroupCostModel{workers, lambda});
    });
    return r;
}

// group_cost.cpp:36-53 with cost_model_evaluator (:26-28)
int ref_oracle_gs_cost(void* owner, int kind, const uint32_t* cands, uint64_t ncand,
                       uint64_t dim, int workers, double lambda, uint32_t* best, double* table) {
    return guard([&] {
        CsrView v = kind ? static_cast<RefPath*>(owner)->p.view()
                         : static_cast<RefGraph*>(owner)->g.view();
        std::vector<VertexId> c(cands, cands + ncand);
        auto sweep = oracle_gs(v, c, cost_model_evaluator(dim, GroupCostModel{workers, lambda}));
        *best = sweep.best_gs;
        for (std::size_t i = 0; i < sweep.table.size(); ++i) table[i] = sweep.table[i].cost;
    });
}

// aggregate.hpp:56-122. `out` is read (accumulate semantics) and written.
// counters[3] = {edges_traversed, groups_executed, atomic_commits}.
int ref_aggregate_pull_f32(void* hgr, const float* in, uint64_t in_rows, uint64_t dim,
                           float* out, int fast, int workers, uint64_t* counters) {
    return guard([&] {
        const GroupedCsr& gr = static_cast<RefGroups*>(hgr)->gr;
        DenseMatrix<float> x(in_rows, dim), y(gr.base.n, dim);
        std::memcpy(x.data.data(), in, in_rows * dim * 4);
        std::memcpy(y.data.data(), out, std::size_t(gr.base.n) * dim * 4);
        StageCounters c;
        aggregate_pull(gr, x, y, fast ? CommitMode::Fast : CommitMode::Deterministic, workers, &c);
        std::memcpy(out, y.data.data(), y.data.size() * 4);
        if (counters) {
            counters[0] = c.edges_traversed;
            counters[1] = c.groups_executed;
            counters[2] = c.atomic_commits;
        }
    });
}

int ref_aggregate_pull_f64(void* hgr, const double* in, uint64_t in_rows, uint64_t dim,
                           double* out, int fast, int workers, uint64_t* counters) {
    return guard([&] {
        const GroupedCsr& gr = static_cast<RefGroups*>(hgr)->gr;
        DenseMatrix<double> x(in_rows, dim), y(gr.base.n, dim);
        std::memcpy(x.data.data(), in, in_rows * dim * 8);
        std::memcpy(y.data.data(), out, std::size_t(gr.base.n) * dim * 8);
        StageCounters c;
        aggregate_pull(gr, x, y, fast ? CommitMode::Fast : CommitMode::Deterministic, workers, &c);
        std::memcpy(out, y.data.data(), y.data.size() * 8);
        if (counters) {
            counters[0] = c.edges_traversed;
            counters[1] = c.groups_executed;
            counters[2] = c.atomic_commits;
        }
    });
}

// dense_matrix.hpp:78-95
int ref_gemm_a_bt_f32(const float* a, uint64_t n, uint64_t k, const float* b, uint64_t m,
                      float* out) {
    return guard([&] {
        DenseMatrix<float> A(n, k), B(m, k);
        std::memcpy(A.data.data(), a, n * k * 4);
        std::memcpy(B.data.data(), b, m * k * 4);
        DenseMatrix<float> C = gemm_a_bt(A, B);
        std::memcpy(out, C.data.data(), n * m * 4);
    });
}

int ref_gemm_a_bt_f64(const double* a, uint64_t n, uint64_t k, const double* b, uint64_t m,
                      double* out) {
    return guard([&] {
        DenseMatrix<double> A(n, k), B(m, k);
        std::memcpy(A.data.data(), a, n * k * 8);
        std::memcpy(B.data.data(), b, m * k * 8);
        DenseMatrix<double> C = gemm_a_bt(A, B);
        std::memcpy(out, C.data.data(), n * m * 8);
    });
}

// The reference's timed backward-aggregation stage, engine.hpp:331-338:
//   y_used = gather_rows(y_grad, path.src_pos_in_parent)
//   aggregate_pull(path_groups[i], y_used, x_grad, commit, workers)
// y_grad rows follow the parent frontier (|levels[i]| rows). The inputs are
// staged into DenseMatrix objects outside the timer, like the reference
// (x_grad is constructed before `StageTimer ta`). Returns the stage seconds.
int ref_backward_aggregation_f32(void* hp, void* hgr, const float* y_grad, uint64_t rows,
                                 uint64_t dim, float* x_grad, int fast, int workers,
                                 double* seconds) {
    return guard([&] {
        const ExecutionPath& path = static_cast<RefPath*>(hp)->p;
        const GroupedCsr& gr = static_cast<RefGroups*>(hgr)->gr;
        DenseMatrix<float> yg(rows, dim);
        std::memcpy(yg.data.data(), y_grad, rows * dim * 4);
        DenseMatrix<float> xg(path.dest_count(), dim);
        StageTimer ta;
        DenseMatrix<float> y_used = detail::gather_rows(yg, path.src_pos_in_parent);
        aggregate_pull(gr, y_used, xg, fast ? CommitMode::Fast : CommitMode::Deterministic,
                       workers, nullptr);
        *seconds = ta.stop();
        if (x_grad) std::memcpy(x_grad, xg.data.data(), xg.data.size() * 4);
    });
}

// Real gradient chain, engine.hpp:70-155 + the Local branch of backward_epp
// (:316-346), replicated step by step so the per-layer operands can be
// captured for the device chain parity test. Sizes follow the frontiers:
//   top_g      |V_t| x c           (gather_rows(top_grad, levels[0]))
//   w[l]       in_dim_l x dims[l]  (params.weights[l], l = 0..L-1)
//   pre_c[i]   |levels[i+1]| x dims[l-1]   for i < L-1 (l = L-1-i > 0)
//   y_grad[i]  |levels[i]| x in_dim_l      (gemm_a_bt(g, W^(l)))
//   x_grad[i]  |levels[i+1]| x in_dim_l    (aggregate_pull output)
// Uses group size `path_gs` for every path and `graph_gs` for forward.
int ref_epp_chain_f32(void* hg, const uint32_t* vt, uint64_t k, uint64_t L, uint64_t f,
                      uint64_t dim0, uint64_t classes, uint64_t seed, uint32_t graph_gs,
                      uint32_t path_gs, float* top_g, float** w, float** pre_c, float** y_grad,
                      float** x_grad) {
    return guard([&] {
        const CsrGraph& g = static_cast<RefGraph*>(hg)->g;
        TrainingSet ts = make_vt(vt, k);
        std::vector<std::size_t> dims(L, dim0);
        dims.back() = classes;
        WorkCounters counters;
        const GroupedCsr grouped = group_neighbors(g.view(), graph_gs);
        ModelParams<float> params = init_params<float>(f, dims, seed);
        const DenseMatrix<float> x0 = random_features<float>(g.n, f, seed);
        const DenseMatrix<float> ref = random_reference<float>(g.n, classes, ts, seed);
        EpochArtifacts<float> arts =
            forward(grouped, x0, params, CommitMode::Deterministic, 0, counters);
        const DenseMatrix<float> top = top_grad_from_probs(arts.x[L], ref, ts);
        const FrontierSets fr = compute_frontiers(g, ts, L);
        auto paths = prepare_all_paths(g, fr);
        std::vector<GroupedCsr> pgroups;
        for (auto& p : paths) pgroups.push_back(group_neighbors(p.view(), path_gs));
        for (std::size_t l = 0; l < L; ++l)
            std::memcpy(w[l], params.weights[l].data.data(), params.weights[l].data.size() * 4);

        DenseMatrix<float> gm = detail::gather_rows(top, fr.levels[0]);
        std::memcpy(top_g, gm.data.data(), gm.data.size() * 4);
        for (std::size_t i = 0; i < L; ++i) {
            const std::size_t l = L - 1 - i;
            DenseMatrix<float> yg = gemm_a_bt(gm, params.weights[l]);
            std::memcpy(y_grad[i], yg.data.data(), yg.data.size() * 4);
            DenseMatrix<float> xg(paths[i].dest_count(), yg.cols);
            DenseMatrix<float> y_used = detail::gather_rows(yg, paths[i].src_pos_in_parent);
            aggregate_pull(pgroups[i], y_used, xg, CommitMode::Deterministic, 0, nullptr);
            std::memcpy(x_grad[i], xg.data.data(), xg.data.size() * 4);
            if (l > 0) {
                DenseMatrix<float> pc = detail::gather_rows(arts.pre_act[l - 1], fr.levels[L - l]);
                std::memcpy(pre_c[i], pc.data.data(), pc.data.size() * 4);
                gm = relu_backward(xg, pc);
            }
        }
    });
}

// The reference's own chain on caller-given inputs: forward (engine.hpp:
// 114-140) over group_neighbors(g, graph_gs), top_grad_from_probs
// (:146-156), then one backward variant, mode 0 = backward_all_active
// (:177-214), 1 = backward_ifelse (:218-257), 2 = backward_epp Local,
// 3 = backward_epp Global (:267-349; paths grouped with path_gs, stamped
// with path_fingerprint). Outputs: y[l] n x in_dim_l, pre[l] n x dims[l],
// x[l] = X^(l+1) n x dims[l], top n x dims[L-1], w_grads[l], x_grads
// (mode 0 only, nullable: n x in_dim per layer, layer L-1 first),
// edges[L] = backward_edges_per_layer.
int ref_chain_f32(void* hg, const uint32_t* vt, uint64_t k, uint64_t L, uint64_t f, const uint64_t* dims,
                  const float* x0, const float* const* w, const float* rmat, uint32_t graph_gs, uint32_t path_gs,
                  int mode, float** y_out, float** pre_out, float** x_out, float* top_out, float** wg_out,
                  float** xg_out, uint64_t* edges) {
    return guard([&] {
        const CsrGraph& g = static_cast<RefGraph*>(hg)->g;
        const TrainingSet ts = make_vt(vt, k);
        const std::size_t c = dims[L - 1];
        ModelParams<float> params;
        std::size_t in_dim = f;
        for (uint64_t l = 0; l < L; ++l) {
            DenseMatrix<float> wl(in_dim, dims[l]);
            std::memcpy(wl.data.data(), w[l], wl.data.size() * 4);
            params.weights.push_back(std::move(wl));
            in_dim = dims[l];
        }
        DenseMatrix<float> x(g.n, f);
        std::memcpy(x.data.data(), x0, x.data.size() * 4);
        DenseMatrix<float> r(g.n, c);
        std::memcpy(r.data.data(), rmat, r.data.size() * 4);
        WorkCounters counters;
        const GroupedCsr grouped = group_neighbors(g.view(), graph_gs);
        EpochArtifacts<float> arts = forward(grouped, x, params, CommitMode::Deterministic, 0, counters);
        const DenseMatrix<float> top = top_grad_from_probs(arts.x[L], r, ts);
        for (uint64_t l = 0; l < L; ++l) {
            std::memcpy(y_out[l], arts.y[l].data.data(), arts.y[l].data.size() * 4);
            std::memcpy(pre_out[l], arts.pre_act[l].data.data(), arts.pre_act[l].data.size() * 4);
            std::memcpy(x_out[l], arts.x[l + 1].data.data(), arts.x[l + 1].data.size() * 4);
        }
        std::memcpy(top_out, top.data.data(), top.data.size() * 4);
        std::vector<DenseMatrix<float>> wg;
        if (mode == 0) {
            std::vector<DenseMatrix<float>> xg;
            wg = backward_all_active(grouped, arts, top, params, CommitMode::Deterministic, 0, counters, &xg);
            if (xg_out)
                for (uint64_t i = 0; i < L; ++i) std::memcpy(xg_out[i], xg[i].data.data(), xg[i].data.size() * 4);
        } else {
            const FrontierSets fr = compute_frontiers(g, ts, L);
            if (mode == 1) {
                wg = backward_ifelse(grouped, fr, arts, top, params, CommitMode::Deterministic, 0, counters);
            } else {
                auto paths = prepare_all_paths(g, fr);
                const uint64_t stamp = path_fingerprint(g, ts, L);
                std::vector<GroupedCsr> pg;
                for (auto& p : paths) {
                    p.fingerprint = stamp;
                    pg.push_back(group_neighbors(p.view(), path_gs));
                }
                wg = backward_epp(paths, pg, fr, arts, top, params,
                                  mode == 2 ? GatherMode::Local : GatherMode::Global, CommitMode::Deterministic, 0,
                                  counters, stamp);
            }
        }
        for (uint64_t l = 0; l < L; ++l) std::memcpy(wg_out[l], wg[l].data.data(), wg[l].data.size() * 4);
        for (uint64_t i = 0; i < L; ++i) edges[i] = counters.backward_edges_per_layer[i];
    });
}

}  // extern "C"
