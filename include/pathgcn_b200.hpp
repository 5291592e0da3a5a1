// pathgcn_b200.hpp — header-only C++20 host side over the C ABI
// (pathgcn_b200.h), re-exposing the reference's operator API for the
// backward-aggregation path (namespace pathgcn, proj/core/include/pathgcn):
//
//   reference                                   here (namespace pathgcn::b200)
//   build_undirected_csr + assign_edge_weights  build_undirected_csr(EdgeList, WeightMode)
//     (csr_graph.hpp:48-51)                     DeviceGraph::from_csr(CsrView-like arrays)
//   compute_frontiers (frontier.hpp:20)         compute_frontiers(g, vt, L) -> DeviceFrontiers
//   extract_execution_path (execution_path.hpp:37-38), prepare_all_paths (:41)
//   path_fingerprint (:35)                      path_fingerprint(g, vt, L)
//   group_neighbors (grouping.hpp:30)           group_neighbors(path, gs) -> DeviceGroups
//   regression_gs (gs_model.hpp:24)             regression_gs(stats) / regression_gs(path)
//   oracle_gs + cost_model_evaluator            oracle_gs_cost(path, dim, {workers, lambda})
//     (group_cost.hpp:19-43)
//   aggregate_pull<float> (aggregate.hpp:56-59) aggregate_pull(groups, in, out, mode, counters)
//   engine.hpp:331-338 stage                    backward_aggregation(groups, y_grad, x_grad)
//   load_edge_list_file / load_training_set_file (edge_list.cpp, training_set.cpp)
//   measured_evaluator + oracle_gs (train.hpp:35-54) oracle_gs_measured(path, dim)
//   forward / backward_epp / backward_all_active / backward_ifelse (engine.hpp:114-349)
//                                               same names over DeviceMatrix artefacts
//
// Errors are thrown as exceptions mirroring error.hpp:10-47 (ConfigError,
// ShapeError, StalenessError, IoError, NumericError) plus DeviceError for
// CUDA failures; calls are synchronous for host buffers, like the
// reference. All compute runs on the GPU (libpathgcn_b200.so, sm_100a).
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pathgcn_b200.h"

namespace pathgcn::b200 {

using VertexId = std::uint32_t;
using EdgeIndex = std::uint64_t;

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct ShapeError : ConfigError {
    using ConfigError::ConfigError;
};
struct StalenessError : ConfigError {
    using ConfigError::ConfigError;
};
struct ParseError : ConfigError {                 // error.hpp:18-22
    ParseError(const std::string& msg, std::size_t line) : ConfigError(msg), line_number(line) {}
    std::size_t line_number;
};
struct IoError : Error {
    using Error::Error;
};
struct NumericError : Error {
    using Error::Error;
};
struct DeviceError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == PG_OK) return;
    std::string msg(512, '\0');
    pg_last_error(msg.data(), msg.size());
    msg.resize(msg.find('\0'));
    std::uint64_t line = 0;
    switch (pg_last_error_kind(&line)) {  // the exact error.hpp type, not a guess from the text
        case PG_KIND_SHAPE: throw ShapeError(msg);
        case PG_KIND_STALENESS: throw StalenessError(msg);
        case PG_KIND_PARSE: throw ParseError(msg, line);
        case PG_KIND_CONFIG: throw ConfigError(msg);
        case PG_KIND_IO: throw IoError(msg);
        case PG_KIND_NUMERIC: throw NumericError(msg);
        case PG_KIND_DEVICE: throw DeviceError(msg);
        default: break;
    }
    switch (rc) {
        case PG_ERR_CONFIG: throw ConfigError(msg);
        case PG_ERR_IO: throw IoError(msg);
        case PG_ERR_NUMERIC: throw NumericError(msg);
        case PG_ERR_DEVICE: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

enum class WeightMode { Unit, SymNorm };          // csr_graph.hpp:13
// aggregate.hpp:21. Fast runs the atomic-free kernel (bit-equal to
// Deterministic); Grouped is Fast on the group-partitioned kernel (a warp per
// neighbour group, atomics across a destination's groups: tolerance-level).
enum class CommitMode { Deterministic, Fast, Grouped };
enum class GatherMode { Local, Global };          // run_config.hpp:19

inline unsigned commit_flags(CommitMode m) {
    return m == CommitMode::Fast ? PG_AGG_FAST : m == CommitMode::Grouped ? (PG_AGG_FAST | PG_AGG_GROUPED) : 0u;
}

struct EdgeList {                                 // edge_list.hpp:14-18
    std::vector<std::pair<VertexId, VertexId>> pairs;
    std::optional<VertexId> n_hint;
    std::uint64_t self_loops_dropped = 0;
};

// edge_list.cpp:34-68 (ParseError carries the line number, IoError)
inline EdgeList load_edge_list_file(const std::string& path) {
    pg_edge_list h = nullptr;
    check(pg_edge_list_load(path.c_str(), &h));
    std::uint64_t n = 0, sl = 0;
    std::vector<VertexId> flat;
    try {
        check(pg_edge_list_info(h, &n, &sl));
        flat.resize(2 * n);
        check(pg_edge_list_export(h, flat.data()));
    } catch (...) {
        pg_edge_list_destroy(h);
        throw;
    }
    pg_edge_list_destroy(h);
    EdgeList el;
    el.self_loops_dropped = sl;
    el.pairs.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i) el.pairs.emplace_back(flat[2 * i], flat[2 * i + 1]);
    return el;
}

inline void write_edge_list_file(const std::string& path, const EdgeList& el) {
    std::vector<VertexId> flat;
    flat.reserve(el.pairs.size() * 2);
    for (const auto& [u, v] : el.pairs) {
        flat.push_back(u);
        flat.push_back(v);
    }
    check(pg_edge_list_write(path.c_str(), flat.data(), el.pairs.size()));
}

// training_set.cpp:51-79: sorted unique ids
inline std::vector<VertexId> load_training_set_file(const std::string& path, VertexId n) {
    std::uint64_t k = 0;
    check(pg_training_set_load(path.c_str(), n, nullptr, 0, &k));
    std::vector<VertexId> out(k);
    check(pg_training_set_load(path.c_str(), n, out.data(), out.size(), &k));
    return out;
}

inline void write_training_set_file(const std::string& path, std::span<const VertexId> vt) {
    check(pg_training_set_write(path.c_str(), vt.data(), vt.size()));
}

struct StageCounters {                            // aggregate.hpp:23-39 (work part)
    std::uint64_t edges_traversed = 0;
    std::uint64_t groups_executed = 0;
    std::uint64_t atomic_commits = 0;
};

struct GraphStats {                               // csr_graph.hpp:40-44
    VertexId n_vertices = 0;
    EdgeIndex n_undirected_edges = 0;
    double avg_degree = 0.0;
};

template <typename T>
struct DenseMatrix {                              // dense_matrix.hpp:14-30 (row-major, ld = cols)
    std::size_t rows = 0, cols = 0;
    std::vector<T> data;
    DenseMatrix() = default;
    DenseMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, T(0)) {}
};
using MatrixF = DenseMatrix<float>;
using MatrixD = DenseMatrix<double>;               // Precision::F64, the reference's default (run_config.hpp:53)

// Host copy of an ExecutionPath (execution_path.hpp:16-33 field names).
struct ExecutionPathHost {
    std::size_t layer = 0;
    std::vector<VertexId> dest_local_to_global, src_local_to_global, src_pos_in_parent;
    std::vector<EdgeIndex> offsets;
    std::vector<VertexId> neighbors;
    std::vector<double> weights;
    std::uint64_t fingerprint = 0;
};

template <typename H, int (*Destroy)(H)>
struct Handle {
    H h = nullptr;
    Handle() = default;
    explicit Handle(H x) : h(x) {}
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;
    Handle(Handle&& o) noexcept : h(std::exchange(o.h, nullptr)) {}
    Handle& operator=(Handle&& o) noexcept {
        if (this != &o) {
            reset();
            h = std::exchange(o.h, nullptr);
        }
        return *this;
    }
    ~Handle() { reset(); }
    void reset() {
        if (h) Destroy(h);
        h = nullptr;
    }
};

class DeviceGraph {                               // CsrGraph (csr_graph.hpp:19-38)
public:
    static DeviceGraph from_csr(VertexId n, std::span<const EdgeIndex> offsets, std::span<const VertexId> neighbors,
                                std::span<const double> weights, int device = 0, bool validate = true) {
        pg_graph g = nullptr;
        check(pg_graph_create(device, n, offsets.data(), neighbors.data(), weights.data(), validate, &g));
        return DeviceGraph(g);
    }
    VertexId n() const { return info().n; }
    EdgeIndex m() const { return info().m; }
    VertexId max_degree() const { return info().maxdeg; }
    std::uint64_t fingerprint() const {
        std::uint64_t fp = 0;
        check(pg_graph_info(h_.h, nullptr, nullptr, nullptr, &fp));
        return fp;
    }
    void assign_edge_weights(WeightMode mode) {
        check(pg_graph_assign_weights(h_.h, mode == WeightMode::SymNorm ? PG_WEIGHTS_SYMNORM : PG_WEIGHTS_UNIT));
    }
    void to_host(std::vector<EdgeIndex>& offsets, std::vector<VertexId>& neighbors, std::vector<double>& weights) const {
        const auto i = info();
        offsets.resize(i.n + 1);
        neighbors.resize(i.m);
        weights.resize(i.m);
        check(pg_graph_export(h_.h, offsets.data(), neighbors.data(), weights.data()));
    }
    pg_graph raw() const { return h_.h; }
    explicit DeviceGraph(pg_graph g) : h_(g) {}

private:
    struct Info {
        VertexId n;
        EdgeIndex m;
        VertexId maxdeg;
    };
    Info info() const {
        Info i{};
        check(pg_graph_info(h_.h, &i.n, &i.m, &i.maxdeg, nullptr));
        return i;
    }
    Handle<pg_graph, pg_graph_destroy> h_;
};

// csr_graph.cpp:33-77 on the device
inline DeviceGraph build_undirected_csr(const EdgeList& el, WeightMode mode = WeightMode::Unit, int device = 0) {
    std::vector<VertexId> flat(el.pairs.size() * 2);
    for (std::size_t i = 0; i < el.pairs.size(); ++i) {
        flat[2 * i] = el.pairs[i].first;
        flat[2 * i + 1] = el.pairs[i].second;
    }
    pg_graph g = nullptr;
    check(pg_graph_build(device, el.n_hint ? static_cast<std::int64_t>(*el.n_hint) : -1, flat.data(),
                         el.pairs.size(), mode == WeightMode::SymNorm ? PG_WEIGHTS_SYMNORM : PG_WEIGHTS_UNIT, &g));
    return DeviceGraph(g);
}

// load_edge_list_file + build_undirected_csr + assign_edge_weights
inline DeviceGraph load_graph_file(const std::string& path, WeightMode mode = WeightMode::Unit, int device = 0) {
    pg_graph g = nullptr;
    check(pg_graph_load_file(device, path.c_str(), mode == WeightMode::SymNorm ? PG_WEIGHTS_SYMNORM : PG_WEIGHTS_UNIT,
                             &g));
    return DeviceGraph(g);
}

class DeviceFrontiers {                           // FrontierSets (frontier.hpp:14-18)
public:
    explicit DeviceFrontiers(pg_frontiers f, std::size_t L) : h_(f), L_(L) {}
    std::size_t depth() const { return L_; }
    std::vector<VertexId> level(std::size_t k) const {
        std::uint64_t sz = 0;
        check(pg_frontiers_size(h_.h, k, &sz));
        std::vector<VertexId> out(sz);
        check(pg_frontiers_export(h_.h, k, out.data()));
        return out;
    }
    std::vector<std::vector<VertexId>> levels() const {
        std::vector<std::vector<VertexId>> out;
        for (std::size_t k = 0; k <= L_; ++k) out.push_back(level(k));
        return out;
    }
    pg_frontiers raw() const { return h_.h; }

private:
    Handle<pg_frontiers, pg_frontiers_destroy> h_;
    std::size_t L_;
};

inline DeviceFrontiers compute_frontiers(const DeviceGraph& g, std::span<const VertexId> vt, std::size_t layers) {
    pg_frontiers f = nullptr;
    check(pg_frontiers_compute(g.raw(), vt.data(), vt.size(), layers, &f));
    return DeviceFrontiers(f, layers);
}

class DevicePath {                                // ExecutionPath (execution_path.hpp:16-33)
public:
    explicit DevicePath(pg_path p) : h_(p) {
        check(pg_path_info(p, &layer_, &D_, &S_, &E_, &P_, &maxdeg_));
    }
    std::size_t layer() const { return layer_; }
    VertexId dest_count() const { return D_; }
    VertexId src_count() const { return S_; }
    EdgeIndex edge_count() const { return E_; }
    VertexId parent_rows() const { return P_; }
    VertexId max_degree() const { return maxdeg_; }
    std::uint64_t fingerprint() const {
        std::uint64_t fp = 0;
        check(pg_path_get_fingerprint(h_.h, &fp));
        return fp;
    }
    void set_fingerprint(std::uint64_t fp) { check(pg_path_set_fingerprint(h_.h, fp)); }
    ExecutionPathHost to_host() const {
        ExecutionPathHost p;
        p.layer = layer_;
        p.dest_local_to_global.resize(D_);
        p.src_local_to_global.resize(S_);
        p.src_pos_in_parent.resize(S_);
        p.offsets.resize(D_ + 1);
        p.neighbors.resize(E_);
        p.weights.resize(E_);
        check(pg_path_export(h_.h, p.dest_local_to_global.data(), p.src_local_to_global.data(),
                             p.src_pos_in_parent.data(), p.offsets.data(), p.neighbors.data(), p.weights.data()));
        p.fingerprint = fingerprint();
        return p;
    }
    pg_path raw() const { return h_.h; }

private:
    Handle<pg_path, pg_path_destroy> h_;
    std::uint64_t layer_ = 0;
    VertexId D_ = 0, S_ = 0, P_ = 0, maxdeg_ = 0;
    EdgeIndex E_ = 0;
};

inline DevicePath extract_execution_path(const DeviceGraph& g, const DeviceFrontiers& f, std::size_t layer) {
    pg_path p = nullptr;
    check(pg_path_extract(g.raw(), f.raw(), layer, &p));
    return DevicePath(p);
}

// execution_path.cpp:90-96: SG_{L-1} first
inline std::vector<DevicePath> prepare_all_paths(const DeviceGraph& g, const DeviceFrontiers& f) {
    std::vector<DevicePath> out;
    for (std::size_t l = f.depth(); l-- > 0;) out.push_back(extract_execution_path(g, f, l));
    return out;
}

inline std::uint64_t path_fingerprint(const DeviceGraph& g, std::span<const VertexId> vt, std::size_t layers) {
    std::uint64_t fp = 0;
    check(pg_path_fingerprint(g.raw(), vt.data(), vt.size(), layers, &fp));
    return fp;
}

struct GsModel {                                  // gs_model.hpp:12-17 / default_gs_model
    double beta0 = 0.65538, beta1 = 1.67431e-5, beta2 = -2.24342e-6, beta3 = 0.63641;
};

inline VertexId regression_gs(const GraphStats& s, const GsModel& m = {}) {
    const double b[4] = {m.beta0, m.beta1, m.beta2, m.beta3};
    VertexId gs = 0;
    check(pg_gs_regression_stats(s.n_vertices, s.n_undirected_edges, s.avg_degree, b, &gs));
    return gs;
}

// regression_gs(path_stats(path)) (train.hpp:16-24)
inline VertexId regression_gs(const DevicePath& p, const GsModel& m = {}) {
    const double b[4] = {m.beta0, m.beta1, m.beta2, m.beta3};
    VertexId gs = 0;
    check(pg_gs_regression(p.raw(), b, &gs));
    return gs;
}

inline std::vector<VertexId> default_gs_candidates(VertexId max_degree) {
    std::vector<VertexId> out(40);
    std::uint64_t k = 0;
    check(pg_gs_default_candidates(max_degree, out.data(), &k));
    out.resize(k);
    return out;
}

struct GroupCostModel {                           // group_cost.hpp:14-17
    int worker_count = 1;
    double atomic_penalty = 0.25;
};
struct GsSweepEntry {
    VertexId gs;
    double cost;
};
struct GsSweepResult {                            // group_cost.hpp:26-29
    VertexId best_gs = 1;
    std::vector<GsSweepEntry> table;
};

// oracle_gs(csr, candidates, cost_model_evaluator(dim, model)) on device
inline GsSweepResult oracle_gs_cost(const DevicePath& p, std::size_t dim, const GroupCostModel& model,
                                    std::vector<VertexId> candidates = {}) {
    if (candidates.empty()) candidates = default_gs_candidates(p.max_degree());
    std::vector<double> table(candidates.size());
    GsSweepResult r;
    std::uint64_t n = 0;
    check(pg_gs_oracle_cost(p.raw(), dim, model.worker_count, model.atomic_penalty, candidates.data(),
                            candidates.size(), &r.best_gs, table.data(), &n));
    for (std::size_t i = 0; i < n; ++i) r.table.push_back({candidates[i], table[i]});
    return r;
}

// train.hpp:35-54 measured_evaluator + oracle_gs on the device: the grouped
// (Fast) aggregation of each candidate timed, median of `repeats` (seconds)
inline GsSweepResult oracle_gs_measured(const DevicePath& p, std::size_t dim, int repeats = 5,
                                        std::uint64_t seed = 42, std::vector<VertexId> candidates = {}) {
    if (candidates.empty()) candidates = default_gs_candidates(p.max_degree());
    std::vector<double> table(candidates.size());
    GsSweepResult r;
    std::uint64_t n = 0;
    check(pg_gs_oracle_measured(p.raw(), dim, repeats, seed, candidates.data(), candidates.size(), &r.best_gs,
                                table.data(), &n));
    for (std::size_t i = 0; i < n; ++i) r.table.push_back({candidates[i], table[i]});
    return r;
}

class DeviceGroups {                              // GroupedCsr (grouping.hpp:14-28)
public:
    explicit DeviceGroups(pg_groups g) : h_(g) { check(pg_groups_info(g, &gs_, &count_, &dests_)); }
    VertexId gs() const { return gs_; }
    std::size_t group_count() const { return count_; }
    VertexId dest_count() const { return dests_; }
    void to_host(std::vector<VertexId>& dest, std::vector<EdgeIndex>& begin, std::vector<EdgeIndex>& end,
                 std::vector<std::uint64_t>& dest_groups) const {
        dest.resize(count_);
        begin.resize(count_);
        end.resize(count_);
        dest_groups.resize(dests_ + 1);
        check(pg_groups_export(h_.h, dest.data(), begin.data(), end.data(), dest_groups.data()));
    }
    double grouping_cost(std::size_t dim, const GroupCostModel& m) const {
        double c = 0;
        check(pg_grouping_cost(h_.h, dim, m.worker_count, m.atomic_penalty, &c));
        return c;
    }
    pg_groups raw() const { return h_.h; }

private:
    Handle<pg_groups, pg_groups_destroy> h_;
    VertexId gs_ = 0, dests_ = 0;
    std::uint64_t count_ = 0;
};

inline DeviceGroups group_neighbors(const DevicePath& p, VertexId gs) {
    pg_groups g = nullptr;
    check(pg_group(p.raw(), gs, &g));
    return DeviceGroups(g);
}
inline DeviceGroups group_neighbors(const DeviceGraph& graph, VertexId gs) {
    pg_groups g = nullptr;
    check(pg_group_graph(graph.raw(), gs, &g));
    return DeviceGroups(g);
}

// aggregate.hpp:56-122 aggregate_pull<float>: output accumulates, like the
// reference (pass a zeroed output). `workers` is accepted for signature
// compatibility; the device schedule is worker independent.
inline void aggregate_pull(const DeviceGroups& grouped, const MatrixF& input, MatrixF& output,
                           CommitMode mode = CommitMode::Deterministic, int workers = 0,
                           StageCounters* counters = nullptr) {
    (void)workers;
    if (output.rows != grouped.dest_count()) throw ShapeError("aggregate_pull: output rows != dest count");
    if (output.cols != input.cols) throw ShapeError("aggregate_pull: input/output dims differ");
    std::uint64_t c[3] = {0, 0, 0};
    check(pg_aggregate_pull_host(grouped.raw(), input.data.data(), input.rows, input.cols, output.data.data(),
                                 commit_flags(mode == CommitMode::Grouped ? CommitMode::Fast : mode), c));
    if (counters) {
        counters->edges_traversed += c[0];
        counters->groups_executed += c[1];
        counters->atomic_commits += c[2];
    }
}

// engine.hpp:331-338: x_grad = aggregate_pull(groups, gather_rows(y_grad,
// src_pos_in_parent)); y_grad rows follow the parent frontier.
inline void backward_aggregation(const DeviceGroups& grouped, const MatrixF& y_grad, MatrixF& x_grad,
                                 CommitMode mode = CommitMode::Deterministic, StageCounters* counters = nullptr) {
    if (x_grad.rows != grouped.dest_count() || x_grad.cols != y_grad.cols)
        throw ShapeError("backward_aggregation: x_grad shape mismatch");
    std::uint64_t c[3] = {0, 0, 0};
    check(pg_backward_aggregate_host(grouped.raw(), y_grad.data.data(), y_grad.rows, y_grad.cols,
                                     x_grad.data.data(),
                                     commit_flags(mode == CommitMode::Grouped ? CommitMode::Fast : mode), c));
    if (counters) {
        counters->edges_traversed += c[0];
        counters->groups_executed += c[1];
        counters->atomic_commits += c[2];
    }
}

// aggregate_pull<double> / the timed stage in the reference's default
// precision (Deterministic order, f64 weights; bit-exact with the f64 build)
inline void aggregate_pull(const DeviceGroups& grouped, const MatrixD& input, MatrixD& output,
                           CommitMode mode = CommitMode::Deterministic, int workers = 0,
                           StageCounters* counters = nullptr) {
    (void)workers;
    if (output.rows != grouped.dest_count()) throw ShapeError("aggregate_pull: output rows != dest count");
    if (output.cols != input.cols) throw ShapeError("aggregate_pull: input/output dims differ");
    std::uint64_t c[3] = {0, 0, 0};
    check(pg_aggregate_pull_host_f64(grouped.raw(), input.data.data(), input.rows, input.cols, output.data.data(),
                                     commit_flags(mode == CommitMode::Grouped ? CommitMode::Fast : mode), c));
    if (counters) {
        counters->edges_traversed += c[0];
        counters->groups_executed += c[1];
        counters->atomic_commits += c[2];
    }
}
inline void backward_aggregation(const DeviceGroups& grouped, const MatrixD& y_grad, MatrixD& x_grad,
                                 CommitMode mode = CommitMode::Deterministic, StageCounters* counters = nullptr) {
    if (x_grad.rows != grouped.dest_count() || x_grad.cols != y_grad.cols)
        throw ShapeError("backward_aggregation: x_grad shape mismatch");
    std::uint64_t c[3] = {0, 0, 0};
    check(pg_backward_aggregate_host_f64(grouped.raw(), y_grad.data.data(), y_grad.rows, y_grad.cols,
                                         x_grad.data.data(),
                                         commit_flags(mode == CommitMode::Grouped ? CommitMode::Fast : mode), c));
    if (counters) {
        counters->edges_traversed += c[0];
        counters->groups_executed += c[1];
        counters->atomic_commits += c[2];
    }
}

// ---------------- the GCN chain (engine.hpp), device resident ----------------

// A device fp32 matrix (row pitch padded to 16-byte rows up to 32 floats,
// 128-byte lines beyond, as the SpMM prefers); upload/download to the
// reference's DenseMatrix layout.
class DeviceMatrix {
public:
    DeviceMatrix() = default;
    DeviceMatrix(std::size_t rows, std::size_t cols, int device = 0) : dev_(device) {
        m_.rows = rows;
        m_.cols = cols;
        m_.ld = cols <= 32 ? (cols + 3) / 4 * 4 : (cols + 31) / 32 * 32;
        void* p = nullptr;
        check(pg_device_alloc(device, m_.rows * m_.ld * 4, &p));
        m_.data = static_cast<float*>(p);
        check(pg_memset_zero(device, p, m_.rows * m_.ld * 4));
    }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    DeviceMatrix(DeviceMatrix&& o) noexcept : m_(std::exchange(o.m_, pg_mat{})), dev_(o.dev_) {}
    DeviceMatrix& operator=(DeviceMatrix&& o) noexcept {
        if (this != &o) {
            release();
            m_ = std::exchange(o.m_, pg_mat{});
            dev_ = o.dev_;
        }
        return *this;
    }
    ~DeviceMatrix() { release(); }

    static DeviceMatrix upload(const MatrixF& h, int device = 0) {
        DeviceMatrix d(h.rows, h.cols, device);
        check(pg_mat_upload(device, d.m_, h.data.data()));
        return d;
    }
    MatrixF download() const {
        MatrixF h(m_.rows, m_.cols);
        check(pg_mat_download(dev_, h.data.data(), m_));
        return h;
    }
    std::size_t rows() const { return m_.rows; }
    std::size_t cols() const { return m_.cols; }
    const pg_mat& raw() const { return m_; }

private:
    void release() {
        if (m_.data) pg_device_free(dev_, m_.data);
        m_ = pg_mat{};
    }
    pg_mat m_{};
    int dev_ = 0;
};

// ---------------- multi-GPU: the library's NCCL communicator ----------------
// One rank per device; rank 0's unique_id() is shipped to every rank by the
// caller's bootstrap (MPI, a file, torch.distributed).
class Communicator {
public:
    using Id = std::array<std::uint8_t, PG_COMM_ID_BYTES>;
    static Id unique_id() {
        Id id{};
        check(pg_comm_unique_id(id.data()));
        return id;
    }
    Communicator(int device, const Id& id, int world, int rank) : dev_(device) {
        check(pg_comm_init_rank(device, id.data(), world, rank, &h_.h));
        check(pg_comm_info(h_.h, &world_, &rank_, &nccl_));
    }
    int world() const { return world_; }
    int rank() const { return rank_; }
    int nccl_version() const { return nccl_; }
    // edge-balanced destination cuts of a path (pg_path_shard_bounds)
    std::vector<std::uint32_t> shard_bounds(const DevicePath& p) const {
        std::vector<std::uint32_t> b(world_ + 1);
        check(pg_path_shard_bounds(p.raw(), static_cast<std::uint32_t>(world_), b.data()));
        return b;
    }
    // engine.hpp:331-338 row-sharded: y_full holds this rank's parent rows;
    // x_rows receives destination rows [dest_bounds[rank], dest_bounds[rank+1])
    void backward_aggregation(const DeviceGroups& grouped, std::span<const std::uint32_t> parent_bounds,
                              std::span<const std::uint32_t> dest_bounds, DeviceMatrix& y_full, DeviceMatrix& x_rows,
                              bool single_pass = false) const {
        if (parent_bounds.size() != static_cast<std::size_t>(world_) + 1 ||
            dest_bounds.size() != static_cast<std::size_t>(world_) + 1)
            throw ConfigError("sharded: bounds need world + 1 cuts");
        if (x_rows.cols() != y_full.cols() ||
            x_rows.rows() != dest_bounds[rank_ + 1] - dest_bounds[rank_])
            throw ShapeError("sharded: x_rows shape mismatch");
        check(pg_backward_aggregate_sharded(h_.h, grouped.raw(), parent_bounds.data(), dest_bounds.data(),
                                            y_full.raw().data, y_full.rows(), y_full.raw().ld, x_rows.raw().data,
                                            x_rows.raw().ld, y_full.cols(),
                                            PG_AGG_OVERWRITE | (single_pass ? PG_SHARD_SINGLE_PASS : 0u), nullptr));
        check(pg_device_synchronize(dev_));
    }
    void allgather_rows(DeviceMatrix& rows, std::span<const std::uint32_t> bounds) const {
        check(pg_comm_allgather_rows(h_.h, rows.raw().data, rows.raw().ld, bounds.data(), nullptr));
        check(pg_device_synchronize(dev_));
    }
    pg_comm raw() const { return h_.h; }

private:
    Handle<pg_comm, pg_comm_destroy> h_;
    int dev_ = 0, world_ = 1, rank_ = 0, nccl_ = 0;
};

struct DeviceArtifacts {                          // EpochArtifacts (engine.hpp:27-31)
    std::vector<DeviceMatrix> x, y, pre_act;      // x[0] is unused (the caller's X^(0))
};

namespace detail {
inline std::vector<pg_mat> raws(const std::vector<DeviceMatrix>& v, std::size_t from = 0) {
    std::vector<pg_mat> out;
    for (std::size_t i = from; i < v.size(); ++i) out.push_back(v[i].raw());
    return out;
}
}  // namespace detail

// engine.hpp:114-140 over a full-graph grouping
inline DeviceArtifacts forward(const DeviceGroups& graph, const DeviceMatrix& x0,
                               const std::vector<DeviceMatrix>& weights, int device = 0) {
    DeviceArtifacts a;
    a.x.emplace_back();
    std::size_t cur = x0.cols();
    for (const auto& w : weights) {
        a.y.emplace_back(x0.rows(), cur, device);
        a.pre_act.emplace_back(x0.rows(), w.cols(), device);
        a.x.emplace_back(x0.rows(), w.cols(), device);
        cur = w.cols();
    }
    auto W = detail::raws(weights), Y = detail::raws(a.y), P = detail::raws(a.pre_act), X = detail::raws(a.x, 1);
    check(pg_forward(graph.raw(), x0.raw(), W.data(), weights.size(), Y.data(), P.data(), X.data(), nullptr));
    return a;
}

// engine.hpp:146-156 (vt on the host)
inline DeviceMatrix top_grad_from_probs(const DeviceMatrix& probs, const DeviceMatrix& ref,
                                        std::span<const VertexId> vt, int device = 0) {
    DeviceMatrix out(probs.rows(), probs.cols(), device);
    void* d = nullptr;
    check(pg_device_alloc(device, vt.size() * 4, &d));
    try {
        check(pg_memcpy_h2d(device, d, vt.data(), vt.size() * 4));
        check(pg_top_grad_from_probs(probs.raw(), ref.raw(), static_cast<const uint32_t*>(d), vt.size(), out.raw(),
                                     nullptr));
        check(pg_device_synchronize(device));
    } catch (...) {
        pg_device_free(device, d);
        throw;
    }
    pg_device_free(device, d);
    return out;
}

struct WorkCounts {                               // WorkCounters::backward_edges_per_layer
    std::vector<std::uint64_t> backward_edges_per_layer;
};

namespace detail {
inline std::vector<DeviceMatrix> wgrads(const std::vector<DeviceMatrix>& w, int device) {
    std::vector<DeviceMatrix> out;
    for (const auto& m : w) out.emplace_back(m.rows(), m.cols(), device);
    return out;
}
}  // namespace detail

// engine.hpp:267-349. groups[i] groups paths[i] (SG_{L-1} first).
inline std::vector<DeviceMatrix> backward_epp(const std::vector<DeviceGroups>& groups, const DeviceFrontiers& F,
                                              const DeviceArtifacts& arts, const DeviceMatrix& top_grad,
                                              const std::vector<DeviceMatrix>& weights, GatherMode gather,
                                              std::uint64_t expected_fingerprint, WorkCounts* counters = nullptr,
                                              int device = 0) {
    const std::size_t L = weights.size();
    if (groups.size() != L || F.depth() != L)
        throw StalenessError("epp backward: paths were prepared for a different layer count");
    std::vector<pg_groups> hs;
    for (const auto& g : groups) hs.push_back(g.raw());
    auto wg = detail::wgrads(weights, device);
    auto Y = detail::raws(arts.y), P = detail::raws(arts.pre_act), W = detail::raws(weights), WG = detail::raws(wg);
    std::vector<std::uint64_t> e(L);
    check(pg_backward_epp(hs.data(), F.raw(), L, Y.data(), P.data(), top_grad.raw(), W.data(), expected_fingerprint,
                          gather == GatherMode::Global ? 1 : 0, WG.data(), nullptr, e.data(), nullptr));
    if (counters) counters->backward_edges_per_layer = e;
    return wg;
}

// engine.hpp:177-214 (Alg. 1)
inline std::vector<DeviceMatrix> backward_all_active(const DeviceGroups& graph, const DeviceArtifacts& arts,
                                                     const DeviceMatrix& top_grad,
                                                     const std::vector<DeviceMatrix>& weights,
                                                     WorkCounts* counters = nullptr, int device = 0) {
    const std::size_t L = weights.size();
    auto wg = detail::wgrads(weights, device);
    auto Y = detail::raws(arts.y), P = detail::raws(arts.pre_act), W = detail::raws(weights), WG = detail::raws(wg);
    std::vector<std::uint64_t> e(L);
    check(pg_backward_all_active(graph.raw(), L, Y.data(), P.data(), top_grad.raw(), W.data(), WG.data(), nullptr,
                                 e.data(), nullptr));
    if (counters) counters->backward_edges_per_layer = e;
    return wg;
}

// engine.hpp:218-257
inline std::vector<DeviceMatrix> backward_ifelse(const DeviceGroups& graph, const DeviceFrontiers& F,
                                                 const DeviceArtifacts& arts, const DeviceMatrix& top_grad,
                                                 const std::vector<DeviceMatrix>& weights,
                                                 WorkCounts* counters = nullptr, int device = 0) {
    const std::size_t L = weights.size();
    auto wg = detail::wgrads(weights, device);
    auto Y = detail::raws(arts.y), P = detail::raws(arts.pre_act), W = detail::raws(weights), WG = detail::raws(wg);
    std::vector<std::uint64_t> e(L);
    check(pg_backward_ifelse(graph.raw(), F.raw(), L, Y.data(), P.data(), top_grad.raw(), W.data(), WG.data(),
                             nullptr, counters ? e.data() : nullptr, nullptr));
    if (counters) counters->backward_edges_per_layer = e;
    return wg;
}

}  // namespace pathgcn::b200
