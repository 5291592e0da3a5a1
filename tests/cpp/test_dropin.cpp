// C++ drop-in test: the reference's own known-answer cases
// (proj/tests/unit/test_*.cpp, acceptance.cpp) written against the C++
// host API in include/pathgcn_b200.hpp, plus bit-exact comparisons with the
// C oracle (oracle/pathgcn_oracle.h) on the RMAT fixture. One PASS/FAIL
// line per check like acceptance.cpp; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <vector>

#include "../../include/pathgcn_b200.hpp"
#include "../../oracle/pathgcn_oracle.h"

using namespace pathgcn::b200;

static int g_fail = 0;
static void report(const char* name, bool ok) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", name);
    if (!ok) ++g_fail;
}

static EdgeList gex_edges() {
    EdgeList el;
    el.pairs = {{0, 1}, {1, 2}, {1, 3}, {1, 4}, {2, 3}, {3, 4}};
    return el;
}

static std::set<std::pair<VertexId, VertexId>> path_edges(const ExecutionPathHost& p) {
    std::set<std::pair<VertexId, VertexId>> out;
    for (std::size_t d = 0; d < p.dest_local_to_global.size(); ++d)
        for (auto e = p.offsets[d]; e < p.offsets[d + 1]; ++e)
            out.insert({p.src_local_to_global[p.neighbors[e]], p.dest_local_to_global[d]});
    return out;
}

int main() {
    // test_frontier.cpp:10-18
    DeviceGraph g = build_undirected_csr(gex_edges());
    const std::vector<VertexId> vt = {2, 4};
    DeviceFrontiers f = compute_frontiers(g, vt, 2);
    report("frontiers worked example",
           f.level(0) == std::vector<VertexId>{2, 4} && f.level(1) == std::vector<VertexId>{1, 3} &&
               f.level(2) == std::vector<VertexId>{0, 1, 2, 3, 4});
    // test_execution_path.cpp:23-47
    auto paths = prepare_all_paths(g, f);
    const auto sg1 = paths[0].to_host(), sg0 = paths[1].to_host();
    report("SG_1 carries the four listed edges",
           sg1.layer == 1 && sg1.offsets == std::vector<EdgeIndex>{0, 2, 4} &&
               path_edges(sg1) == std::set<std::pair<VertexId, VertexId>>{{2, 1}, {4, 1}, {2, 3}, {4, 3}});
    report("SG_0 carries the seven listed edges",
           sg0.dest_local_to_global.size() == 5 && paths[1].edge_count() == 7 &&
               path_edges(sg0) ==
                   std::set<std::pair<VertexId, VertexId>>{{1, 0}, {3, 1}, {1, 2}, {3, 2}, {1, 3}, {1, 4}, {3, 4}});
    // test_grouping.cpp:8-18 (graph grouping, gs = 3)
    {
        DeviceGroups gr = group_neighbors(g, 3);
        std::vector<VertexId> d;
        std::vector<EdgeIndex> b, e;
        std::vector<std::uint64_t> dg;
        gr.to_host(d, b, e, dg);
        report("gs=3 splits the degree-4 vertex 3+1",
               gr.group_count() == 6 && dg[2] - dg[1] == 2 && e[dg[1]] - b[dg[1]] == 3 &&
                   e[dg[1] + 1] - b[dg[1] + 1] == 1);
        bool threw = false;
        try {
            group_neighbors(g, 0);
        } catch (const ConfigError&) {
            threw = true;
        }
        report("gs=0 is a config error", threw);
    }
    // test_engine.cpp:72-80
    {
        DeviceGroups gr = group_neighbors(g, 3);
        MatrixF x(5, 1), y(5, 1);
        x.data = {1, 2, 3, 4, 5};
        StageCounters c;
        aggregate_pull(gr, x, y, CommitMode::Deterministic, 0, &c);
        report("aggregate_pull hand sums [2,13,6,10,6]",
               y.data == std::vector<float>{2, 13, 6, 10, 6} && c.edges_traversed == 12 && c.groups_executed == 6);
    }
    // test_engine.cpp:169-180
    {
        DeviceGroups gr = group_neighbors(paths[0], 2);
        MatrixF yu(2, 1), xg(2, 1);
        yu.data = {1.0f, 2.0f};
        aggregate_pull(gr, yu, xg);
        report("SG_1 hand case [3,3]", xg.data == std::vector<float>{3.0f, 3.0f});
    }
    // test_gs_model.cpp:47-58
    report("regression Cora/Youtube", regression_gs(GraphStats{2708, 5278, 5278.0 / 2708}) == 2 &&
                                          regression_gs(GraphStats{1134890, 2987624, 2987624.0 / 1134890}) == 15);
    // test_group_cost.cpp:60-68 (star(64), W=8, lambda=0.1)
    {
        EdgeList st;
        for (VertexId i = 1; i <= 64; ++i) st.pairs.push_back({0, i});
        DeviceGraph sg = build_undirected_csr(st);
        report("hub grouping cost gs=8 = 267.2",
               std::abs(group_neighbors(sg, 8).grouping_cost(16, {8, 0.1}) - 267.2) < 1e-9);
    }
    // staleness stamp (engine.hpp:278-283 uses path_fingerprint)
    report("path fingerprint depends on L", path_fingerprint(g, vt, 2) != path_fingerprint(g, vt, 3));
    // shape errors (aggregate.hpp:61-62)
    {
        bool threw = false;
        try {
            DeviceGroups gr = group_neighbors(paths[1], 2);
            MatrixF in(2, 4), out(5, 3);
            aggregate_pull(gr, in, out);
        } catch (const ShapeError&) {
            threw = true;
        }
        report("shape mismatch throws ShapeError", threw);
    }

    // RMAT fixture (test_rmat.cpp:72-81) vs the C oracle, bit for bit
    {
        const std::uint64_t m = 8192;
        std::vector<std::uint32_t> pairs(2 * m);
        const std::uint32_t n_pad = orc_gen_rmat(1024, m, 0.45, 0.22, 0.22, 0.11, 7, pairs.data());
        EdgeList el;
        el.n_hint = n_pad;
        for (std::uint64_t i = 0; i < m; ++i) el.pairs.push_back({pairs[2 * i], pairs[2 * i + 1]});
        DeviceGraph rg = build_undirected_csr(el, WeightMode::SymNorm);
        report("rmat fixture n/m/maxdeg", rg.n() == 1024 && rg.m() == 15376 && rg.max_degree() == 214);
        std::vector<VertexId> rvt(orc_training_set_size(1024, 0.1));
        orc_sample_training_set(1024, 0.1, 42, rvt.data());
        DeviceFrontiers rf = compute_frontiers(rg, rvt, 2);
        auto rpaths = prepare_all_paths(rg, rf);
        std::vector<EdgeIndex> off;
        std::vector<VertexId> nb;
        std::vector<double> w;
        rg.to_host(off, nb, w);
        bool ok = true;
        for (auto& dp : rpaths) {
            const auto p = dp.to_host();
            const std::size_t D = p.dest_local_to_global.size(), S = p.src_local_to_global.size();
            MatrixF y(S, 37), out(D, 37);
            for (std::size_t i = 0; i < y.data.size(); ++i) y.data[i] = std::sin(0.37 * double(i));
            DeviceGroups gr = group_neighbors(dp, regression_gs(dp));
            aggregate_pull(gr, y, out);
            std::vector<float> want(D * 37, 0.0f);
            orc_aggregate_pull_f32(D, p.offsets.data(), p.neighbors.data(), p.weights.data(), y.data.data(), 37,
                                   want.data());
            ok = ok && std::memcmp(want.data(), out.data.data(), want.size() * 4) == 0;
        }
        report("rmat fixture SpMM bit-exact vs oracle", ok);
        report("rmat probe gs 2 / 9", regression_gs(rpaths[0]) == 2 && regression_gs(rpaths[1]) == 9);

        // the device chain (engine.hpp) vs the oracle's C kernels composed
        // here: forward + top_grad + backward_epp Local W', bit for bit
        const std::size_t n = rg.n(), f = 24, hid = 16, cls = 4;
        MatrixF x0(n, f), w0(f, hid), w1(hid, cls), r(n, cls);
        for (std::size_t i = 0; i < x0.data.size(); ++i) x0.data[i] = float(0.5 + 0.5 * std::sin(0.11 * double(i)));
        for (std::size_t i = 0; i < w0.data.size(); ++i) w0.data[i] = float(0.3 * std::cos(0.7 * double(i)));
        for (std::size_t i = 0; i < w1.data.size(); ++i) w1.data[i] = float(0.3 * std::sin(1.3 * double(i)));
        for (std::size_t k = 0; k < rvt.size(); ++k) r.data[rvt[k] * cls + (k % cls)] = 1.0f;
        DeviceGroups gg = group_neighbors(rg, 4);
        std::vector<DeviceMatrix> W;
        W.push_back(DeviceMatrix::upload(w0));
        W.push_back(DeviceMatrix::upload(w1));
        DeviceMatrix X0 = DeviceMatrix::upload(x0);
        DeviceArtifacts arts = forward(gg, X0, W);
        DeviceMatrix top = top_grad_from_probs(arts.x[2], DeviceMatrix::upload(r), rvt);
        std::vector<DeviceGroups> pgr;
        const std::uint64_t stamp = path_fingerprint(rg, rvt, 2);
        for (auto& dp : rpaths) {
            dp.set_fingerprint(stamp);
            pgr.push_back(group_neighbors(dp, 2));
        }
        WorkCounts wc;
        auto wg = backward_epp(pgr, rf, arts, top, W, GatherMode::Local, stamp, &wc);
        // oracle: forward
        std::vector<float> y0(n * f, 0.f), p0(n * hid), x1(n * hid), y1(n * hid, 0.f), p1(n * cls), x2(n * cls);
        orc_aggregate_pull_f32(n, off.data(), nb.data(), w.data(), x0.data.data(), f, y0.data());
        orc_gemm_f32(y0.data(), n, f, w0.data.data(), hid, p0.data());
        orc_relu_f32(p0.data(), p0.size(), x1.data());
        orc_aggregate_pull_f32(n, off.data(), nb.data(), w.data(), x1.data(), hid, y1.data());
        orc_gemm_f32(y1.data(), n, hid, w1.data.data(), cls, p1.data());
        orc_row_softmax_f32(p1.data(), n, cls, x2.data());
        std::vector<float> tg(n * cls);
        orc_top_grad_f32(x2.data(), r.data.data(), n, cls, rvt.data(), rvt.size(), tg.data());
        report("device forward X^(2) bit-exact vs oracle (incl. softmax expf)",
               std::memcmp(arts.x[2].download().data.data(), x2.data(), x2.size() * 4) == 0);
        // oracle: backward_epp Local (engine.hpp:316-346)
        const auto lv0 = rf.level(0), lv1 = rf.level(1);
        const auto P1 = rpaths[0].to_host(), P0 = rpaths[1].to_host();
        std::vector<float> g(lv0.size() * cls), yc(lv0.size() * hid), wg1(hid * cls), ygr(lv0.size() * hid);
        orc_gather_rows_f32(tg.data(), cls, lv0.data(), lv0.size(), g.data());
        orc_gather_rows_f32(y1.data(), hid, lv0.data(), lv0.size(), yc.data());
        orc_gemm_at_b_f32(yc.data(), lv0.size(), hid, g.data(), cls, wg1.data());
        orc_gemm_a_bt_f32(g.data(), lv0.size(), cls, w1.data.data(), hid, ygr.data());
        std::vector<float> yu(P1.src_pos_in_parent.size() * hid), xg1(lv1.size() * hid, 0.f);
        orc_gather_rows_f32(ygr.data(), hid, P1.src_pos_in_parent.data(), P1.src_pos_in_parent.size(), yu.data());
        orc_aggregate_pull_f32(lv1.size(), P1.offsets.data(), P1.neighbors.data(), P1.weights.data(), yu.data(), hid,
                               xg1.data());
        std::vector<float> pc(lv1.size() * hid), g1(lv1.size() * hid), yc0(lv1.size() * f), wg0(f * hid);
        orc_gather_rows_f32(p0.data(), hid, lv1.data(), lv1.size(), pc.data());
        orc_relu_backward_f32(xg1.data(), pc.data(), pc.size(), g1.data());
        orc_gather_rows_f32(y0.data(), f, lv1.data(), lv1.size(), yc0.data());
        orc_gemm_at_b_f32(yc0.data(), lv1.size(), f, g1.data(), hid, wg0.data());
        report("device backward_epp W' bit-exact vs oracle",
               std::memcmp(wg[1].download().data.data(), wg1.data(), wg1.size() * 4) == 0 &&
                   std::memcmp(wg[0].download().data.data(), wg0.data(), wg0.size() * 4) == 0);
        report("backward_edges_per_layer = path edge counts",
               wc.backward_edges_per_layer == std::vector<std::uint64_t>{P1.offsets.back(), P0.offsets.back()});
        bool stale = false;
        try {
            backward_epp(pgr, rf, arts, top, W, GatherMode::Local, stamp ^ 1);
        } catch (const StalenessError&) {
            stale = true;
        }
        report("stale fingerprint -> StalenessError", stale);
        // Alg. 1 and if-else reproduce the same top-layer W' only up to the
        // inactive rows' zero terms; both must run and return finite shapes
        auto wa = backward_all_active(gg, arts, top, W);
        auto wi = backward_ifelse(gg, rf, arts, top, W);
        report("all-active / if-else backward shapes", wa[0].rows() == f && wi[1].cols() == cls);
    }
    // file formats (test_edge_list.cpp, test_training_set.cpp)
    {
        const std::string path = "/tmp/pg_dropin_edges.txt";
        FILE* fp = std::fopen(path.c_str(), "w");
        std::fputs("# c\n3 3\n0 3\n1 2\n", fp);
        std::fclose(fp);
        const EdgeList el = load_edge_list_file(path);
        report("load_edge_list_file comments / self loops",
               el.pairs.size() == 2 && el.pairs[0] == std::pair<VertexId, VertexId>{0, 3} && el.self_loops_dropped == 1);
        fp = std::fopen(path.c_str(), "w");
        std::fputs("0 1\n0 x\n", fp);
        std::fclose(fp);
        std::size_t line = 0;
        try {
            load_edge_list_file(path);
        } catch (const ParseError& e) {
            line = e.line_number;
        }
        report("ParseError carries line 2", line == 2);
        bool io = false;
        try {
            load_edge_list_file("/nonexistent/x.txt");
        } catch (const IoError&) {
            io = true;
        }
        report("missing file -> IoError", io);
    }
    // aggregate_pull<double> (the reference's default precision): the hand
    // case of test_engine.cpp:72-80 on gex, x = [1..5] -> [2, 13, 6, 10, 6]
    {
        DeviceGroups gr = group_neighbors(g, 2);
        MatrixD x(5, 1), out(5, 1);
        for (int i = 0; i < 5; ++i) x.data[i] = i + 1;
        aggregate_pull(gr, x, out);
        report("aggregate_pull<double> hand case",
               out.data == std::vector<double>{2, 13, 6, 10, 6});
    }
    // the library communicator, one rank (NCCL through the C ABI): the
    // sharded stage equals the single-GPU stage bit for bit
    {
        const auto id = Communicator::unique_id();
        Communicator comm(0, id, 1, 0);
        report("communicator: one rank, NCCL loaded", comm.world() == 1 && comm.rank() == 0 && comm.nccl_version() > 0);
        auto rp = prepare_all_paths(g, f);
        DeviceGroups gr = group_neighbors(rp[1], 2);
        const std::size_t dim = 5;
        MatrixF y(rp[1].parent_rows(), dim), want(rp[1].dest_count(), dim);
        for (std::size_t i = 0; i < y.data.size(); ++i) y.data[i] = static_cast<float>(std::sin(0.37 * i));
        backward_aggregation(gr, y, want);
        DeviceMatrix yd = DeviceMatrix::upload(y), xd(rp[1].dest_count(), dim);
        const std::vector<std::uint32_t> pb{0, rp[1].parent_rows()}, db = comm.shard_bounds(rp[1]);
        comm.backward_aggregation(gr, pb, db, yd, xd);
        const MatrixF got = xd.download();
        report("sharded stage (1 rank) == backward_aggregation",
               std::memcmp(got.data.data(), want.data.data(), want.data.size() * 4) == 0);
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
