// C ABI of libpathgcn_b200.so (include/pathgcn_b200.h): status codes,
// handle plumbing, host-side input synthesis with the reference's exact
// libstdc++ random streams, and the host-buffer drop-ins.
#include <chrono>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <emmintrin.h>

#include "../../include/pathgcn_b200.h"
#include "pg_internal.h"

using namespace pg;

namespace {

thread_local std::string g_err;
thread_local int g_kind = PG_KIND_NONE;
thread_local uint64_t g_line = 0;

}  // namespace

// the calling thread's last failure (pg_last_error / pg_last_error_kind),
// shared with the communicator entry points (comm.cu)
void pg::record_error(const pg::Error& e) {
    g_err = e.what();
    g_kind = e.kind;
    g_line = e.line;
}

namespace {

template <typename F>
int guard(F&& f) {
    try {
        f();
        return PG_OK;
    } catch (const pg::Error& e) {
        record_error(e);
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        g_kind = PG_KIND_DEVICE;
        g_line = 0;
        return PG_ERR_DEVICE;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_kind = PG_KIND_CONFIG;
        g_line = 0;
        return PG_ERR_CONFIG;
    }
}

template <typename T>
T* need(T* p, const char* what) {
    if (!p) fail(kConfig, std::string(what) + ": null handle");
    return p;
}

Graph* G_(pg_graph h) { return need(reinterpret_cast<Graph*>(h), "graph"); }
Frontiers* F_(pg_frontiers h) { return need(reinterpret_cast<Frontiers*>(h), "frontiers"); }
Path* P_(pg_path h) { return need(reinterpret_cast<Path*>(h), "path"); }
Groups* R_(pg_groups h) { return need(reinterpret_cast<Groups*>(h), "groups"); }

// engine.hpp:60-68 derive_seed (splitmix-style stream derivation)
uint64_t derive_seed(uint64_t seed, uint64_t stream) {
    uint64_t h = seed ^ (0x9e3779b97f4a7c15ull + stream);
    h ^= h >> 30;
    h *= 0xbf58476d1ce4e5b9ull;
    h ^= h >> 27;
    h *= 0x94d049bb133111ebull;
    h ^= h >> 31;
    return h;
}

void fnv_mix(uint64_t& h, uint64_t x) {
    for (int i = 0; i < 8; ++i) {
        h ^= (x >> (8 * i)) & 0xFF;
        h *= 1099511628211ull;
    }
}

// csr_graph.cpp:19-31 (host: FNV-1a is sequential by definition)
uint64_t graph_fp(Graph& g) {
    if (g.fp_valid) return g.fp;
    DeviceGuard dg(g.device);
    cudaStream_t s = lib_stream(g.device);
    std::vector<uint64_t> off(static_cast<uint64_t>(g.n) + 1);
    std::vector<uint32_t> nb(g.m);
    PG_CUDA(cudaMemcpyAsync(off.data(), g.offsets.get(), off.size() * 8, cudaMemcpyDeviceToHost, s));
    if (g.m) PG_CUDA(cudaMemcpyAsync(nb.data(), g.nbrs.get(), g.m * 4, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    uint64_t h = 1469598103934665603ull;
    fnv_mix(h, g.n);
    for (uint64_t o : off) fnv_mix(h, o);
    for (uint32_t u : nb) fnv_mix(h, u);
    g.fp = h;
    g.fp_valid = true;
    return h;
}

// training_set.cpp:15-26
uint64_t training_fp(const uint32_t* vt, uint64_t k) {
    uint64_t h = 1469598103934665603ull;
    fnv_mix(h, k);
    for (uint64_t i = 0; i < k; ++i) fnv_mix(h, vt[i]);
    return h;
}

// The CSR a grouping runs over.
struct Base {
    uint32_t D;
    const uint64_t* offsets;
    uint64_t E;
    uint32_t in_rows_local;  // rows of a local-indexed input
};

Base base_of(Groups& G) {
    if (G.path) return {G.path->D, G.path->offsets.get(), G.path->E, G.path->S};
    return {G.graph->n, G.graph->offsets.get(), G.graph->m, G.graph->n};
}

uint64_t fast_atomic_groups(Groups& G) {
    // sum over destinations owning more than one group of their group count
    const Base b = base_of(G);
    std::vector<uint64_t> dg(static_cast<uint64_t>(b.D) + 1);
    DeviceGuard dev(G.device);
    cudaStream_t s = lib_stream(G.device);
    PG_CUDA(cudaMemcpyAsync(dg.data(), G.dest_groups.get(), dg.size() * 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    uint64_t t = 0;
    for (uint32_t v = 0; v < b.D; ++v) {
        const uint64_t k = dg[v + 1] - dg[v];
        if (k > 1) t += k;
    }
    return t;
}

void counters_of(Groups& G, uint64_t dim, unsigned flags, uint64_t* c) {
    if (!c) return;
    const Base b = base_of(G);
    c[0] = b.E;
    c[1] = G.G;
    c[2] = (flags & PG_AGG_FAST) ? fast_atomic_groups(G) * dim : 0;
}

// rows of the parent-indexed input: the parent frontier, or the padded
// allgather layout once pg_groups_remap_sources installed a map
uint64_t y_rows_of(const Groups& G) { return G.edges_remap.get() ? G.remap_rows : G.path->P; }

DMat dm(const pg_mat& m) {
    if (m.ld < m.cols) fail_shape("matrix leading dimension smaller than its columns");
    if (!m.data && m.rows * m.cols) fail(kConfig, "null matrix data");
    return DMat{m.data, m.rows, m.cols, m.ld};
}

void check_dims(uint64_t dim, uint64_t ld_in, uint64_t ld_out) {
    if (ld_in < dim || ld_out < dim) fail_shape("aggregate_pull: leading dimension smaller than dim");
}

// Source segments for a whole-path SpMM (tuning "src_segs": 0 = this
// rule): two when one chunk-major pass would gather from more than ~80 MB
// (P rows x 512 B) and at most ~400 MB; more passes cost an output
// read+write each and lost in the measured sweep (K = 3, 4, 6).
// hub threshold of a (segment) range: the row kernel's own knob, else the
// measured default rule
uint64_t heavy_degree(uint64_t dim, uint64_t range_edges) {
    if (!heavy_min_forced()) {
        if (row_kernel_on(dim) && tuning(kTuneRowHeavy) > 0) return static_cast<uint64_t>(tuning(kTuneRowHeavy));
        // wide-row hubs inlined as the main kernel's destination-major front
        if ((dim + 3) / 4 > 16 && tuning(kTuneHubInline) != 0 && tuning(kTuneHubFrontMin) > 0)
            return static_cast<uint64_t>(tuning(kTuneHubFrontMin));
    }
    return heavy_min_degree(dim, range_edges);
}

uint32_t auto_src_segments(uint64_t P, uint64_t D, uint64_t E, uint64_t dim) {
    const int64_t forced = tuning(kTuneSrcSegs);
    if (forced > 0) return static_cast<uint32_t>(std::min<int64_t>(forced, 16));
    if ((dim + 3) / 4 <= 16) return 1;  // narrow rows: one pass, the rows are small
    // an extra pass re-reads and re-writes every output row: only worth it
    // when gathers dominate (measured: products' top path, E/D = 4, lost
    // 1.5 -> 2.8 ms with two passes)
    if (E < 64 * D) return 1;
    if (row_kernel_on(dim)) {
        // whole-row warps gather whole rows: segments of ~row_seg_mb MB
        const uint64_t rowb = ((dim + 31) / 32) * 128;
        const uint64_t tgt = static_cast<uint64_t>(std::max<int64_t>(8, tuning(kTuneRowSegMb))) << 20;
        return static_cast<uint32_t>(std::min<uint64_t>(16, (P * rowb + tgt - 1) / tgt));
    }
    const uint64_t w = P * 512;
    return (w > (80ull << 20) && w <= (400ull << 20)) ? 2 : 1;
}

// Core launch over the grouping's base: which edge stream and which schedule.
}  // namespace

// degree-ordered schedule of path rows [rb, re) of a grouping (cached; the
// caller holds G.mu)
Groups::RowSched* pg::row_sched(Groups& G, uint32_t rb, uint32_t re) {
    Path& p = *G.path;
    for (auto& x : G.row_scheds)
        if (x.rb == rb && x.re == re) return &x;
    G.row_scheds.emplace_back();
    Groups::RowSched* rs = &G.row_scheds.back();
    rs->rb = rb;
    rs->re = re;
    degree_order(p.offsets.get() + rb, re - rb, rs->order, lib_stream(p.device), &rs->hist);
    return rs;
}

// destinations of a row range with degree >= min_degree (a prefix of its
// degree order)
uint32_t pg::range_heavy(Groups& G, uint32_t rb, uint32_t re, uint64_t min_degree) {
    return row_sched(G, rb, re)->hist.heavy(min_degree);
}

namespace {
// Per-destination bounds of K L2-sized source segments of a path (cached on
// the grouping): cuts at equal source rows (tuning src_seg_balance 0,
// default) or rows weighted by edge count (100), a percentage mix.
void auto_segment_bounds(Groups& G, Path& p, uint32_t K) {
    const int64_t bal = std::clamp<int64_t>(tuning(kTuneSrcSegBalance), 0, 100);
    if (G.auto_seg_k == K && G.auto_seg_bal == bal) return;
    std::vector<uint64_t> cuts(K + 1);
    for (uint32_t k = 0; k <= K; ++k) cuts[k] = static_cast<uint64_t>(p.P) * k / K;
    if (bal > 0) {
        cudaStream_t ls = lib_stream(p.device);
        DevBuf<uint32_t> cnt(p.P, ls);
        source_edge_counts(p.edges_parent.get(), p.E, p.P, cnt.get(), ls);
        std::vector<uint32_t> hc(p.P);
        PG_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), p.P * 4ull, cudaMemcpyDeviceToHost, ls));
        PG_CUDA(cudaStreamSynchronize(ls));
        const double tot = static_cast<double>(p.E) * bal / 100.0 + static_cast<double>(p.P) * (100 - bal) / 100.0;
        double acc = 0;
        uint32_t k = 1;
        for (uint64_t r = 0; r < p.P && k < K; ++r) {
            acc += hc[r] * (bal / 100.0) + (100 - bal) / 100.0;
            while (k < K && acc >= tot * k / K) cuts[k++] = r + 1;
        }
        for (uint32_t j = 1; j <= K; ++j) cuts[j] = std::max(cuts[j], cuts[j - 1]);
    }
    segment_bounds(p.offsets.get(), p.edges_parent.get(), p.D, cuts.data(), K, G.auto_seg_bnd, lib_stream(p.device));
    G.auto_seg_k = K;
    G.auto_seg_bal = bal;
}
}  // namespace

void pg::run_aggregate(Groups& G, bool parent_indexed, uint32_t rb, uint32_t re, const float* in, uint64_t ld_in,
                   float* out, uint64_t ld_out, uint64_t dim, unsigned flags, cudaStream_t s, SegSel sel,
                   const AggExt& ext, const Edge* edges_override) {
    const bool accumulate = !(flags & PG_AGG_OVERWRITE);
    DeviceGuard dg(G.device);
    std::lock_guard<std::recursive_mutex> lk(G.mu);  // lazily built caches below
    if (flags & PG_AGG_GROUPED) {  // aggregate.hpp:84-115 over the groups
        const Base b = base_of(G);
        if (rb != 0 || re != b.D || sel.seg >= 0 || ext.any())
            fail(kConfig, "grouped aggregation runs over a whole grouping (no row ranges, segments or chains)");
        const Edge* edges = nullptr;
        if (G.path) {
            Path& p = *G.path;
            edges = p.edges_parent.get();
            if (parent_indexed && G.edges_remap.get()) edges = G.edges_remap.get();
            if (edges_override) edges = edges_override;
            if (!edges_override && !parent_indexed && p.S != p.P) {
                path_pack_local(p, lib_stream(p.device));
                PG_CUDA(cudaStreamSynchronize(lib_stream(p.device)));
                edges = p.edges_local.get();
            }
        } else {
            Graph& g = *G.graph;
            if (!g.edges.get()) {
                graph_pack_edges(g, lib_stream(g.device));
                PG_CUDA(cudaStreamSynchronize(lib_stream(g.device)));
            }
            edges = g.edges.get();
        }
        // tuning "grouped_seg": 0 (default) = atomic-free k_agg_grp + hub
        // fixup; 1 = the CTA-segmented kernel with atomics at CTA edges;
        // 2 = one atomic commit per extra group (the reference's omp atomic)
        if (tuning(kTuneGroupedSeg) == 0) {
            // L2-sized source segments for wide rows, like the Deterministic
            // path (tuning grouped_src_segs): each pass takes every group's
            // part of one segment. Partials per segment re-associate the sum
            // further, inside Fast mode's tolerance like its per-group partials.
            // (groups below 32 edges lose: each pass re-stages whole windows
            // for little work per group; Reddit layer 0 gs 8: 38 -> 58 ms,
            // gs 128: 22.3 -> 20.5 ms)
            const uint32_t K = G.path && parent_indexed && !G.edges_remap.get() && !edges_override &&
                                       tuning(kTuneGroupedSrcSegs) && G.gs >= 32
                                   ? auto_src_segments(G.path->P, G.path->D, G.path->E, dim)
                                   : 1;
            if (K > 1) {
                auto_segment_bounds(G, *G.path, K);
                for (uint32_t k = 0; k < K; ++k)
                    aggregate_groups_af(G, b.offsets, b.D, edges, in, ld_in, out, ld_out, dim, accumulate || k > 0, s,
                                        G.auto_seg_bnd.get() + static_cast<uint64_t>(k) * b.D,
                                        G.auto_seg_bnd.get() + static_cast<uint64_t>(k + 1) * b.D);
            } else {
                aggregate_groups_af(G, b.offsets, b.D, edges, in, ld_in, out, ld_out, dim, accumulate, s);
            }
        } else
            aggregate_groups(G.gbegin.get(), G.gend.get(), G.gdest.get(), G.dest_groups.get(), b.D, G.G, edges, in,
                             ld_in, out, ld_out, dim, accumulate, s);
        return;
    }
    if (G.path) {
        Path& p = *G.path;
        const Edge* edges = p.edges_parent.get();
        if (parent_indexed && G.edges_remap.get()) edges = G.edges_remap.get();
        if (edges_override) edges = edges_override;
        if (!edges_override && !parent_indexed && p.S != p.P) {
            path_pack_local(p, lib_stream(p.device));
            PG_CUDA(cudaStreamSynchronize(lib_stream(p.device)));
            edges = p.edges_local.get();
        }
        // Wide rows over a large parent frontier: split the sources into K
        // row segments run as accumulate passes (bit-identical: edges are
        // sorted by source row within a destination) so each chunk-major
        // pass gathers from a working set of P/K rows x 512 B that stays in
        // L2 (measured on the Reddit layer-0 path: K = 2 17.9 -> 16.3 ms).
        if (sel.seg < 0 && parent_indexed && !G.edges_remap.get() && !edges_override) {
            const uint32_t K = auto_src_segments(p.P, p.D, p.E, dim);
            if (K > 1) {
                auto_segment_bounds(G, p, K);
                for (uint32_t k = 0; k < K; ++k) {
                    AggExt ek = ext;
                    if (k + 1 < K) ek.relu_pre = nullptr;  // the epilogue applies to finished rows only
                    run_aggregate(G, parent_indexed, rb, re, in, ld_in, out, ld_out, dim,
                                  k == 0 ? flags : (flags & ~PG_AGG_OVERWRITE), s,
                                  SegSel{G.auto_seg_bnd.get(), static_cast<int>(k), K}, ek, nullptr);
                }
                return;
            }
        }
        // edge ranges: whole lists, or source segment `seg`
        const uint64_t* eb = p.offsets.get();
        const uint64_t* ee = p.offsets.get() + 1;
        uint64_t range_div = 1;
        if (sel.seg >= 0) {  // segments [seg, seg_end): bnd holds nseg + 1 boundary rows of D entries
            const int end = sel.seg_end < 0 ? sel.seg + 1 : sel.seg_end;
            eb = sel.bnd + static_cast<uint64_t>(sel.seg) * p.D;
            ee = sel.bnd + static_cast<uint64_t>(end) * p.D;
            range_div = std::max<uint64_t>(1, sel.nseg / static_cast<uint64_t>(end - sel.seg));
        }
        if (rb == 0 && re == p.D) {
            AggExt ew = ext;
            ew.avg_degree = p.E / range_div / std::max<uint64_t>(1, p.D);
            ew.n_edges = p.E / range_div;
            aggregate_det(eb, ee, edges, p.order.get(), p.D, 0, p.D,
                          p.hist.heavy(heavy_degree(dim, p.E / range_div)), in, ld_in, out, ld_out, dim,
                          accumulate, s, ew);
            return;
        }
        // row range: schedule of rows [rb, re) relative to rb (cached)
        Groups::RowSched* rs = row_sched(G, rb, re);
        AggExt er = ext;
        // a row range: hub chains on the deeper-pipelined side kernel
        // (tuning range_side_hubs 0: as the main kernel's front instead)
        er.side_hubs = tuning(kTuneRangeSideHubs) != 0;
        er.avg_degree = rs->hist.edges / range_div / std::max<uint64_t>(1, re - rb);
        er.n_edges = rs->hist.edges / range_div;
        const uint32_t nh = rs->hist.heavy(heavy_degree(dim, rs->hist.edges / range_div));
        const uint32_t nd = re - rb;
        if (ext.part) {
            const uint32_t np = std::min(rs->hist.heavy(std::max<uint64_t>(1, ext.part_min_degree)), nd);
            if (ext.part == 1) {  // the hub prefix only, all of it on the side kernel
                if (np) aggregate_det(eb + rb, ee + rb, edges, rs->order.get(), nd, 0, np, np, in, ld_in, out, ld_out,
                                      dim, accumulate, s, er);
            } else if (np < nd) {  // the rest; its own heavy ones (past the prefix) still on the side kernel
                aggregate_det(eb + rb, ee + rb, edges, rs->order.get(), nd, np, nd, nh > np ? nh - np : 0, in, ld_in,
                              out, ld_out, dim, accumulate, s, er);
            }
            return;
        }
        aggregate_det(eb + rb, ee + rb, edges, rs->order.get(), nd, 0, nd, nh, in, ld_in, out, ld_out, dim, accumulate,
                      s, er);
        return;
    }
    Graph& g = *G.graph;
    if (!g.edges.get()) {
        graph_pack_edges(g, lib_stream(g.device));
        PG_CUDA(cudaStreamSynchronize(lib_stream(g.device)));
    }
    if (!G.graph_order.get() && g.n)
        degree_order(g.offsets.get(), g.n, G.graph_order, lib_stream(g.device), &G.graph_hist);
    // the same L2-sized source segments as a path (forward / all-active /
    // if-else pulls over the whole graph): rows of g.edges are sorted by
    // neighbour id, so segment passes in order are the serial order
    const uint32_t K = auto_src_segments(g.n, g.n, g.m, dim);
    if (K > 1) {
        if (G.auto_seg_k != K) {
            std::vector<uint64_t> cuts(K + 1);
            for (uint32_t k = 0; k <= K; ++k) cuts[k] = static_cast<uint64_t>(g.n) * k / K;
            segment_bounds(g.offsets.get(), g.edges.get(), g.n, cuts.data(), K, G.auto_seg_bnd, lib_stream(g.device));
            G.auto_seg_k = K;
        }
        for (uint32_t k = 0; k < K; ++k) {
            AggExt ek = ext;
            if (k + 1 < K) ek.relu_pre = nullptr;  // the epilogue applies to finished rows only
            ek.avg_degree = g.m / K / std::max<uint64_t>(1, g.n);
            ek.n_edges = g.m / K;
            const uint64_t* eb = G.auto_seg_bnd.get() + static_cast<uint64_t>(k) * g.n;
            aggregate_det(eb, eb + g.n, g.edges.get(), G.graph_order.get(), g.n, 0, g.n,
                          G.graph_hist.heavy(heavy_degree(dim, g.m / K)), in, ld_in, out, ld_out, dim,
                          accumulate || k > 0, s, ek);
        }
        return;
    }
    AggExt ew = ext;
    ew.avg_degree = g.m / std::max<uint64_t>(1, g.n);
    ew.n_edges = g.m;
    aggregate_det(g.offsets.get(), g.offsets.get() + 1, g.edges.get(), G.graph_order.get(), g.n, 0, g.n,
                  G.graph_hist.heavy(heavy_degree(dim, g.m)), in, ld_in, out, ld_out, dim, accumulate, s, ew);
}

namespace {

struct CopyStreams {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    // repack streams: the odd-width row repacks run beside the DMA streams,
    // so a segment's / chunk's copy never queues behind the previous repack
    cudaStream_t rup = nullptr, rdn = nullptr;
    cudaStream_t hub = nullptr;  // the last pass's hub chunk, concurrent with the other chunks
    // per-chunk completion counters of the sequenced last pass: plain
    // cudaMalloc memory (stream memory operations reject pool allocations)
    unsigned* counters = nullptr;
    std::vector<cudaEvent_t> ev;  // sync events
    std::vector<cudaEvent_t> tev;  // timing events (host_trace)
    std::mutex call;              // one host-buffer call at a time per device owns them
};

// the caller holds c.call (taken here) for the whole host-buffer call
CopyStreams& copy_streams(int device, size_t nev, std::unique_lock<std::mutex>& held) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<CopyStreams>> per_dev;
    CopyStreams* cp;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (static_cast<int>(per_dev.size()) <= device) per_dev.resize(device + 1);
        if (!per_dev[device]) per_dev[device] = std::make_unique<CopyStreams>();
        cp = per_dev[device].get();
    }
    held = std::unique_lock<std::mutex>(cp->call);
    CopyStreams& c = *cp;
    if (!c.h2d) {
        // highest priority: the repack kernels of odd-width rows on these
        // streams must get SMs as soon as SpMM blocks retire, not after the
        // whole pass (their segment / chunk copy waits on them)
        int lo = 0, hi = 0;
        PG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int prio = tuning(kTuneHostCopyPrio) ? hi : 0;
        PG_CUDA(cudaStreamCreateWithPriority(&c.h2d, cudaStreamNonBlocking, prio));
        PG_CUDA(cudaStreamCreateWithPriority(&c.d2h, cudaStreamNonBlocking, prio));
        PG_CUDA(cudaStreamCreateWithPriority(&c.rup, cudaStreamNonBlocking, prio));
        PG_CUDA(cudaStreamCreateWithPriority(&c.rdn, cudaStreamNonBlocking, prio));
        PG_CUDA(cudaStreamCreateWithPriority(&c.hub, cudaStreamNonBlocking, prio));
        PG_CUDA(cudaMalloc(&c.counters, 64 * sizeof(unsigned)));
    }
    while (c.ev.size() < nev) {
        cudaEvent_t e;
        PG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c.ev.push_back(e);
        PG_CUDA(cudaEventCreate(&e));
        c.tev.push_back(e);
    }
    return c;
}

// Pageable host buffers (a reference DenseMatrix is a std::vector) cannot
// be DMA'd asynchronously: the driver would stage them synchronously at
// ~10 GB/s. Instead they go through library-owned pinned slots: a few host
// threads memcpy pageable <-> slot while the copy engine moves the previous
// slot, so the link still streams.
// cuStreamWaitValue32 (driver API, loaded at first use): a stream waits
// until a 32-bit word in device memory reaches a value
using WaitValueFn = int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
WaitValueFn wait_value_fn() {
    static WaitValueFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WaitValueFn>(p);
        else
            cudaGetLastError();
    });
    return fn;
}
constexpr unsigned kWaitValueGeq = 0;  // CU_STREAM_WAIT_VALUE_GEQ

__global__ void k_add_offset(const uint32_t* __restrict__ src, uint32_t n, uint32_t off, uint32_t* __restrict__ dst) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i] + off;
}

bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Streaming (non-temporal) copy for the staging pipeline: the destination is
// written without a read-for-ownership and without displacing the cache
// (the pinned slot is next read by the DMA engine; a downloaded row is not
// read back by this call), so each staged byte costs one host-memory read
// and one write instead of two reads and a write. $PG_STAGE_NT=0: memcpy.
void stream_copy(char* dst, const char* src, size_t n) {
    static const bool nt = [] {
        const char* e = std::getenv("PG_STAGE_NT");
        return !(e && std::atoi(e) == 0);
    }();
    if (!nt || n < 4096) {
        std::memcpy(dst, src, n);
        return;
    }
    const size_t head = (16 - reinterpret_cast<uintptr_t>(dst) % 16) % 16;
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
    const size_t body = n & ~size_t(63);
    for (size_t i = 0; i < body; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
        const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    std::memcpy(dst + body, src + body, n - body);
    _mm_sfence();  // the streamed bytes are globally visible before the DMA / the caller reads them
}

// memcpy split over a small persistent thread pool (the caller takes part)
class ParallelCopy {
public:
    explicit ParallelCopy(unsigned n) : nthreads_(n) {
        for (unsigned t = 1; t < n; ++t) workers_.emplace_back([this, t] { loop(t); });
    }
    ~ParallelCopy() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    void copy(void* dst, const void* src, size_t n) {
        if (n < (1u << 20) || nthreads_ == 1) {
            stream_copy(static_cast<char*>(dst), static_cast<const char*>(src), n);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            n_ = n;
            pending_ = nthreads_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [this] { return pending_ == 0; });
    }

private:
    void part(unsigned t) {
        const size_t per = ((n_ + nthreads_ - 1) / nthreads_ + 63) & ~size_t(63);  // ceil: parts cover all n_ bytes
        const size_t b = std::min(n_, per * t), e = std::min(n_, per * (t + 1));
        if (e > b) stream_copy(dst_ + b, src_ + b, e - b);
    }
    void loop(unsigned t) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            part(t);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    unsigned nthreads_;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t n_ = 0;
};

struct Staging {
    static constexpr size_t kSlot = 16u << 20;
    static constexpr int kSlots = 4;
    void* up[kSlots] = {};
    void* down[kSlots] = {};
    cudaEvent_t up_ev[kSlots] = {}, down_ev[kSlots] = {};
    std::unique_ptr<ParallelCopy> pc;
    std::mutex mu;  // one host call at a time per device uses the slots
};

Staging& staging(int device) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<Staging>> per_dev;
    std::lock_guard<std::mutex> lk(mu);
    if (static_cast<int>(per_dev.size()) <= device) per_dev.resize(device + 1);
    if (!per_dev[device]) {
        auto st = std::make_unique<Staging>();
        for (int i = 0; i < Staging::kSlots; ++i) {
            PG_CUDA(cudaHostAlloc(&st->up[i], Staging::kSlot, cudaHostAllocDefault));
            PG_CUDA(cudaHostAlloc(&st->down[i], Staging::kSlot, cudaHostAllocDefault));
            PG_CUDA(cudaEventCreateWithFlags(&st->up_ev[i], cudaEventDisableTiming));
            PG_CUDA(cudaEventCreateWithFlags(&st->down_ev[i], cudaEventDisableTiming));
        }
        const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
        // host copy threads: the calling thread is blocked in the call anyway;
        // 12-16 of the box's 16 cores measured best (Reddit layer 0 31 ms vs
        // 36 ms at 8, 41 ms at 4)
        const char* e = std::getenv("PG_STAGE_THREADS");
        const unsigned nt = e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : std::clamp(hc, 1u, 16u);
        st->pc = std::make_unique<ParallelCopy>(nt);
        per_dev[device] = std::move(st);
    }
    return *per_dev[device];
}

// H2D of n bytes from pageable src through the up slots on stream st
// (returns once the last piece is queued; the host part is done)
void staged_h2d(Staging& sg, void* dst, const void* src, size_t n, cudaStream_t st, int& slot) {
    for (size_t off = 0; off < n; off += Staging::kSlot) {
        const size_t len = std::min(Staging::kSlot, n - off);
        PG_CUDA(cudaEventSynchronize(sg.up_ev[slot]));  // the slot's previous DMA has read it
        sg.pc->copy(sg.up[slot], static_cast<const char*>(src) + off, len);
        PG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, sg.up[slot], len, cudaMemcpyHostToDevice, st));
        PG_CUDA(cudaEventRecord(sg.up_ev[slot], st));
        slot = (slot + 1) % Staging::kSlots;
    }
}

// D2H into pageable dst: pieces DMA'd to the down slots on stream st (after
// whatever st already waits for), each copied out by the host as soon as it
// lands while the next piece is in flight
struct StagedD2H {
    Staging& sg;
    cudaStream_t st;
    int slot = 0;
    struct Pending {
        int slot;
        char* dst;
        size_t len;
    };
    std::vector<Pending> q;
    void drain_one() {
        const Pending pd = q.front();
        q.erase(q.begin());
        PG_CUDA(cudaEventSynchronize(sg.down_ev[pd.slot]));
        sg.pc->copy(pd.dst, sg.down[pd.slot], pd.len);
    }
    void enqueue(void* dst, const void* src, size_t n) {
        for (size_t off = 0; off < n; off += Staging::kSlot) {
            const size_t len = std::min(Staging::kSlot, n - off);
            if (q.size() + 1 >= static_cast<size_t>(Staging::kSlots)) drain_one();  // keep one slot free
            PG_CUDA(cudaMemcpyAsync(sg.down[slot], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                    st));
            PG_CUDA(cudaEventRecord(sg.down_ev[slot], st));
            q.push_back({slot, static_cast<char*>(dst) + off, len});
            slot = (slot + 1) % Staging::kSlots;
        }
    }
    void finish() {
        while (!q.empty()) drain_one();
    }
};

// Host buffers (row-major, ld = dim) through a copy/compute pipeline:
//  * the input goes up in K source-row segments on the H2D stream (flat
//    copies at full link rate, then an on-device repack to 16-byte rows when
//    dim % 4 != 0); SpMM pass k (every destination, the edges whose source
//    row lies in segment k) starts as soon as segment k is resident. Edges
//    are sorted by source row within a destination, so running the
//    segments in order as accumulate passes is exactly the serial fp32 order;
//  * the last pass runs in R edge-balanced destination-row chunks, and each
//    chunk's rows go down on the D2H stream while the next chunk computes.
// K = tuning "host_segs" and R = "host_chunks" for path groupings above a
// size floor (1 and 1 otherwise); "host_trace" = 1 prints phase times.
void run_host(Groups& G, bool parent_indexed, const float* in_host, uint64_t in_rows, uint64_t dim,
              float* out_host, unsigned flags) {
    const auto t_entry = std::chrono::steady_clock::now();
    const Base b = base_of(G);
    std::lock_guard<std::recursive_mutex> lk(G.mu);  // caches stay put for the whole pipeline
    if (parent_indexed && G.edges_remap.get())
        fail(kConfig, "backward_aggregate_host: a multi-GPU source remap is installed on this grouping");
    DeviceGuard dg(G.device);
    cudaStream_t s = lib_stream(G.device);
    const bool packed = dim % 4 == 0;  // host rows are already 16-byte rows
    const uint64_t ld = (dim + 3) & ~3ull;
    const uint64_t D = b.D;
    DevBuf<float> fin(packed ? 0 : in_rows * dim, s), din(in_rows * ld, s);
    DevBuf<float> fout(packed ? 0 : D * dim, s), dout(D * ld, s);
    // pipelined (segments / chunks) above an output size floor (tuning
    // host_min_mb, MB of output rows)
    const uint64_t floor_mb = static_cast<uint64_t>(std::max<int64_t>(0, tuning(kTuneHostMinMb)));
    const bool big = G.path && D >= 16384 && dim * 4 * D >= (floor_mb << 20);
    // source segments re-read and re-write the output once per extra pass:
    // only when gathers dominate (E >= 64 D), like the device-side rule
    const uint32_t K = (big && parent_indexed && in_rows >= 4 && b.E >= 64ull * D)
                           ? static_cast<uint32_t>(std::clamp<int64_t>(tuning(kTuneHostSegs), 1, 8)) : 1;
    // below the floor, paths with >= 4 MB of output still overlap their D2H
    // with a few destination chunks (tuning host_small_chunks; no source
    // segments: the input is small)
    const bool small_pipe = !big && G.path && D >= 16384 && dim * 4 * D >= (4ull << 20) &&
                            tuning(kTuneHostSmallChunks) > 1;
    const uint32_t R = big ? static_cast<uint32_t>(std::clamp<int64_t>(tuning(kTuneHostChunks), 1, 16))
                       : small_pipe ? static_cast<uint32_t>(std::clamp<int64_t>(tuning(kTuneHostSmallChunks), 1, 16))
                                    : 1;
    // the last F segments form the chunked last pass (its D2H overlaps the
    // next chunk); the K - F before it are whole-row passes under the H2D
    const uint32_t F = static_cast<uint32_t>(std::clamp<int64_t>(tuning(kTuneHostFinalSegs), 1, K));
    const bool trace = tuning(kTuneHostTrace) != 0;
    // Source-row segments: equal rows, or (default) equal edges — frontier
    // order puts the hubs first (RMAT, power-law graphs), so equal-row
    // segments give the first pass most of the edges while only its small
    // slice of rows has arrived
    const int bal = K > 1 ? static_cast<int>(tuning(kTuneHostSegBalance) != 0) : 0;
    const int bal_key = bal ? (1 + static_cast<int>(tuning(kTuneHostLastSegPct))) * 16 + static_cast<int>(F) : 0;
    if (K > 1 && (G.host_seg_rows != in_rows || G.host_seg_k != K || G.host_seg_bal != bal_key)) {
        std::vector<uint64_t> rc(K + 1);
        for (uint32_t k = 0; k <= K; ++k) rc[k] = in_rows * k / K;
        if (bal) {
            DevBuf<uint32_t> cnt(in_rows, s);
            source_edge_counts(G.path->edges_parent.get(), b.E, in_rows, cnt.get(), s);
            std::vector<uint32_t> hc(in_rows);
            PG_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), in_rows * 4, cudaMemcpyDeviceToHost, s));
            PG_CUDA(cudaStreamSynchronize(s));
            // edge fraction of the last pass's F segments (host_last_seg_pct,
            // 0 = F/K), shared equally; the first K-F share the rest equally
            const int64_t pct = tuning(kTuneHostLastSegPct);
            const double last = pct > 0 ? std::clamp<double>(pct / 100.0, 0.01, 0.99) : static_cast<double>(F) / K;
            std::vector<double> tgt(K);
            for (uint32_t j = 1; j < K; ++j)
                tgt[j] = (j <= K - F ? (1.0 - last) * j / (K - F) : (1.0 - last) + last * (j - (K - F)) / F) *
                         static_cast<double>(b.E);
            uint64_t acc = 0, k = 1;
            for (uint64_t r = 0; r < in_rows && k < K; ++r) {
                acc += hc[r];
                while (k < K && static_cast<double>(acc) >= tgt[k]) rc[k++] = r + 1;
            }
            for (uint32_t j = 1; j <= K; ++j) rc[j] = std::max(rc[j], rc[j - 1]);
        }
        segment_bounds(G.path->offsets.get(), G.path->edges_parent.get(), static_cast<uint32_t>(D), rc.data(), K,
                       G.host_seg_bnd, s);
        G.host_seg_cuts = rc;
        G.host_seg_rows = in_rows;
        G.host_seg_k = K;
        G.host_seg_bal = bal_key;
    }
    std::vector<uint64_t> rcut = K > 1 ? G.host_seg_cuts : std::vector<uint64_t>{0, in_rows};
    std::vector<uint32_t> cuts{0, static_cast<uint32_t>(D)};
    if (R > 1) {
        // cut where alpha * (edges so far) + (1 - alpha) * (rows so far)
        // crosses r / R: edge-balanced chunks (alpha = 1) isolate the hub
        // rows (frontier order: hubs first) into tiny, latency-bound chunks
        const int alpha = static_cast<int>(std::clamp<int64_t>(tuning(kTuneHostChunkBalance), 0, 100));
        // the last chunk (computed first under the reverse order) at
        // host_first_chunk_pct % of the others: the first D2H starts sooner
        const int64_t fpct = std::clamp<int64_t>(tuning(kTuneHostFirstChunkPct), 10, 100);
        const int key = alpha * 1000 + static_cast<int>(fpct);
        if (G.host_chunks.size() != R + 1 || G.host_chunk_alpha != key) {
            std::vector<uint64_t> off(D + 1);
            PG_CUDA(cudaMemcpyAsync(off.data(), G.path->offsets.get(), off.size() * 8, cudaMemcpyDeviceToHost, s));
            PG_CUDA(cudaStreamSynchronize(s));
            G.host_chunks.assign(1, 0);
            const double E = std::max<double>(1.0, static_cast<double>(off[D]));
            const double total = (R - 1) + fpct / 100.0;
            uint64_t row = 0;
            for (uint32_t r = 1; r < R; ++r) {
                const double target = static_cast<double>(r) / total;
                while (row < D && (alpha * (off[row] / E) + (100 - alpha) * (static_cast<double>(row) / D)) / 100.0 <
                                      target)
                    ++row;
                G.host_chunks.push_back(std::max(G.host_chunks.back(), static_cast<uint32_t>(row)));
            }
            G.host_chunks.push_back(static_cast<uint32_t>(D));
            G.host_chunk_alpha = key;
        }
        cuts = G.host_chunks;
    }
    std::unique_lock<std::mutex> cs_lock;
    // sync events: 1 + K + R + 1 used; trace events: up to 1 + K + (K - F)
    // + 2 R (start, uploads, whole passes, chunks, downloads)
    CopyStreams& cs = copy_streams(G.device, 4 + 2 * K + 3 * R, cs_lock);
    size_t nt = 0;  // trace events used
    auto mark = [&](cudaStream_t st) {
        if (trace && nt < cs.tev.size()) PG_CUDA(cudaEventRecord(cs.tev[nt++], st));
    };
    std::vector<std::string> tname;
    auto tmark = [&](cudaStream_t st, std::string name) {
        if (!trace) return;
        tname.push_back(std::move(name));
        mark(st);
    };
    tmark(s, "start");
    // the (h2d, d2h) streams join s's prior work
    PG_CUDA(cudaEventRecord(cs.ev[0], s));
    PG_CUDA(cudaStreamWaitEvent(cs.h2d, cs.ev[0], 0));
    PG_CUDA(cudaStreamWaitEvent(cs.d2h, cs.ev[0], 0));
    // pageable host buffers go through the pinned staging slots
    const bool in_pg = dim && in_rows && !host_pinned(in_host);
    const bool out_pg = dim && D && !host_pinned(out_host);
    Staging* sg = (in_pg || out_pg) ? &staging(G.device) : nullptr;
    std::unique_lock<std::mutex> sg_lock;
    if (sg) sg_lock = std::unique_lock<std::mutex>(sg->mu);
    int up_slot = 0;
    auto upload = [&](void* dst, const void* src, size_t n, bool pageable) {
        if (pageable)
            staged_h2d(*sg, dst, src, n, cs.h2d, up_slot);
        else
            PG_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, cs.h2d));
    };
    // pinned rows of width dim go straight into the 16-byte-pitched device
    // rows with a 2-D copy: a repack kernel on the copy stream would queue
    // behind the SpMM's blocks and hold the segment back until the pass ends
    const bool pitch2d = !packed && tuning(kTuneHostPitch2d) != 0;
    // returns the stream the rows are ready on (h2d, or rup after the repack
    // when `split`: the next segment's DMA does not wait for this repack)
    auto upload_rows = [&](float* dst_pitched, float* dst_flat, const float* src, uint64_t rows, bool pageable,
                           cudaEvent_t copied, bool split) -> cudaStream_t {
        if (!rows) return cs.h2d;
        if (packed) {
            upload(dst_pitched, src, rows * dim * 4, pageable);
        } else if (pitch2d && !pageable) {
            PG_CUDA(cudaMemcpy2DAsync(dst_pitched, ld * 4, src, dim * 4, dim * 4, rows, cudaMemcpyHostToDevice,
                                      cs.h2d));
        } else {
            upload(dst_flat, src, rows * dim * 4, pageable);
            if (!split) {
                copy_rows(dst_flat, dim, dst_pitched, ld, rows, dim, cs.h2d);
                return cs.h2d;
            }
            PG_CUDA(cudaEventRecord(copied, cs.h2d));
            PG_CUDA(cudaStreamWaitEvent(cs.rup, copied, 0));
            copy_rows(dst_flat, dim, dst_pitched, ld, rows, dim, cs.rup);
            return cs.rup;
        }
        return cs.h2d;
    };
    if (D && dim && !(flags & PG_AGG_OVERWRITE))  // accumulate: current output goes up first
        upload_rows(dout.get(), fout.get(), out_host, D, out_pg, nullptr, false);
    // extra sync events after the 2 + K + R of the pipeline: segment k's
    // flat copy done (before its repack), chunk r repacked (before its D2H)
    cudaEvent_t* ev_copied = cs.ev.data() + 2 + K + R;
    cudaEvent_t* ev_packed = cs.ev.data() + 2 + 2 * K + R;
    // trace events on rup/rdn are not needed: the pass / D2H marks follow them
    // segment k up, then pass k (every destination, segment k's edges) for
    // the K - F segments before the chunked last pass
    for (uint32_t k = 0; k < K; ++k) {
        const uint64_t r0 = rcut[k], r1 = rcut[k + 1];
        cudaStream_t ready = cs.h2d;
        if (r1 > r0 && dim)
            ready = upload_rows(din.get() + r0 * ld, fin.get() + r0 * dim, in_host + r0 * dim, r1 - r0, in_pg,
                                ev_copied[k], true);
        PG_CUDA(cudaEventRecord(cs.ev[1 + k], ready));
        tmark(cs.h2d, "h2d" + std::to_string(k));
        if (k + F < K) {
            PG_CUDA(cudaStreamWaitEvent(s, cs.ev[1 + k], 0));
            run_aggregate(G, parent_indexed, 0, static_cast<uint32_t>(D), din.get(), ld, dout.get(), ld, dim,
                          k == 0 ? flags : (flags & ~PG_AGG_OVERWRITE), s,
                          SegSel{G.host_seg_bnd.get(), static_cast<int>(k), K});
            tmark(s, "pass" + std::to_string(k));
        }
    }
    PG_CUDA(cudaStreamWaitEvent(s, cs.ev[K], 0));
    const unsigned last_flags = K > F ? (flags & ~PG_AGG_OVERWRITE) : flags;
    const SegSel last =
        K > 1 ? SegSel{G.host_seg_bnd.get(), static_cast<int>(K - F), K, static_cast<int>(K)} : SegSel{};
    // Chunks are edge-balanced, so in destination order (hubs first) the
    // first chunks hold few rows and the last hold most of them: run them
    // last-first (tuning "host_chunk_order" = 1, default) so the big D2H
    // copies start early and the tail after the final chunk is a small one.
    // Every chunk is queued before any D2H, so a host that blocks on a
    // staged (pageable) download never starves the SpMM stream.
    const bool reverse = tuning(kTuneHostChunkOrder) == 1;
    // Hub split (tuning "host_hub_chunk_side" = 1): the hub prefix of every
    // chunk's degree order (latency-bound chains, a handful of small CTAs on
    // the side kernel) goes first on its own stream; the rest of each chunk
    // runs on s. A chunk's D2H waits for its own part on s and, only when it
    // has hubs, for its hub part. The chunks without hubs (the low-degree
    // tail, copied first) no longer queue behind the hub chains, and the hub
    // chunk is finished long before its turn in the D2H order.
    // Mode 2: the whole hub chunk (chunk 0) on its own stream instead.
    const int hub_mode = reverse && cuts.size() > 2 ? static_cast<int>(tuning(kTuneHostHubChunkSide)) : 0;
    std::vector<uint32_t> nh(cuts.size() - 1, 0);
    bool any_hub = false;
    const uint64_t hub_min = static_cast<uint64_t>(std::max<int64_t>(1, tuning(kTuneHostHubMin)));
    if (hub_mode == 1) {
        for (size_t r = 0; r + 1 < cuts.size(); ++r) {
            if (cuts[r] == cuts[r + 1]) continue;
            nh[r] = range_heavy(G, cuts[r], cuts[r + 1], hub_min);
            any_hub |= nh[r] > 0;
        }
    }
    cudaEvent_t* ev_hub = cs.ev.data() + 2 + 2 * K + 2 * R;  // per chunk: its hub part done
    if (any_hub || hub_mode == 2) {
        PG_CUDA(cudaEventRecord(cs.ev[0], s));
        PG_CUDA(cudaStreamWaitEvent(cs.hub, cs.ev[0], 0));
    }
    if (any_hub) {
        for (size_t r = 0; r + 1 < cuts.size(); ++r) {  // destination order: the real hubs first
            if (!nh[r]) continue;
            AggExt hx;
            hx.part = 1;
            hx.part_min_degree = hub_min;
            run_aggregate(G, parent_indexed, cuts[r], cuts[r + 1], din.get(), ld, dout.get() + cuts[r] * ld, ld, dim,
                          last_flags, cs.hub, last, hx);
            PG_CUDA(cudaEventRecord(ev_hub[r], cs.hub));
        }
        tmark(cs.hub, "hubs");
    } else if (hub_mode == 2 && cuts[0] < cuts[1]) {
        run_aggregate(G, parent_indexed, cuts[0], cuts[1], din.get(), ld, dout.get(), ld, dim, last_flags, cs.hub,
                      last);
        PG_CUDA(cudaEventRecord(cs.ev[1 + K], cs.hub));
        tmark(cs.hub, "chunk0");
    }
    // Sequenced last pass (tuning "host_seq"): ONE launch over every chunk,
    // each finished item counted per chunk; chunk r's D2H stream waits on its
    // counter (cuStreamWaitValue32) instead of a per-chunk launch boundary.
    // Run order below: the first chunk of the D2H order, chunk 0's hub front,
    // the other chunks in D2H order, chunk 0's rest.
    const uint32_t nq_h = static_cast<uint32_t>((dim + 3) / 4);
    const bool seq = tuning(kTuneHostSeq) != 0 && reverse && R > 1 && (K == 1 || F == 1) && hub_mode == 0 &&
                     nq_h > 16 && !row_kernel_on(dim) && wait_value_fn() && ld % 4 == 0 && G.path;
    DevBuf<uint32_t> seq_dlist;
    unsigned* seq_counters = nullptr;
    bool seq_side_hubs = false;
    std::vector<uint32_t> seq_target(cuts.size() - 1, 0);
    std::vector<size_t> order;
    if (seq) {
        const uint32_t nrc = static_cast<uint32_t>(cuts.size() - 1);
        const uint32_t chunks = (nq_h + 31) / 32;
        seq_dlist = DevBuf<uint32_t>(D, s);
        seq_counters = cs.counters;  // R <= 16 <= 64
        PG_CUDA(cudaMemsetAsync(seq_counters, 0, nrc * sizeof(unsigned), s));
        // the waiting streams must see THIS call's zeroed counters, not the
        // final counts a previous call of the same shape left behind
        PG_CUDA(cudaEventRecord(cs.ev[0], s));
        PG_CUDA(cudaStreamWaitEvent(cs.rdn, cs.ev[0], 0));
        PG_CUDA(cudaStreamWaitEvent(cs.d2h, cs.ev[0], 0));
        const uint64_t rdiv = K > 1 ? K : 1;  // the last pass covers one of K segments
        SeqTable tab;
        std::vector<uint32_t> dofs(nrc, 0);
        uint32_t pos = 0, nh0 = 0;
        uint64_t thr0 = 0;
        auto put = [&](uint32_t r) {  // chunk r's degree-ordered rows, absolute ids
            Groups::RowSched* rs = row_sched(G, cuts[r], cuts[r + 1]);
            const uint32_t nd = cuts[r + 1] - cuts[r];
            k_add_offset<<<(nd + 255) / 256, 256, 0, s>>>(rs->order.get(), nd, cuts[r], seq_dlist.get() + pos);
            PG_LAUNCH("k_add_offset");
            dofs[r] = pos;
            pos += nd;
            if (r == 0) {
                thr0 = heavy_degree(dim, rs->hist.edges / rdiv);
                nh0 = std::min(nd, rs->hist.heavy(thr0));
            }
        };
        for (uint32_t r = 0; r < nrc; ++r)
            if (cuts[r] < cuts[r + 1]) put(r);
        uint64_t item = 0;
        // runs start on CTA boundaries (8 items): a CTA marks its items done
        // together, so a run sharing a CTA with the next one (a hub chain)
        // would wait for it; the padding items do nothing
        auto run = [&](uint32_t r, uint32_t off, uint32_t nd, uint32_t dest_major) {
            if (!nd) return;
            tab.seg[tab.nseg++] = SeqSeg{item, nd, dofs[r] + off, dest_major, r};
            item += (static_cast<uint64_t>(nd) * chunks + 7) & ~7ull;
        };
        // the first chunk of the D2H order first (the copies start as soon
        // as possible), then the hub front (its chains have until chunk 0's
        // turn), then the other chunks in D2H order, then chunk 0's rest.
        // host_seq 2: chunk 0's hubs on the side kernel (deeper-pipelined
        // chains, a few small CTAs) on the hub stream instead of the front.
        seq_side_hubs = tuning(kTuneHostSeq) == 2 && nh0 > 0;
        uint32_t first = nrc - 1;
        while (first > 0 && cuts[first] == cuts[first + 1]) --first;
        if (seq_side_hubs) {
            PG_CUDA(cudaEventRecord(cs.ev[0], s));
            PG_CUDA(cudaStreamWaitEvent(cs.hub, cs.ev[0], 0));
            AggExt hx;
            hx.part = 1;
            hx.part_min_degree = thr0;
            run_aggregate(G, parent_indexed, cuts[0], cuts[1], din.get(), ld, dout.get(), ld, dim, last_flags, cs.hub,
                          last, hx);
            PG_CUDA(cudaEventRecord(ev_hub[0], cs.hub));
        }
        if (first > 0) run(first, 0, cuts[first + 1] - cuts[first], 0);
        if (cuts[0] < cuts[1] && !seq_side_hubs) run(0, 0, nh0, 1);  // the hub front
        for (uint32_t r = first; r-- > 1;) {
            if (cuts[r] == cuts[r + 1]) continue;
            run(r, 0, cuts[r + 1] - cuts[r], 0);
        }
        if (cuts[0] < cuts[1]) run(0, nh0, cuts[1] - cuts[0] - nh0, 0);
        for (uint32_t r = 0; r < nrc; ++r) seq_target[r] = (cuts[r + 1] - cuts[r]) * chunks;
        if (seq_side_hubs) seq_target[0] -= nh0 * chunks;
        const uint64_t* eb = K > 1 ? G.host_seg_bnd.get() + static_cast<uint64_t>(K - 1) * D : G.path->offsets.get();
        const uint64_t* ee = K > 1 ? G.host_seg_bnd.get() + static_cast<uint64_t>(K) * D : G.path->offsets.get() + 1;
        aggregate_seq(eb, ee, G.path->edges_parent.get(), seq_dlist.get(), tab, item, chunks, din.get(), ld, dout.get(),
                      ld, static_cast<uint32_t>(dim), !(last_flags & PG_AGG_OVERWRITE), seq_counters, s);
        tmark(s, "seqpass");
        for (size_t ri = 0; ri + 1 < cuts.size(); ++ri) {
            const size_t r = cuts.size() - 2 - ri;
            if (cuts[r] < cuts[r + 1]) order.push_back(r);
        }
    }
    for (size_t ri = 0; !seq && ri + 1 < cuts.size(); ++ri) {
        const size_t r = reverse ? cuts.size() - 2 - ri : ri;
        if (cuts[r] == cuts[r + 1]) continue;
        order.push_back(r);
        if (hub_mode == 2 && !any_hub && r == 0) continue;
        AggExt cx;
        cx.part = any_hub && nh[r] ? 2 : 0;
        cx.part_min_degree = hub_min;
        if (K > 1 && F > 1) {
            // the chunk's F final segments one by one, in source order: each
            // launch gathers from one segment's rows (L2-sized when K is)
            for (uint32_t k = K - F; k < K; ++k)
                run_aggregate(G, parent_indexed, cuts[r], cuts[r + 1], din.get(), ld, dout.get() + cuts[r] * ld, ld,
                              dim, k == K - F ? last_flags : (last_flags & ~PG_AGG_OVERWRITE), s,
                              SegSel{G.host_seg_bnd.get(), static_cast<int>(k), K}, cx);
        } else {
            run_aggregate(G, parent_indexed, cuts[r], cuts[r + 1], din.get(), ld, dout.get() + cuts[r] * ld, ld, dim,
                          last_flags, s, last, cx);
        }
        PG_CUDA(cudaEventRecord(cs.ev[1 + K + r], s));
        tmark(s, "chunk" + std::to_string(r));
    }
    if (any_hub || hub_mode == 2 || seq_side_hubs) {  // s joins the hub stream (buffers are freed on s)
        PG_CUDA(cudaEventRecord(cs.ev[0], cs.hub));
        PG_CUDA(cudaStreamWaitEvent(s, cs.ev[0], 0));
    }
    std::unique_ptr<StagedD2H> down;
    if (out_pg) down = std::make_unique<StagedD2H>(StagedD2H{*sg, cs.d2h});
    for (const size_t r : order) {
        const uint32_t rb = cuts[r], re = cuts[r + 1];
        if (seq) {  // the chunk's items all counted: its rows are final
            cudaStream_t w = packed || (pitch2d && !down) ? cs.d2h : cs.rdn;
            const int rc = wait_value_fn()(w, reinterpret_cast<unsigned long long>(seq_counters + r), seq_target[r],
                                           kWaitValueGeq);
            if (rc != 0) fail(kDevice, "cuStreamWaitValue32 failed (CUresult " + std::to_string(rc) + ")");
            tmark(w, "rdy" + std::to_string(r));
            if (seq_side_hubs && r == 0) {  // and chunk 0's hub rows from the hub stream
                PG_CUDA(cudaStreamWaitEvent(cs.d2h, ev_hub[0], 0));
                PG_CUDA(cudaStreamWaitEvent(cs.rdn, ev_hub[0], 0));
            }
        } else {
            PG_CUDA(cudaStreamWaitEvent(cs.d2h, cs.ev[1 + K + r], 0));
        }
        if (any_hub && nh[r]) {  // the chunk's hub rows come from the hub stream
            PG_CUDA(cudaStreamWaitEvent(cs.d2h, ev_hub[r], 0));
            PG_CUDA(cudaStreamWaitEvent(cs.rdn, ev_hub[r], 0));
        }
        if (!dim) continue;
        const float* src = dout.get() + rb * ld;
        if (!packed && pitch2d && !down) {
            PG_CUDA(cudaMemcpy2DAsync(out_host + rb * dim, dim * 4, src, ld * 4, dim * 4, re - rb,
                                      cudaMemcpyDeviceToHost, cs.d2h));
            tmark(cs.d2h, "d2h" + std::to_string(r));
            continue;
        }
        if (!packed) {
            // repack on rdn (waits for the chunk), the D2H stream waits for
            // the repack: chunk r+1's repack overlaps chunk r's DMA
            if (!seq) PG_CUDA(cudaStreamWaitEvent(cs.rdn, cs.ev[1 + K + r], 0));
            copy_rows(dout.get() + rb * ld, ld, fout.get() + rb * dim, dim, re - rb, dim, cs.rdn);
            PG_CUDA(cudaEventRecord(ev_packed[r], cs.rdn));
            PG_CUDA(cudaStreamWaitEvent(cs.d2h, ev_packed[r], 0));
            src = fout.get() + rb * dim;
        }
        if (down)
            down->enqueue(out_host + rb * dim, src, (re - rb) * dim * 4);
        else
            PG_CUDA(cudaMemcpyAsync(out_host + rb * dim, src, (re - rb) * dim * 4, cudaMemcpyDeviceToHost, cs.d2h));
        tmark(cs.d2h, "d2h" + std::to_string(r));
    }
    if (down) down->finish();
    // buffers are freed stream-ordered on s: s waits for both copy streams
    PG_CUDA(cudaEventRecord(cs.ev[1 + K + R], cs.d2h));
    PG_CUDA(cudaStreamWaitEvent(s, cs.ev[1 + K + R], 0));
    const auto t_queued = std::chrono::steady_clock::now();
    PG_CUDA(cudaStreamSynchronize(s));
    if (trace) {
        const auto t_done = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        char wb[96];
        std::snprintf(wb, sizeof(wb), " host: queued=%.2f wall=%.2f |", ms(t_entry, t_queued), ms(t_entry, t_done));
        std::string line = "[host_trace] D=" + std::to_string(D) + " dim=" + std::to_string(dim) +
                           " K=" + std::to_string(K) + " F=" + std::to_string(F) + " R=" + std::to_string(R) + ":" +
                           wb;
        for (size_t i = 1; i < nt; ++i) {
            float ms = 0.f;
            PG_CUDA(cudaEventElapsedTime(&ms, cs.tev[0], cs.tev[i]));
            char buf[64];
            std::snprintf(buf, sizeof(buf), " %s=%.2f", tname[i].c_str(), ms);
            line += buf;
        }
        std::fprintf(stderr, "%s\n", line.c_str());
    }
}

}  // namespace

extern "C" {

int pg_last_error(char* buf, size_t cap) {
    if (buf && cap) std::snprintf(buf, cap, "%s", g_err.c_str());
    return static_cast<int>(g_err.size());
}

int pg_last_error_kind(uint64_t* line) {
    if (line) *line = g_line;
    return g_kind;
}

int pg_version(void) { return 2; }

int pg_set_heavy_min_degree(uint64_t min_degree) {
    return guard([&] { set_heavy_min_degree(min_degree); });
}

int pg_set_tuning(const char* key, int64_t value) {
    return guard([&] {
        if (!key || !set_tuning(key, value)) fail(kConfig, std::string("pg_set_tuning: unknown key ") + (key ? key : "(null)"));
    });
}

int pg_device_count(int* count) {
    return guard([&] {
        int c = 0;
        PG_CUDA(cudaGetDeviceCount(&c));
        *count = c;
    });
}

// ---------------- graph load ----------------

int pg_gen_rmat(uint32_t n, uint64_t m, double a, double b, double c, double d, uint64_t seed, uint32_t* pairs,
                uint32_t* n_pad) {
    return guard([&] {
        // rmat.cpp:10-44: pad n to 2^levels; per pair and level one
        // U(0,1) draw from mt19937_64(seed) picks the quadrant.
        if (n == 0) fail(kConfig, "rmat: vertex count must be positive");
        if (std::abs(a + b + c + d - 1.0) > 1e-9) fail(kConfig, "rmat: quadrant probabilities must sum to 1");
        int levels = 0;
        while ((uint32_t{1} << levels) < n) ++levels;
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unit(0.0, 1.0);
        for (uint64_t i = 0; i < m; ++i) {
            uint32_t src = 0, dst = 0;
            for (int lvl = levels - 1; lvl >= 0; --lvl) {
                const double r = unit(rng);
                const uint32_t bit = uint32_t{1} << lvl;
                if (r < a) {
                } else if (r < a + b) {
                    dst |= bit;
                } else if (r < a + b + c) {
                    src |= bit;
                } else {
                    src |= bit;
                    dst |= bit;
                }
            }
            pairs[2 * i] = src;
            pairs[2 * i + 1] = dst;
        }
        if (n_pad) *n_pad = uint32_t{1} << levels;
    });
}

int pg_training_set_size(uint32_t n, double ratio, uint64_t* k) {
    return guard([&] {
        if (n == 0) fail(kConfig, "training set: graph has no vertices");
        if (!(ratio > 0.0) || ratio > 1.0) fail(kConfig, "training ratio must be in (0, 1]");
        *k = std::max<uint64_t>(1, static_cast<uint64_t>(std::llround(ratio * static_cast<double>(n))));
    });
}

int pg_sample_training_set(uint32_t n, double ratio, uint64_t seed, uint32_t* out) {
    return guard([&] {
        // training_set.cpp:28-49: partial Fisher-Yates over mt19937_64(seed)
        uint64_t k = 0;
        if (int rc = pg_training_set_size(n, ratio, &k)) fail(rc, g_err);
        std::vector<uint32_t> ids(n);
        std::iota(ids.begin(), ids.end(), 0u);
        std::mt19937_64 rng(seed);
        for (std::size_t i = 0; i < k; ++i) {
            std::uniform_int_distribution<std::size_t> pick(i, n - 1);
            std::swap(ids[i], ids[pick(rng)]);
        }
        std::sort(ids.begin(), ids.begin() + static_cast<std::ptrdiff_t>(k));
        std::memcpy(out, ids.data(), k * 4);
    });
}

int pg_graph_build(int device, int64_t n_hint, const uint32_t* pairs, uint64_t npairs, int weight_mode,
                   pg_graph* out) {
    return guard([&] {
        auto g = graph_build(device, n_hint, pairs, npairs, weight_mode);
        *out = reinterpret_cast<pg_graph>(g.release());
    });
}

int pg_edge_list_load(const char* path, pg_edge_list* out) {
    return guard([&] {
        if (!out) fail(kConfig, "edge_list_load: null output handle");
        auto el = std::make_unique<EdgeListData>(load_edge_list(path));
        *out = reinterpret_cast<pg_edge_list>(el.release());
    });
}

int pg_edge_list_info(pg_edge_list h, uint64_t* npairs, uint64_t* self_loops_dropped) {
    return guard([&] {
        auto* el = need(reinterpret_cast<EdgeListData*>(h), "edge list");
        if (npairs) *npairs = el->pairs.size() / 2;
        if (self_loops_dropped) *self_loops_dropped = el->self_loops;
    });
}

int pg_edge_list_export(pg_edge_list h, uint32_t* pairs) {
    return guard([&] {
        auto* el = need(reinterpret_cast<EdgeListData*>(h), "edge list");
        if (!el->pairs.empty()) std::memcpy(pairs, el->pairs.data(), el->pairs.size() * 4);
    });
}

int pg_edge_list_destroy(pg_edge_list h) {
    delete reinterpret_cast<EdgeListData*>(h);
    return PG_OK;
}

int pg_edge_list_write(const char* path, const uint32_t* pairs, uint64_t npairs) {
    return guard([&] { write_edge_list(path, pairs, npairs); });
}

int pg_graph_load_file(int device, const char* path, int weight_mode, pg_graph* out) {
    return guard([&] {
        const EdgeListData el = load_edge_list(path);
        auto g = graph_build(device, -1, el.pairs.data(), el.pairs.size() / 2, weight_mode);
        *out = reinterpret_cast<pg_graph>(g.release());
    });
}

int pg_training_set_load(const char* path, uint32_t n, uint32_t* out, uint64_t cap, uint64_t* k) {
    return guard([&] {
        const std::vector<uint32_t> vt = load_training_set(path, n);
        if (k) *k = vt.size();
        if (!out) return;
        if (cap < vt.size()) fail(kConfig, "training_set_load: output capacity too small");
        std::memcpy(out, vt.data(), vt.size() * 4);
    });
}

int pg_training_set_write(const char* path, const uint32_t* vt, uint64_t k) {
    return guard([&] { write_training_set(path, vt, k); });
}

int pg_graph_create(int device, uint32_t n, const uint64_t* offsets, const uint32_t* neighbors,
                    const double* weights, int validate, pg_graph* out) {
    return guard([&] {
        if (!offsets) fail(kConfig, "graph: offsets required");
        auto g = graph_upload(device, n, offsets, neighbors, weights, validate != 0);
        *out = reinterpret_cast<pg_graph>(g.release());
    });
}

int pg_graph_assign_weights(pg_graph h, int weight_mode) {
    return guard([&] {
        Graph& g = *G_(h);
        DeviceGuard dg(g.device);
        graph_assign_weights(g, weight_mode, lib_stream(g.device));
        PG_CUDA(cudaStreamSynchronize(lib_stream(g.device)));
    });
}

int pg_graph_info(pg_graph h, uint32_t* n, uint64_t* m, uint32_t* max_degree, uint64_t* fingerprint) {
    return guard([&] {
        Graph& g = *G_(h);
        if (n) *n = g.n;
        if (m) *m = g.m;
        if (max_degree) *max_degree = g.max_degree;
        if (fingerprint) *fingerprint = graph_fp(g);
    });
}

int pg_graph_export(pg_graph h, uint64_t* offsets, uint32_t* neighbors, double* weights) {
    return guard([&] {
        Graph& g = *G_(h);
        DeviceGuard dg(g.device);
        cudaStream_t s = lib_stream(g.device);
        if (offsets)
            PG_CUDA(cudaMemcpyAsync(offsets, g.offsets.get(), (static_cast<uint64_t>(g.n) + 1) * 8,
                                    cudaMemcpyDeviceToHost, s));
        if (neighbors && g.m) PG_CUDA(cudaMemcpyAsync(neighbors, g.nbrs.get(), g.m * 4, cudaMemcpyDeviceToHost, s));
        if (weights && g.m) PG_CUDA(cudaMemcpyAsync(weights, g.w64.get(), g.m * 8, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
    });
}

int pg_graph_destroy(pg_graph h) {
    return guard([&] {
        Graph* g = reinterpret_cast<Graph*>(h);
        if (!g) return;
        DeviceGuard dg(g->device);
        drain_device();  // kernels on caller streams may still read its buffers
        delete g;
    });
}

int pg_path_fingerprint(pg_graph h, const uint32_t* vt, uint64_t k, uint64_t layers, uint64_t* fp) {
    return guard([&] {
        // execution_path.cpp:17-22
        uint64_t x = graph_fp(*G_(h));
        x ^= training_fp(vt, k) + 0x9e3779b97f4a7c15ull + (x << 6) + (x >> 2);
        x ^= layers + 0x9e3779b97f4a7c15ull + (x << 6) + (x >> 2);
        *fp = x;
    });
}

// ---------------- execution-path build ----------------

int pg_frontiers_compute(pg_graph h, const uint32_t* vt, uint64_t k, uint64_t layers, pg_frontiers* out) {
    return guard([&] {
        auto f = frontiers_compute(*G_(h), vt, k, layers);
        *out = reinterpret_cast<pg_frontiers>(f.release());
    });
}

int pg_frontiers_size(pg_frontiers h, uint64_t level, uint64_t* size) {
    return guard([&] {
        Frontiers& f = *F_(h);
        if (level > f.L) fail(kConfig, "frontiers: level out of range");
        *size = f.levels[level].size;
    });
}

int pg_frontiers_export(pg_frontiers h, uint64_t level, uint32_t* out) {
    return guard([&] {
        Frontiers& f = *F_(h);
        if (level > f.L) fail(kConfig, "frontiers: level out of range");
        const Level& lv = f.levels[level];
        DeviceGuard dg(f.device);
        cudaStream_t s = lib_stream(f.device);
        if (lv.size) PG_CUDA(cudaMemcpyAsync(out, lv.ids.get(), lv.size * 4, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
    });
}

int pg_frontiers_destroy(pg_frontiers h) {
    return guard([&] {
        Frontiers* f = reinterpret_cast<Frontiers*>(h);
        if (!f) return;
        DeviceGuard dg(f->device);
        drain_device();  // kernels on caller streams may still read its buffers
        delete f;
    });
}

int pg_path_extract(pg_graph g, pg_frontiers f, uint64_t layer, pg_path* out) {
    return guard([&] {
        auto p = path_extract(*G_(g), *F_(f), layer);
        *out = reinterpret_cast<pg_path>(p.release());
    });
}

int pg_path_info(pg_path h, uint64_t* layer, uint32_t* dests, uint32_t* srcs, uint64_t* edges,
                 uint32_t* parent_rows, uint32_t* max_degree) {
    return guard([&] {
        Path& p = *P_(h);
        if (layer) *layer = p.layer;
        if (dests) *dests = p.D;
        if (srcs) *srcs = p.S;
        if (edges) *edges = p.E;
        if (parent_rows) *parent_rows = p.P;
        if (max_degree) *max_degree = p.max_degree;
    });
}

int pg_path_export(pg_path h, uint32_t* dest, uint32_t* src, uint32_t* srcpos, uint64_t* offsets,
                   uint32_t* neighbors, double* weights) {
    return guard([&] {
        Path& p = *P_(h);
        DeviceGuard dg(p.device);
        cudaStream_t s = lib_stream(p.device);
        auto cp = [&](void* dst, const void* srcp, uint64_t bytes) {
            if (dst && bytes) PG_CUDA(cudaMemcpyAsync(dst, srcp, bytes, cudaMemcpyDeviceToHost, s));
        };
        cp(dest, p.dest.get(), static_cast<uint64_t>(p.D) * 4);
        cp(src, p.src.get(), static_cast<uint64_t>(p.S) * 4);
        cp(srcpos, p.srcpos.get(), static_cast<uint64_t>(p.S) * 4);
        cp(offsets, p.offsets.get(), (static_cast<uint64_t>(p.D) + 1) * 8);
        cp(neighbors, p.nbr_local.get(), p.E * 4);
        cp(weights, p.w64.get(), p.E * 8);
        PG_CUDA(cudaStreamSynchronize(s));
    });
}

int pg_path_set_fingerprint(pg_path h, uint64_t fp) {
    return guard([&] { P_(h)->fingerprint = fp; });
}

int pg_path_get_fingerprint(pg_path h, uint64_t* fp) {
    return guard([&] { *fp = P_(h)->fingerprint; });
}

int pg_path_destroy(pg_path h) {
    return guard([&] {
        Path* p = reinterpret_cast<Path*>(h);
        if (!p) return;
        DeviceGuard dg(p->device);
        drain_device();  // kernels on caller streams may still read its buffers
        delete p;
    });
}

int pg_path_device_arrays(pg_path h, const uint32_t** dest, const uint32_t** srcpos, const uint64_t** offsets) {
    return guard([&] {
        Path& p = *P_(h);
        if (dest) *dest = p.dest.get();
        if (srcpos) *srcpos = p.srcpos.get();
        if (offsets) *offsets = p.offsets.get();
    });
}

// ---------------- group partition ----------------

int pg_gs_regression_stats(uint32_t n_vertices, uint64_t n_edges, double avg_degree, const double* beta,
                           uint32_t* gs) {
    return guard([&] {
        // gs_model.cpp:64-74
        const double b0 = beta ? beta[0] : 0.65538, b1 = beta ? beta[1] : 1.67431e-5;
        const double b2 = beta ? beta[2] : -2.24342e-6, b3 = beta ? beta[3] : 0.63641;
        const double raw = b0 + b1 * static_cast<double>(n_vertices) + b2 * static_cast<double>(n_edges) +
                           b3 * avg_degree;
        const long long rounded = std::llround(raw);
        *gs = rounded < 1 ? 1u : static_cast<uint32_t>(rounded);
    });
}

int pg_gs_regression(pg_path h, const double* beta, uint32_t* gs) {
    return guard([&] {
        // train.hpp:16-24 path_stats
        Path& p = *P_(h);
        const double avg = p.D == 0 ? 0.0 : static_cast<double>(p.E) / static_cast<double>(p.D);
        if (int rc = pg_gs_regression_stats(p.D, p.E, avg, beta, gs)) fail(rc, g_err);
    });
}

int pg_gs_default_candidates(uint32_t max_degree, uint32_t* out, uint64_t* count) {
    return guard([&] {
        // group_cost.cpp:30-34
        uint64_t c = 0;
        out[c++] = 1;
        while (out[c - 1] < std::max<uint32_t>(max_degree, 1)) {
            out[c] = out[c - 1] * 2;
            ++c;
        }
        *count = c;
    });
}

int pg_gs_oracle_cost(pg_path h, uint64_t dim, int workers, double lambda, const uint32_t* cands,
                      uint64_t ncand, uint32_t* best, double* table, uint64_t* ncand_out) {
    return guard([&] {
        // group_cost.cpp:36-53 over cost_model_evaluator (:26-28)
        Path& p = *P_(h);
        std::vector<uint32_t> c;
        if (cands) {
            c.assign(cands, cands + ncand);
        } else {
            uint32_t tmp[40];
            uint64_t k = 0;
            if (int rc = pg_gs_default_candidates(p.max_degree, tmp, &k)) fail(rc, g_err);
            c.assign(tmp, tmp + k);
        }
        if (c.empty()) fail(kConfig, "oracle_gs: empty candidate list");
        if (workers < 1) fail(kConfig, "cost model: worker count must be >= 1");
        DeviceGuard dg(p.device);
        cudaStream_t s = lib_stream(p.device);
        double best_cost = 0.0;
        uint32_t best_gs = 1;
        bool first = true;
        for (std::size_t i = 0; i < c.size(); ++i) {
            uint64_t max_load = 0, atomic = 0;
            grouping_cost_dev(p.D, p.offsets.get(), c[i], dim, static_cast<uint64_t>(workers), &max_load, &atomic, s);
            const double cost = static_cast<double>(max_load) + lambda * static_cast<double>(atomic);
            if (table) table[i] = cost;
            if (first || cost < best_cost || (cost == best_cost && c[i] < best_gs)) {
                first = false;
                best_cost = cost;
                best_gs = c[i];
            }
        }
        *best = best_gs;
        if (ncand_out) *ncand_out = c.size();
    });
}

int pg_gs_oracle_measured(pg_path h, uint64_t dim, int repeats, uint64_t seed, const uint32_t* cands,
                          uint64_t ncand, uint32_t* best, double* table, uint64_t* ncand_out) {
    return guard([&] {
        Path& p = *P_(h);
        std::vector<uint32_t> c;
        if (cands) {
            c.assign(cands, cands + ncand);
        } else {
            uint32_t tmp[40];
            uint64_t k = 0;
            if (int rc = pg_gs_default_candidates(p.max_degree, tmp, &k)) fail(rc, g_err);
            c.assign(tmp, tmp + k);
        }
        if (c.empty()) fail(kConfig, "oracle_gs: empty candidate list");
        if (repeats < 1) fail(kConfig, "measured oracle: repeats must be >= 1");
        DeviceGuard dg(p.device);
        cudaStream_t s = lib_stream(p.device);
        // measured_evaluator's input (train.hpp:38-41): U(0,1) from
        // mt19937_64(derive_seed(seed, 17)), row-major rows x dim
        const uint64_t rows = p.P, ld = (dim + 3) & ~3ull;
        std::vector<float> host(rows * dim);
        std::mt19937_64 rng(derive_seed(seed, 17));
        std::uniform_real_distribution<double> u(0.0, 1.0);
        for (float& v : host) v = static_cast<float>(u(rng));
        DevBuf<float> in(std::max<uint64_t>(rows * ld, 1), s), out(std::max<uint64_t>(uint64_t(p.D) * ld, 1), s);
        if (rows * dim)
            PG_CUDA(cudaMemcpy2DAsync(in.get(), ld * 4, host.data(), dim * 4, dim * 4, rows, cudaMemcpyHostToDevice, s));
        cudaEvent_t e0, e1;
        PG_CUDA(cudaEventCreate(&e0));
        PG_CUDA(cudaEventCreate(&e1));
        double best_t = 0.0;
        uint32_t best_gs = 1;
        bool first = true;
        for (std::size_t i = 0; i < c.size(); ++i) {
            auto G = groups_build(p.D, p.offsets.get(), c[i], p.device);
            G->path = &p;
            std::vector<double> ts;
            for (int r = 0; r < repeats; ++r) {
                PG_CUDA(cudaEventRecord(e0, s));
                run_aggregate(*G, true, 0, p.D, in.get(), ld, out.get(), ld, dim, PG_AGG_OVERWRITE | PG_AGG_GROUPED, s);
                PG_CUDA(cudaEventRecord(e1, s));
                PG_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                PG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                ts.push_back(ms * 1e-3);
            }
            std::sort(ts.begin(), ts.end());
            const double cost = ts[ts.size() / 2];
            if (table) table[i] = cost;
            if (first || cost < best_t || (cost == best_t && c[i] < best_gs)) {
                first = false;
                best_t = cost;
                best_gs = c[i];
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        PG_CUDA(cudaStreamSynchronize(s));
        *best = best_gs;
        if (ncand_out) *ncand_out = c.size();
    });
}

int pg_grouping_cost(pg_groups h, uint64_t dim, int workers, double lambda, double* cost) {
    return guard([&] {
        Groups& G = *R_(h);
        if (workers < 1) fail(kConfig, "cost model: worker count must be >= 1");
        const Base b = base_of(G);
        DeviceGuard dg(G.device);
        uint64_t max_load = 0, atomic = 0;
        grouping_cost_dev(b.D, b.offsets, G.gs, dim, static_cast<uint64_t>(workers), &max_load, &atomic,
                          lib_stream(G.device));
        *cost = static_cast<double>(max_load) + lambda * static_cast<double>(atomic);
    });
}

int pg_group(pg_path h, uint32_t gs, pg_groups* out) {
    return guard([&] {
        Path& p = *P_(h);
        auto G = groups_build(p.D, p.offsets.get(), gs, p.device);
        G->path = &p;
        *out = reinterpret_cast<pg_groups>(G.release());
    });
}

int pg_group_graph(pg_graph h, uint32_t gs, pg_groups* out) {
    return guard([&] {
        Graph& g = *G_(h);
        auto G = groups_build(g.n, g.offsets.get(), gs, g.device);
        G->graph = &g;
        *out = reinterpret_cast<pg_groups>(G.release());
    });
}

int pg_groups_info(pg_groups h, uint32_t* gs, uint64_t* count, uint32_t* dests) {
    return guard([&] {
        Groups& G = *R_(h);
        if (gs) *gs = G.gs;
        if (count) *count = G.G;
        if (dests) *dests = base_of(G).D;
    });
}

int pg_groups_export(pg_groups h, uint32_t* dest, uint64_t* edge_begin, uint64_t* edge_end, uint64_t* dest_groups) {
    return guard([&] {
        Groups& G = *R_(h);
        DeviceGuard dg(G.device);
        cudaStream_t s = lib_stream(G.device);
        auto cp = [&](void* dst, const void* srcp, uint64_t bytes) {
            if (dst && bytes) PG_CUDA(cudaMemcpyAsync(dst, srcp, bytes, cudaMemcpyDeviceToHost, s));
        };
        cp(dest, G.gdest.get(), G.G * 4);
        cp(edge_begin, G.gbegin.get(), G.G * 8);
        cp(edge_end, G.gend.get(), G.G * 8);
        cp(dest_groups, G.dest_groups.get(), (static_cast<uint64_t>(base_of(G).D) + 1) * 8);
        PG_CUDA(cudaStreamSynchronize(s));
    });
}

int pg_groups_destroy(pg_groups h) {
    return guard([&] {
        Groups* G = reinterpret_cast<Groups*>(h);
        if (!G) return;
        DeviceGuard dg(G->device);
        drain_device();  // kernels on caller streams may still read its buffers
        delete G;
    });
}

// ---------------- backward aggregate ----------------

int pg_aggregate_pull(pg_groups h, const float* in_dev, uint64_t in_rows, uint64_t ld_in, float* out_dev,
                      uint64_t ld_out, uint64_t dim, unsigned flags, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        const Base b = base_of(G);
        check_dims(dim, ld_in, ld_out);
        if (in_rows != b.in_rows_local)
            fail_shape("aggregate_pull: input rows != source count of the grouping's base");
        run_aggregate(G, false, 0, b.D, in_dev, ld_in, out_dev, ld_out, dim, flags,
                      static_cast<cudaStream_t>(stream));
    });
}

int pg_backward_aggregate(pg_groups h, const float* y_dev, uint64_t y_rows, uint64_t ld_in, float* x_dev,
                          uint64_t ld_out, uint64_t dim, unsigned flags, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        check_dims(dim, ld_in, ld_out);
        if (y_rows != y_rows_of(G)) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        run_aggregate(G, true, 0, G.path->D, y_dev, ld_in, x_dev, ld_out, dim, flags,
                      static_cast<cudaStream_t>(stream));
    });
}

int pg_backward_aggregate_rows(pg_groups h, uint32_t row_begin, uint32_t row_end, const float* y_dev,
                               uint64_t y_rows, uint64_t ld_in, float* x_dev, uint64_t ld_out, uint64_t dim,
                               unsigned flags, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        check_dims(dim, ld_in, ld_out);
        if (y_rows != y_rows_of(G)) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        if (row_begin > row_end || row_end > G.path->D) fail(kConfig, "backward_aggregate: bad row range");
        if (row_begin == row_end) return;
        run_aggregate(G, true, row_begin, row_end, y_dev, ld_in, x_dev, ld_out, dim, flags,
                      static_cast<cudaStream_t>(stream));
    });
}

// ---- aggregate_pull<double> (the reference's default precision) ----
namespace {
// the f64 SpMM over a grouping's base: parent-indexed (the engine.hpp:334
// gather folded in) or local / vertex-indexed sources
// aggregate_pull<double> hubs: rows of <= 32 doubles whose lists are longer
// than this go to k_agg_f64_hub (k_agg_f64 pays one gather round trip per
// batch of 8 edges of a list). Measured on the Reddit top path (width 16,
// 75.6M edges): no hub kernel 4.65 ms, lists >= 10.6K 2.21, >= 4096 1.39,
// >= 1024 1.98. Wide rows keep every list in k_agg_f64 (layer 0, width 602:
// 46.6 ms, 62.9 with the hubs >= 4096 on the hub kernel, 100 with >= 1024),
// and chunk-major without a destination-major front (the front cost
// 42.9 -> 54.2 ms). Tuning "f64_hub_min" > 0 forces the threshold.
constexpr uint64_t kNoHubs = 0;  // DegHist::heavy(0) = no destinations
uint64_t f64_hub_degree(uint64_t dim) {
    const int64_t forced = tuning(kTuneF64HubMin);
    if (forced > 0) return static_cast<uint64_t>(forced);
    return dim <= 32 ? 4096 : kNoHubs;
}

void run_aggregate_f64(Groups& G, bool parent_indexed, const double* in, uint64_t ld_in, double* out, uint64_t ld_out,
                       uint64_t dim, unsigned flags, cudaStream_t s) {
    DeviceGuard dg(G.device);
    std::lock_guard<std::recursive_mutex> lk(G.mu);
    const bool accumulate = !(flags & PG_AGG_OVERWRITE);
    if (G.path) {
        Path& p = *G.path;
        const uint32_t* src = parent_indexed ? reinterpret_cast<const uint32_t*>(p.edges_parent.get())
                                             : p.nbr_local.get();
        const uint32_t stride = parent_indexed ? 2u : 1u;
        // the f32 path's L2-sized source segments (a 32-lane double2 chunk
        // is 512 B, the f32 chunk's size): accumulate passes in source order
        const uint32_t K = parent_indexed ? auto_src_segments(p.P, p.D, p.E, dim) : 1u;
        if (K > 1) {
            auto_segment_bounds(G, p, K);
            for (uint32_t k = 0; k < K; ++k) {
                const uint64_t* eb = G.auto_seg_bnd.get() + static_cast<uint64_t>(k) * p.D;
                aggregate_f64(eb, eb + p.D, src, stride, p.w64.get(), p.order.get(), p.D,
                              p.hist.heavy(f64_hub_degree(dim)), 0u, in, ld_in,
                              out, ld_out, dim, accumulate || k > 0, s, p.E / K);
            }
            return;
        }
        aggregate_f64(p.offsets.get(), p.offsets.get() + 1, src, stride, p.w64.get(), p.order.get(), p.D,
                      p.hist.heavy(f64_hub_degree(dim)), 0u, in, ld_in, out, ld_out,
                      dim, accumulate, s, p.E);
        return;
    }
    Graph& g = *G.graph;
    if (!G.graph_order.get() && g.n)
        degree_order(g.offsets.get(), g.n, G.graph_order, lib_stream(g.device), &G.graph_hist);
    aggregate_f64(g.offsets.get(), g.offsets.get() + 1, g.nbrs.get(), 1u, g.w64.get(), G.graph_order.get(), g.n,
                  G.graph_hist.heavy(f64_hub_degree(dim)), 0u, in, ld_in, out,
                  ld_out, dim, accumulate, s, g.m);
}

// host DenseMatrix<double> drop-in: copy in (pitched to even ld), run, copy out
void run_host_f64(Groups& G, bool parent_indexed, const double* in_host, uint64_t in_rows, uint64_t dim,
                  double* out_host, uint64_t out_rows, unsigned flags) {
    DeviceGuard dg(G.device);
    cudaStream_t s = lib_stream(G.device);
    // 128-byte device rows past 16 columns (256-bit gathers need a 4-double
    // pitch), else 16-byte
    const uint64_t ld = dim > 16 ? (dim + 15) & ~15ull : (dim + 1) & ~1ull;
    DevBuf<double> din(in_rows * ld, s), dout(out_rows * ld, s);
    if (in_rows && dim)
        PG_CUDA(cudaMemcpy2DAsync(din.get(), ld * 8, in_host, dim * 8, dim * 8, in_rows, cudaMemcpyHostToDevice, s));
    if (!(flags & PG_AGG_OVERWRITE) && out_rows && dim)
        PG_CUDA(cudaMemcpy2DAsync(dout.get(), ld * 8, out_host, dim * 8, dim * 8, out_rows, cudaMemcpyHostToDevice, s));
    run_aggregate_f64(G, parent_indexed, din.get(), ld, dout.get(), ld, dim, flags, s);
    if (out_rows && dim)
        PG_CUDA(cudaMemcpy2DAsync(out_host, dim * 8, dout.get(), ld * 8, dim * 8, out_rows, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

int pg_aggregate_pull_f64(pg_groups h, const double* in_dev, uint64_t in_rows, uint64_t ld_in, double* out_dev,
                          uint64_t ld_out, uint64_t dim, unsigned flags, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        check_dims(dim, ld_in, ld_out);
        if (in_rows != base_of(G).in_rows_local)
            fail_shape("aggregate_pull: input rows != source count of the grouping's base");
        if (flags & PG_AGG_GROUPED) fail(kConfig, "aggregate_pull<double>: the grouped Fast kernel is fp32 only");
        run_aggregate_f64(G, false, in_dev, ld_in, out_dev, ld_out, dim, flags, static_cast<cudaStream_t>(stream));
    });
}

int pg_backward_aggregate_f64(pg_groups h, const double* y_dev, uint64_t y_rows, uint64_t ld_in, double* x_dev,
                              uint64_t ld_out, uint64_t dim, unsigned flags, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        check_dims(dim, ld_in, ld_out);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        if (y_rows != G.path->P) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        if (flags & PG_AGG_GROUPED) fail(kConfig, "aggregate_pull<double>: the grouped Fast kernel is fp32 only");
        run_aggregate_f64(G, true, y_dev, ld_in, x_dev, ld_out, dim, flags, static_cast<cudaStream_t>(stream));
    });
}

int pg_aggregate_pull_host_f64(pg_groups h, const double* in_host, uint64_t in_rows, uint64_t dim, double* out_host,
                               unsigned flags, uint64_t* counters) {
    return guard([&] {
        Groups& G = *R_(h);
        const Base b = base_of(G);
        if (in_rows != b.in_rows_local)
            fail_shape("aggregate_pull: input rows != source count of the grouping's base");
        if (flags & PG_AGG_GROUPED) fail(kConfig, "aggregate_pull<double>: the grouped Fast kernel is fp32 only");
        run_host_f64(G, false, in_host, in_rows, dim, out_host, b.D, flags);
        counters_of(G, dim, flags, counters);
    });
}

int pg_backward_aggregate_host_f64(pg_groups h, const double* y_host, uint64_t y_rows, uint64_t dim, double* x_host,
                                   unsigned flags, uint64_t* counters) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        if (y_rows != G.path->P) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        if (flags & PG_AGG_GROUPED) fail(kConfig, "aggregate_pull<double>: the grouped Fast kernel is fp32 only");
        run_host_f64(G, true, y_host, y_rows, dim, x_host, G.path->D, flags);
        counters_of(G, dim, flags, counters);
    });
}

int pg_aggregate_pull_host(pg_groups h, const float* in_host, uint64_t in_rows, uint64_t dim, float* out_host,
                           unsigned flags, uint64_t* counters) {
    return guard([&] {
        Groups& G = *R_(h);
        if (in_rows != base_of(G).in_rows_local)
            fail_shape("aggregate_pull: input rows != source count of the grouping's base");
        run_host(G, false, in_host, in_rows, dim, out_host, flags);
        counters_of(G, dim, flags, counters);
    });
}

int pg_backward_aggregate_host(pg_groups h, const float* y_host, uint64_t y_rows, uint64_t dim, float* x_host,
                               unsigned flags, uint64_t* counters) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        if (y_rows != y_rows_of(G)) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        run_host(G, true, y_host, y_rows, dim, x_host, flags);
        counters_of(G, dim, flags, counters);
    });
}

int pg_groups_remap_sources(pg_groups h, const uint32_t* map, uint64_t map_len, uint64_t new_rows) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "remap: grouping is not over an execution path");
        Path& p = *G.path;
        DeviceGuard dg(G.device);
        std::lock_guard<std::recursive_mutex> lk(G.mu);
        cudaStream_t s = lib_stream(G.device);
        if (!map) {
            retire(G.edges_remap);
            G.remap_rows = 0;
            return;
        }
        if (map_len != p.P) fail_shape("remap: map length != parent frontier size");
        for (uint64_t i = 0; i < map_len; ++i)
            if (map[i] >= new_rows) fail(kConfig, "remap: map entry out of range");
        DevBuf<uint32_t> dmap(map_len, s);
        if (map_len) PG_CUDA(cudaMemcpyAsync(dmap.get(), map, map_len * 4, cudaMemcpyHostToDevice, s));
        DevBuf<Edge> out = edge_buf(p.E, s);
        remap_edges(p.edges_parent.get(), p.E, dmap.get(), out.get(), s);
        PG_CUDA(cudaStreamSynchronize(s));
        retire(G.edges_remap);
        G.edges_remap = std::move(out);
        G.remap_rows = new_rows;
    });
}

int pg_groups_set_segments(pg_groups h, const uint64_t* cuts, uint32_t nseg) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "segments: grouping is not over an execution path");
        Path& p = *G.path;
        DeviceGuard dg(G.device);
        std::lock_guard<std::recursive_mutex> lk(G.mu);
        if (!cuts || nseg == 0) {
            G.seg_cuts.clear();
            retire(G.seg_bnd);
            return;
        }
        const uint64_t rows = y_rows_of(G);
        if (cuts[0] != 0 || cuts[nseg] != (G.edges_remap.get() ? G.remap_rows : p.P))
            fail(kConfig, "segments: cuts must start at 0 and end at the input row count");
        for (uint32_t k = 0; k < nseg; ++k)
            if (cuts[k + 1] < cuts[k]) fail(kConfig, "segments: cuts must be non-decreasing");
        (void)rows;
        const Edge* edges = G.edges_remap.get() ? G.edges_remap.get() : p.edges_parent.get();
        segment_bounds(p.offsets.get(), edges, p.D, cuts, nseg, G.seg_bnd, lib_stream(G.device));
        G.seg_cuts.assign(cuts, cuts + nseg + 1);
    });
}

int pg_backward_aggregate_segment(pg_groups h, uint32_t seg, uint32_t row_begin, uint32_t row_end,
                                  const float* y_dev, uint64_t y_rows, uint64_t ld_in, float* x_dev, uint64_t ld_out,
                                  uint64_t dim, unsigned flags, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        if (G.seg_cuts.empty() || seg + 1 >= G.seg_cuts.size()) fail(kConfig, "segments: segment index out of range");
        check_dims(dim, ld_in, ld_out);
        if (y_rows != y_rows_of(G)) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        if (row_begin > row_end || row_end > G.path->D) fail(kConfig, "backward_aggregate: bad row range");
        if (row_begin == row_end) return;
        run_aggregate(G, true, row_begin, row_end, y_dev, ld_in, x_dev, ld_out, dim, flags,
                      static_cast<cudaStream_t>(stream),
                      SegSel{G.seg_bnd.get(), static_cast<int>(seg), static_cast<uint32_t>(G.seg_cuts.size() - 1)});
    });
}

int pg_stage_counters(pg_groups h, uint64_t dim, unsigned flags, uint64_t* counters) {
    return guard([&] { counters_of(*R_(h), dim, flags, counters); });
}

int pg_path_shard_bounds(pg_path h, uint32_t world, uint32_t* bounds) {
    return guard([&] {
        Path& p = *P_(h);
        if (world < 1) fail(kConfig, "shard: world size must be >= 1");
        std::vector<uint64_t> off(static_cast<uint64_t>(p.D) + 1);
        DeviceGuard dg(p.device);
        cudaStream_t s = lib_stream(p.device);
        PG_CUDA(cudaMemcpyAsync(off.data(), p.offsets.get(), off.size() * 8, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
        bounds[0] = 0;
        for (uint32_t r = 1; r < world; ++r) {
            const uint64_t target = (p.E * r) / world;
            const uint32_t row = static_cast<uint32_t>(
                std::lower_bound(off.begin(), off.end() - 1, target) - off.begin());
            bounds[r] = std::max(bounds[r - 1], std::min(row, p.D));
        }
        bounds[world] = p.D;
    });
}

// ---------------- dense helpers ----------------

int pg_gemm_a_bt(const float* a, uint64_t lda, const float* b, uint64_t ldb, float* out, uint64_t ldo, uint64_t n,
                 uint64_t m, uint64_t k, void* stream) {
    return guard([&] {
        if (lda < k || ldb < k || ldo < m) fail_shape("gemm_a_bt: leading dimension too small");
        gemm(DMat{const_cast<float*>(a), n, k, lda}, DMat{const_cast<float*>(b), m, k, ldb}, DMat{out, n, m, ldo},
             true, static_cast<cudaStream_t>(stream));
    });
}

int pg_gemm_a_bt_ex(const float* a, uint64_t lda, const float* b, uint64_t ldb, float* out, uint64_t ldo,
                    uint64_t n, uint64_t m, uint64_t k, unsigned flags, void* stream) {
    return guard([&] {
        if (lda < k || ldb < k || ldo < m) fail_shape("gemm_a_bt: leading dimension too small");
        if (flags & ~PG_GEMM_TF32X3) fail(kConfig, "gemm_a_bt: unknown flags");
        const DMat A{const_cast<float*>(a), n, k, lda}, B{const_cast<float*>(b), m, k, ldb}, O{out, n, m, ldo};
        if (flags & PG_GEMM_TF32X3) {
            gemm_a_bt_tc(A, B, O, static_cast<cudaStream_t>(stream));
        } else {
            gemm(A, B, O, true, static_cast<cudaStream_t>(stream));
        }
    });
}

int pg_relu_backward(const float* grad, uint64_t ldg, const float* pre, uint64_t ldp, float* out, uint64_t ldo,
                     uint64_t rows, uint64_t cols, void* stream) {
    return guard([&] { relu_backward(grad, ldg, pre, ldp, out, ldo, rows, cols, static_cast<cudaStream_t>(stream)); });
}

int pg_gather_rows(const float* src, uint64_t lds, const uint32_t* ids_dev, uint64_t k, float* out, uint64_t ldo,
                   uint64_t cols, void* stream) {
    return guard([&] { gather_rows(src, lds, ids_dev, k, out, ldo, cols, static_cast<cudaStream_t>(stream)); });
}

// ---- device memory helpers (header-only C++ callers) ----

int pg_device_alloc(int device, uint64_t bytes, void** out) {
    return guard([&] {
        DeviceGuard dg(device);
        *out = nullptr;
        if (bytes) PG_CUDA(cudaMalloc(out, bytes));
    });
}

int pg_device_free(int device, void* p) {
    return guard([&] {
        DeviceGuard dg(device);
        if (p) PG_CUDA(cudaFree(p));
    });
}

int pg_memcpy_h2d(int device, void* dst, const void* src, uint64_t bytes) {
    return guard([&] {
        DeviceGuard dg(device);
        if (bytes) PG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    });
}

int pg_memcpy_d2h(int device, void* dst, const void* src, uint64_t bytes) {
    return guard([&] {
        DeviceGuard dg(device);
        if (bytes) PG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    });
}

int pg_memset_zero(int device, void* dst, uint64_t bytes) {
    return guard([&] {
        DeviceGuard dg(device);
        if (bytes) PG_CUDA(cudaMemset(dst, 0, bytes));
    });
}

int pg_mat_upload(int device, pg_mat dst, const float* host) {
    return guard([&] {
        if (dst.rows && dst.cols && (!dst.data || !host)) fail(kConfig, "pg_mat_upload: null buffer");
        if (dst.ld < dst.cols) fail_shape("pg_mat_upload: ld < cols");
        if (!dst.rows || !dst.cols) return;
        DeviceGuard dg(device);
        cudaStream_t s = lib_stream(device);
        const uint64_t bytes = dst.rows * dst.cols * 4;
        if (dst.ld == dst.cols) {
            PG_CUDA(cudaMemcpyAsync(dst.data, host, bytes, cudaMemcpyHostToDevice, s));
        } else {
            DevBuf<float> flat(dst.rows * dst.cols, s);
            PG_CUDA(cudaMemcpyAsync(flat.get(), host, bytes, cudaMemcpyHostToDevice, s));
            copy_rows(flat.get(), dst.cols, dst.data, dst.ld, dst.rows, dst.cols, s);
        }
        PG_CUDA(cudaStreamSynchronize(s));
    });
}

int pg_mat_download(int device, float* host, pg_mat src) {
    return guard([&] {
        if (src.rows && src.cols && (!src.data || !host)) fail(kConfig, "pg_mat_download: null buffer");
        if (src.ld < src.cols) fail_shape("pg_mat_download: ld < cols");
        if (!src.rows || !src.cols) return;
        DeviceGuard dg(device);
        PG_CUDA(cudaDeviceSynchronize());  // the matrix may have been written on any stream
        cudaStream_t s = lib_stream(device);
        const uint64_t bytes = src.rows * src.cols * 4;
        if (src.ld == src.cols) {
            PG_CUDA(cudaMemcpyAsync(host, src.data, bytes, cudaMemcpyDeviceToHost, s));
        } else {
            DevBuf<float> flat(src.rows * src.cols, s);
            copy_rows(src.data, src.ld, flat.get(), src.cols, src.rows, src.cols, s);
            PG_CUDA(cudaMemcpyAsync(host, flat.get(), bytes, cudaMemcpyDeviceToHost, s));
        }
        PG_CUDA(cudaStreamSynchronize(s));
    });
}

uint64_t pg_launch_count(void) { return pg::launch_counter(); }

int pg_device_synchronize(int device) {
    return guard([&] {
        DeviceGuard dg(device);
        PG_CUDA(cudaDeviceSynchronize());
    });
}

// ---- the GCN chain (engine.cu) ----

int pg_gemm(pg_mat a, pg_mat b, int b_transposed, pg_mat out, void* stream) {
    return guard([&] { gemm(dm(a), dm(b), dm(out), b_transposed != 0, static_cast<cudaStream_t>(stream)); });
}

int pg_gemm_at_b(pg_mat a, const uint32_t* a_rows, pg_mat b, pg_mat out, void* stream) {
    return guard([&] { gemm_at_b(dm(a), a_rows, dm(b), dm(out), static_cast<cudaStream_t>(stream)); });
}

int pg_gemm_at_b_ex(pg_mat a, const uint32_t* a_rows, pg_mat b, pg_mat out, unsigned flags, void* stream) {
    return guard([&] {
        if (flags & ~PG_GEMM_TF32X3) fail(kConfig, "gemm_at_b: unknown flags");
        if (flags & PG_GEMM_TF32X3)
            gemm_at_b_tc(dm(a), a_rows, dm(b), dm(out), static_cast<cudaStream_t>(stream));
        else
            gemm_at_b(dm(a), a_rows, dm(b), dm(out), static_cast<cudaStream_t>(stream));
    });
}

int pg_relu(pg_mat x, pg_mat out, void* stream) {
    return guard([&] { relu(dm(x), dm(out), static_cast<cudaStream_t>(stream)); });
}

int pg_row_softmax(pg_mat x, pg_mat out, void* stream) {
    return guard([&] { row_softmax(dm(x), dm(out), static_cast<cudaStream_t>(stream)); });
}

int pg_top_grad_from_probs(pg_mat probs, pg_mat ref, const uint32_t* vt_dev, uint64_t k, pg_mat out, void* stream) {
    return guard([&] {
        top_grad_from_probs(dm(probs), dm(ref), vt_dev, k, dm(out), static_cast<cudaStream_t>(stream));
    });
}

int pg_aggregate_pull_filtered(pg_groups h, pg_frontiers hf, uint64_t dest_level, uint64_t src_level,
                               const float* in_dev, uint64_t in_rows, uint64_t ld_in, float* out_dev,
                               uint64_t ld_out, uint64_t dim, unsigned flags, uint64_t* counters, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        Frontiers& F = *F_(hf);
        if (!G.graph) fail(kConfig, "aggregate_pull_filtered: needs a grouping of the full graph");
        if (dest_level > F.L || src_level > F.L) fail(kConfig, "aggregate_pull_filtered: level out of range");
        if (F.n != G.graph->n) fail(kConfig, "aggregate_pull_filtered: frontiers are for another graph");
        if (in_rows != G.graph->n) fail_shape("aggregate_pull_filtered: input rows != vertex count");
        check_dims(dim, ld_in, ld_out);
        AggExt ext;
        ext.dst_bits = F.levels[dest_level].bits.get();
        ext.src_bits = F.levels[src_level].bits.get();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        run_aggregate(G, false, 0, G.graph->n, in_dev, ld_in, out_dev, ld_out, dim, flags, s, SegSel{}, ext);
        if (counters) {
            DeviceGuard dg(G.device);
            filter_counts(*G.graph, G.gs, ext.dst_bits, ext.src_bits, counters, s);
        }
    });
}

int pg_forward(pg_groups h, pg_mat x0, const pg_mat* w, uint64_t layers, pg_mat* y, pg_mat* pre, pg_mat* x,
               void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        if (!w || !y || !pre || !x) fail(kConfig, "forward: null matrix array");
        std::vector<DMat> W(layers), Y(layers), P(layers), X(layers);
        for (uint64_t l = 0; l < layers; ++l) {
            W[l] = dm(w[l]);
            Y[l] = dm(y[l]);
            P[l] = dm(pre[l]);
            X[l] = dm(x[l]);
        }
        DeviceGuard dg(G.device);
        forward(G, dm(x0), W.data(), layers, Y.data(), P.data(), X.data(), static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

namespace {

// BackwardIO over the caller's arrays (storage kept alive by the holder)
struct IoHolder {
    std::vector<DMat> y, pre, w, wg, xg;
    BackwardIO io;
    IoHolder(uint64_t L, const pg_mat* py, const pg_mat* ppre, pg_mat top, const pg_mat* pw, pg_mat* pwg,
             pg_mat* pxg, uint64_t* edges) {
        if (!py || !ppre || !pw || !pwg) fail(kConfig, "backward: null matrix array");
        for (uint64_t l = 0; l < L; ++l) {
            y.push_back(dm(py[l]));
            pre.push_back(dm(ppre[l]));
            w.push_back(dm(pw[l]));
            wg.push_back(dm(pwg[l]));
            if (pxg) xg.push_back(dm(pxg[l]));
        }
        io.L = L;
        io.y = y.data();
        io.pre = pre.data();
        io.top_grad = dm(top);
        io.w = w.data();
        io.w_grads = wg.data();
        io.x_grads = pxg ? xg.data() : nullptr;
        io.edges = edges;
    }
};

}  // namespace

extern "C" {

int pg_backward_epp(const pg_groups* path_groups, pg_frontiers hf, uint64_t layers, const pg_mat* y,
                    const pg_mat* pre, pg_mat top_grad, const pg_mat* w, uint64_t expected_fingerprint,
                    int gather_mode, pg_mat* w_grads, pg_mat* x_grads, uint64_t* edges_per_layer, void* stream) {
    return guard([&] {
        Frontiers& F = *F_(hf);
        if (!path_groups) fail(kConfig, "epp backward: null path groupings");
        if (gather_mode != 0 && gather_mode != 1) fail(kConfig, "epp backward: gather mode must be 0 or 1");
        std::vector<Groups*> PGs(layers);
        for (uint64_t i = 0; i < layers; ++i) PGs[i] = R_(path_groups[i]);
        IoHolder h(layers, y, pre, top_grad, w, w_grads, x_grads, edges_per_layer);
        DeviceGuard dg(F.device);
        backward_epp(PGs.data(), F, h.io, gather_mode, expected_fingerprint, static_cast<cudaStream_t>(stream));
    });
}

int pg_backward_all_active(pg_groups h, uint64_t layers, const pg_mat* y, const pg_mat* pre, pg_mat top_grad,
                           const pg_mat* w, pg_mat* w_grads, pg_mat* x_grads, uint64_t* edges_per_layer,
                           void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        IoHolder io(layers, y, pre, top_grad, w, w_grads, x_grads, edges_per_layer);
        DeviceGuard dg(G.device);
        backward_all_active(G, io.io, static_cast<cudaStream_t>(stream));
    });
}

int pg_backward_ifelse(pg_groups h, pg_frontiers hf, uint64_t layers, const pg_mat* y, const pg_mat* pre,
                       pg_mat top_grad, const pg_mat* w, pg_mat* w_grads, pg_mat* x_grads,
                       uint64_t* edges_per_layer, void* stream) {
    return guard([&] {
        Groups& G = *R_(h);
        Frontiers& F = *F_(hf);
        IoHolder io(layers, y, pre, top_grad, w, w_grads, x_grads, edges_per_layer);
        DeviceGuard dg(G.device);
        backward_ifelse(G, F, io.io, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
