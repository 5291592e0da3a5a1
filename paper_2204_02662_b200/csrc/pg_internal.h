// Internal handle layouts and kernel launchers of libpathgcn_b200.so.
// The public surface is the C ABI in include/pathgcn_b200.h; nothing here
// crosses the library boundary.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace pg {

// One library-owned non-blocking stream per device for the build calls
// (graph load, frontiers, paths, groups, gs sweep), which are synchronous at
// the ABI like the reference's functions.
cudaStream_t lib_stream(int device);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) PG_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Packed edge record streamed by the SpMM: (source row, fp32 weight bits).
using Edge = uint2;
// Every edge stream carries kEdgePad zeroed records past its end, so a
// 16-byte bulk copy (cp.async.bulk) of any record window may round its end
// up (the grouped kernel stages its CTA's window that way).
constexpr uint64_t kEdgePad = 2;
inline DevBuf<Edge> edge_buf(uint64_t E, cudaStream_t s) {
    DevBuf<Edge> b(E + kEdgePad, s);
    PG_CUDA(cudaMemsetAsync(b.get() + E, 0, kEdgePad * sizeof(Edge), s));
    return b;
}

// Degree-bucket histogram of a schedule (bucket b = floor(log2 deg) + 1).
struct DegHist {
    unsigned long long h[65] = {};
    uint64_t edges = 0;  // edges of the scheduled range
    // destinations of degree >= min_deg (rounded up to a power of two): the
    // prefix of the descending-bucket order
    uint32_t heavy(uint64_t min_deg) const {
        if (min_deg == 0) return 0;
        int b0 = 1;
        while ((1ull << (b0 - 1)) < min_deg) ++b0;
        unsigned long long c = 0;
        for (int b = b0; b < 65; ++b) c += h[b];
        return static_cast<uint32_t>(c);
    }
};

// csr_graph.hpp:19-38 CsrGraph, device resident.
struct Graph {
    int device = 0;
    uint32_t n = 0;
    uint64_t m = 0;
    uint32_t max_degree = 0;
    DevBuf<uint64_t> offsets;   // n+1
    DevBuf<uint32_t> nbrs;      // m, sorted per row
    DevBuf<double> w64;         // m
    DevBuf<Edge> edges;         // m, lazily packed (nbr, (float)w) for graph aggregation
    bool fp_valid = false;
    uint64_t fp = 0;
};

// One frontier level: sorted ids, membership bitmap, per-word rank prefix.
struct Level {
    uint64_t size = 0;
    DevBuf<uint32_t> ids;
    DevBuf<uint32_t> bits;    // ceil(n/32) words
    DevBuf<uint32_t> prefix;  // ceil(n/32)+1 (exclusive popcount prefix)
};

// frontier.hpp:14-18 FrontierSets.
struct Frontiers {
    int device = 0;
    uint32_t n = 0;
    uint64_t L = 0;
    std::vector<Level> levels;
    const Graph* graph = nullptr;  // borrowed
};

// execution_path.hpp:16-33 ExecutionPath, plus the SpMM's own layout.
struct Path {
    int device = 0;
    uint64_t layer = 0;
    uint32_t D = 0, S = 0, P = 0;  // dests, referenced sources, parent frontier size
    uint64_t E = 0;
    uint32_t max_degree = 0;
    uint64_t fingerprint = 0;
    DevBuf<uint32_t> dest;        // dest_local_to_global (copy of frontier level L-l)
    DevBuf<uint32_t> src;         // src_local_to_global
    DevBuf<uint32_t> srcpos;      // src_pos_in_parent
    DevBuf<uint64_t> offsets;     // D+1
    DevBuf<uint32_t> nbr_local;   // E local source ids (reference layout)
    DevBuf<double> w64;           // E, bitwise copies of the parent weights
    DevBuf<Edge> edges_parent;    // E (src_pos_in_parent[nbr], (float)w): gather folded
    DevBuf<Edge> edges_local;     // E (nbr_local, (float)w), lazily, only when S < P
    DevBuf<Edge> edges_global;    // E (src_local_to_global[nbr], (float)w), lazily (GatherMode::Global)
    DevBuf<uint32_t> order;       // D dests in descending-degree-bucket order (SpMM schedule)
    DegHist hist;                 // degree buckets of `order`
    std::mutex mu;                // guards the lazily built edge streams (groupings share a path)
};

// grouping.hpp:14-28 GroupedCsr over a path (or the whole graph).
struct Groups {
    int device = 0;
    uint32_t gs = 0;
    uint64_t G = 0;
    Path* path = nullptr;    // borrowed base (path grouping)
    Graph* graph = nullptr;  // borrowed base (graph grouping)
    DevBuf<uint32_t> gdest;
    DevBuf<uint64_t> gbegin, gend;
    DevBuf<uint64_t> dest_groups;  // D+1
    DevBuf<uint32_t> graph_order;  // schedule for graph groupings (lazy)
    DegHist graph_hist;
    // schedules of destination-row ranges (multi-GPU shards, host-call
    // copy/compute chunks), built lazily and cached
    struct RowSched {
        uint32_t rb = 0, re = 0;
        DevBuf<uint32_t> order;
        DegHist hist;
    };
    std::vector<RowSched> row_scheds;
    std::vector<uint32_t> host_chunks;  // edge-balanced cuts for pg_*_host overlap
    // multi-GPU: parent rows remapped into a padded allgather layout
    DevBuf<Edge> edges_remap;
    uint64_t remap_rows = 0;
    // source-row segments [cuts[k], cuts[k+1]) of the parent frontier:
    // seg_bnd[k*D + d] = first edge of d with source row >= cuts[k]
    // (k = 0..K), so segment k of d is [seg_bnd[k*D+d], seg_bnd[(k+1)*D+d]).
    // Edges are sorted by source row within a destination, so running the
    // segments in order as accumulate passes is exactly the serial order.
    std::vector<uint64_t> seg_cuts;
    DevBuf<uint64_t> seg_bnd;
    // the host-buffer drop-in's own K-segment source split (H2D overlap)
    DevBuf<uint64_t> host_seg_bnd;
    uint64_t host_seg_rows = 0;
    uint32_t host_seg_k = 0;
    int host_seg_bal = -1;
    int host_chunk_alpha = -1;
    std::vector<uint64_t> host_seg_cuts;  // source-row cuts of the host pipeline
    // automatic L2-sized source segments of a whole-path SpMM (api.cu)
    DevBuf<uint64_t> auto_seg_bnd;
    uint32_t auto_seg_k = 0;
    int64_t auto_seg_bal = 0;
    // schedule of the atomic-free group-partitioned Fast kernel (aggregate.cu
    // k_agg_grp), one per worker count (256 / lanes per group): CTA ranges of
    // consecutive groups that hold whole destinations, each hub destination
    // (more groups or edges than a CTA takes) cut into slices whose partial
    // sums are combined in slice order by k_grp_fixup — no global atomics
    struct GrpSched {
        uint32_t workers = 0;
        DevBuf<uint4> ranges;  // {g0 lo, g0 hi, groups, hub slot or ~0u}
        uint32_t nranges = 0;
        DevBuf<uint4> hubs;    // {dest, first slot, slices, 0}
        uint32_t nhubs = 0, nslots = 0;
        DevBuf<uint32_t> empty;  // destinations without groups (written on overwrite)
        uint32_t nempty = 0;
    };
    std::vector<std::unique_ptr<GrpSched>> grp_scheds;
    // guards every lazily built cache above: aggregate calls on one grouping
    // may come from several host threads (the reference's aggregate_pull takes
    // a const GroupedCsr and is re-entrant); recursive because the segmented
    // whole-path SpMM re-enters run_aggregate
    std::recursive_mutex mu;
};

// seg_bnd for cuts[0..K] over the path's edge stream (binary search per
// (destination, cut)); cuts[0] = 0, cuts[K] = parent rows.
void segment_bounds(const uint64_t* offsets, const Edge* edges, uint32_t D, const uint64_t* cuts_host, uint32_t K,
                    DevBuf<uint64_t>& bnd, cudaStream_t s);

// edges_out[e] = (map[edges_in[e].x], edges_in[e].y)
void remap_edges(const Edge* in, uint64_t E, const uint32_t* map, Edge* out, cudaStream_t s);
// per source row: number of path edges reading it (counts[P], zeroed here)
void source_edge_counts(const Edge* edges, uint64_t E, uint64_t P, uint32_t* counts, cudaStream_t s);

// ---- file formats (io.cu) ----
struct EdgeListData {  // edge_list.hpp:14-18
    std::vector<uint32_t> pairs;  // 2 ids per pair
    uint64_t self_loops = 0;
};
EdgeListData load_edge_list(const char* path);
void write_edge_list(const char* path, const uint32_t* pairs, uint64_t npairs);
std::vector<uint32_t> load_training_set(const char* path, uint32_t n);
void write_training_set(const char* path, const uint32_t* vt, uint64_t k);

// ---- launchers (implemented in graph.cu / path.cu / aggregate.cu) ----
std::unique_ptr<Graph> graph_build(int device, int64_t n_hint, const uint32_t* pairs_host,
                                   uint64_t npairs, int weight_mode);
std::unique_ptr<Graph> graph_upload(int device, uint32_t n, const uint64_t* offsets,
                                    const uint32_t* nbrs, const double* w, bool validate);
void graph_assign_weights(Graph& g, int weight_mode, cudaStream_t s);
void graph_pack_edges(Graph& g, cudaStream_t s);
// max over v < n of offsets[v+1] - offsets[v] (synchronises s)
uint32_t max_degree_dev(const uint64_t* offsets, uint32_t n, cudaStream_t s);

std::unique_ptr<Frontiers> frontiers_compute(const Graph& g, const uint32_t* vt_host, uint64_t k,
                                             uint64_t L);
std::unique_ptr<Path> path_extract(const Graph& g, const Frontiers& f, uint64_t layer);
void path_pack_local(Path& p, cudaStream_t s);
void degree_order(const uint64_t* offsets, uint32_t D, DevBuf<uint32_t>& order, cudaStream_t s,
                  DegHist* hist = nullptr);

std::unique_ptr<Groups> groups_build(uint32_t D, const uint64_t* offsets_dev, uint32_t gs,
                                     int device);
// group_cost.cpp:9-24 for one candidate: returns (max_load, atomic_writes).
void grouping_cost_dev(uint32_t D, const uint64_t* offsets_dev, uint32_t gs, uint64_t dim,
                       uint64_t workers, uint64_t* max_load, uint64_t* atomic_writes,
                       cudaStream_t s);

// Optional extensions of the SpMM used by the engine chains (engine.hpp):
// output-row remap (GatherMode::Global), a fused relu_backward epilogue
// (dense_matrix.hpp:107-113 applied to the finished row), and the if-else
// activity filters of aggregate_pull_filtered (aggregate.hpp:127-170).
struct AggExt {
    const uint32_t* out_rows = nullptr;  // output row of destination d (default d)
    const float* relu_pre = nullptr;     // epilogue: out = pre[prow] > 0 ? acc : +0
    uint64_t ld_pre = 0;
    const uint32_t* pre_rows = nullptr;  // prow of destination d (default: the output row)
    const uint32_t* src_bits = nullptr;  // skip edges whose source (edges[e].x) bit is 0
    const uint32_t* dst_bits = nullptr;  // skip destinations whose bit (of d) is 0: row untouched
    // scheduling only: hubs of wide rows on the concurrent side kernel even
    // when tuning hub_inline is on (row ranges: a host-pipeline chunk or a
    // shard is short, and its hub chains would set its length)
    bool side_hubs = false;
    // scheduling only, row ranges: 0 every destination, 1 only the hub
    // prefix of the range's degree order, 2 all but that prefix
    int part = 0;
    uint64_t part_min_degree = 0;  // the hub prefix of part 1 / 2: degree >= this
    // scheduling only: the call's average edges per destination (0 unknown);
    // very short lists (< 8) gather 4 edges per batch instead of 8
    uint64_t avg_degree = 0;
    // scheduling only: the call's edge count (0 unknown); 256-bit gathers
    // (tuning vec8 auto) from 2^21 edges on
    uint64_t n_edges = 0;
    bool any() const { return out_rows || relu_pre || src_bits || dst_bits; }
};

// aggregate.hpp:56-122 Deterministic, ascending edge order per element.
//   out[d] (+)= sum_{e in [ebeg[d], eend[d])} w_e * in[edges[e].x],  d = order[i]
// (ebeg = offsets, eend = offsets + 1 for whole lists; source-range segments
// pass per-destination sub-ranges)
// The first n_heavy entries of order[d_begin..] (the high-degree prefix of
// the degree-bucket order) run on the TMA-ring kernel concurrently.
void aggregate_det(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order, uint32_t D,
                   uint32_t d_begin, uint32_t d_end, uint32_t n_heavy, const float* in, uint64_t ld_in,
                   float* out, uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s,
                   const AggExt& ext = AggExt{});
// Source-segment selector for run_aggregate: bounds array [(nseg+1) x D] and
// the segment to run (seg < 0: whole edge lists).
struct SegSel {
    const uint64_t* bnd = nullptr;
    int seg = -1;         // first segment of the span, -1 = whole lists
    uint32_t nseg = 1;    // segments in bnd
    int seg_end = -1;     // one past the last segment of the span (-1: seg + 1)
};
// The SpMM over a grouping's base (path: parent-indexed or local sources;
// graph: vertex ids), destination rows [rb, re) with their cached degree
// schedule; flags = PG_AGG_* of the C ABI. edges_override replaces the
// path's edge stream (same destinations and order, other source ids).
// A launch over a sequence of destination runs with per-run completion
// counters (aggregate_seq, k_agg_vec4_seq): run s = items [item0, item0 +
// nd * chunks) of destinations dlist[dofs, dofs + nd), destination-major or
// column-chunk-major; each finished item adds 1 to counters[counter].
struct SeqSeg {
    uint64_t item0;
    uint32_t nd, dofs, dest_major, counter;
};
constexpr int kSeqMax = 24;
struct SeqTable {
    SeqSeg seg[kSeqMax];
    uint32_t nseg = 0;
};
// wide rows (ld % 4 == 0, 16-byte aligned), LPD 32: the k_agg_vec4 body
void aggregate_seq(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* dlist,
                   const SeqTable& tab, uint64_t n_items, uint32_t chunks, const float* in, uint64_t ld_in, float* out,
                   uint64_t ld_out, uint32_t dim, bool accumulate, unsigned* counters, cudaStream_t s);

// degree-ordered schedule of path rows [rb, re) (cached on the grouping;
// caller holds G.mu) and the hub count of that range's SpMM call
Groups::RowSched* row_sched(Groups& G, uint32_t rb, uint32_t re);
uint32_t range_heavy(Groups& G, uint32_t rb, uint32_t re, uint64_t min_degree);
void run_aggregate(Groups& G, bool parent_indexed, uint32_t rb, uint32_t re, const float* in, uint64_t ld_in,
                   float* out, uint64_t ld_out, uint64_t dim, unsigned flags, cudaStream_t s, SegSel sel = {},
                   const AggExt& ext = AggExt{}, const Edge* edges_override = nullptr);

// aggregate.hpp:84-115 CommitMode::Fast over the groups (PG_AGG_GROUPED):
// warp per (group, chunk), plain commit for single-group destinations,
// atomics otherwise; zeroes the D output rows first unless accumulate.
void aggregate_groups(const uint64_t* gbeg, const uint64_t* gend, const uint32_t* gdest, const uint64_t* dest_groups,
                      uint32_t D, uint64_t G, const Edge* edges, const float* in, uint64_t ld_in, float* out,
                      uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s);

// aggregate.hpp:56-122 with T = double (Deterministic order, f64 weights):
// destination d sums edges [ebeg[d], eend[d]) (whole lists or one source
// segment), source of edge e = src[e * src_stride]; destinations in the
// descending-degree `order`: its first n_hub on the hub kernel (forked side
// stream), its first n_front (multi-chunk rows) started destination-major.
void aggregate_f64(const uint64_t* ebeg, const uint64_t* eend, const uint32_t* src, uint32_t src_stride,
                   const double* w, const uint32_t* order, uint32_t D, uint32_t n_hub, uint32_t n_front,
                   const double* in, uint64_t ld_in, double* out, uint64_t ld_out, uint64_t dim, bool accumulate,
                   cudaStream_t s, uint64_t n_edges);

// record a failure as the calling thread's pg_last_error / _kind (api.cu)
void record_error(const Error& e);

// The atomic-free group-partitioned Fast aggregation (default for
// PG_AGG_GROUPED): builds / reuses G's schedule for this width, then the
// main kernel and the hub fixup.
// seg_lo / seg_hi (per destination, optional): only each group's edges in
// [seg_lo[d], seg_hi[d]) — one L2-sized source segment pass
void aggregate_groups_af(Groups& G, const uint64_t* offsets_dev, uint32_t D, const Edge* edges, const float* in,
                         uint64_t ld_in, float* out, uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s,
                         const uint64_t* seg_lo = nullptr, const uint64_t* seg_hi = nullptr);

// PG_HEAVY_MIN_DEG / pg_set_heavy_min_degree (0 disables; UINT64_MAX restores
// the width-dependent default)
uint64_t heavy_min_degree(uint64_t dim, uint64_t range_edges);
void set_heavy_min_degree(uint64_t v);
bool heavy_min_forced();  // pg_set_heavy_min_degree / $PG_HEAVY_MIN_DEG in effect
// scheduling knobs of the SpMM kernels (pg_set_tuning): never change results
enum TuneKeyId {
    kTuneHeavyTma = 0,
    kTuneVecU = 1,
    kTuneChunkMajor = 2,
    kTuneHostSegs = 3,
    kTuneHostChunks = 4,
    kTuneHostTrace = 5,
    kTuneHeavyNarrow = 6,
    kTuneWideLpd = 7,
    kTuneSrcSegs = 8,
    kTuneLdCg = 9,
    kTuneHostChunkOrder = 10,
    kTuneGroupedSeg = 11,
    kTuneHeavyWidePipe = 12,
    kTuneHostFinalSegs = 13,
    kTuneHostPitch2d = 14,
    kTuneHostCopyPrio = 15,
    kTuneHostSegBalance = 16,
    kTuneHostChunkBalance = 17,
    kTuneAtbSplit = 18,
    kTuneAtbPairs = 19,
    kTuneGemmPacked = 20,
    kTuneHostLastSegPct = 21,
    kTuneWgradFork = 22,
    kTuneGemmTc = 23,
    kTuneRecWindow = 24,
    kTuneSrcSegBalance = 25,
    kTuneHostMinMb = 26,
    kTuneRowKernel = 27,
    kTuneRowU = 28,
    kTuneRowSegMb = 29,
    kTuneRowHeavy = 30,
    kTuneVecBlock = 31,
    kTuneHubInline = 32,
    kTuneHubFrontMin = 33,
    kTuneGemm3Rows = 34,
    kTuneGemmBesideWgrad = 35,
    kTuneHostHubChunkSide = 36,
    kTuneVecWindow = 37,
    kTuneHostHubMin = 38,
    kTuneGroupedSrcSegs = 39,
    kTuneNarrowU = 40,
    kTuneAtbDepth = 41,
    kTuneHostFirstChunkPct = 42,
    kTuneHostSeq = 43,
    kTuneAtbQuad = 44,
    kTuneHostSmallChunks = 45,
    kTuneVec8 = 46,
    kTuneF64HubMin = 47,
    kTuneGrpDynamic = 48,
    kTuneVec8U = 49,
    kTuneRangeSideHubs = 50
};
// whole-row SpMM warps (k_agg_row) for this width (tuning "row_kernel")
bool row_kernel_on(uint64_t dim);

int64_t tuning(int key);
bool set_tuning(const char* name, int64_t value);

// dense_matrix.hpp:114-121
void relu_backward(const float* grad, uint64_t ldg, const float* pre, uint64_t ldp, float* out,
                   uint64_t ldo, uint64_t rows, uint64_t cols, cudaStream_t s);
// row-pitch change (host-layout <-> 16-byte device rows)
void copy_rows(const float* src, uint64_t lds, float* dst, uint64_t ldd, uint64_t rows, uint64_t cols,
               cudaStream_t s);
// engine.hpp:162-169
void gather_rows(const float* src, uint64_t lds, const uint32_t* ids, uint64_t k, float* out,
                 uint64_t ldo, uint64_t cols, cudaStream_t s);

// ---- the GCN chain (engine.cu) -----------------------------------------------
// A dense fp32 device matrix: rows x cols, row pitch ld floats.
struct DMat {
    float* p = nullptr;
    uint64_t rows = 0, cols = 0, ld = 0;
};
// row pitch of the library's own temporaries: 16-byte rows up to 32 floats,
// whole 128-byte lines beyond
inline uint64_t pad_ld(uint64_t c) { return c <= 32 ? (c + 3) & ~3ull : (c + 31) & ~31ull; }

// dense_matrix.hpp:40-96: out = a * b (b_transposed: a * b^T, gemm_a_bt)
// packed: -1 = tuning "gemm_packed", else the kernel choice (0 k_gemm, 1 k_gemm2, 2 k_gemm3)
void gemm(DMat a, DMat b, DMat out, bool b_transposed, cudaStream_t s, int packed = -1);
// dense_matrix.hpp:78-95 on the tensor cores (gemm_tc.cu): tcgen05 kind::tf32
// with 3xTF32 operand splitting — within fp32 tolerance, NOT bit-exact.
// supported(): A base 16-byte aligned, ld % 4 == 0, the driver's TMA encoder.
bool gemm_a_bt_tc_supported(DMat a);
void gemm_a_bt_tc(DMat a, DMat b, DMat out, cudaStream_t s);
// dense_matrix.hpp:57-76 W' = gather_rows(a, a_rows)^T b on the tensor cores
// (split-K over the rows, 3xTF32, CTA partials added in fixed order):
// fp32 tolerance, NOT bit-exact. Any shape (blocks of <= 640 x 256 outputs
// per launch); Y and g need 16-byte aligned rows.
bool gemm_at_b_tc_supported(uint64_t in_dim, uint64_t out_dim);
void gemm_at_b_tc(DMat a, const uint32_t* a_rows, DMat b, DMat out, cudaStream_t s);
// dense_matrix.hpp:57-76: out = a[a_rows]^T * b (a_rows nullable: all rows)
void gemm_at_b(DMat a, const uint32_t* a_rows, DMat b, DMat out, cudaStream_t s);
void relu(DMat x, DMat out, cudaStream_t s);
// out[r] = pre[pre_rows[r]] > 0 ? g[r] : 0 (pre_rows nullable)
void relu_backward_rows(DMat g, DMat pre, const uint32_t* pre_rows, DMat out, cudaStream_t s);
void row_softmax(DMat x, DMat out, cudaStream_t s);
void top_grad_from_probs(DMat probs, DMat ref, const uint32_t* vt, uint64_t k, DMat out, cudaStream_t s);
// aggregate_pull_filtered counters {edges, groups, edges_skipped,
// groups_skipped} over the full graph (synchronises s)
void filter_counts(const Graph& g, uint32_t gs, const uint32_t* dst_bits, const uint32_t* src_bits, uint64_t* c4,
                   cudaStream_t s);

// engine.hpp:114-140 forward over a full-graph grouping: x[l] = X^(l+1)
void forward(Groups& graph_groups, DMat x0, const DMat* w, uint64_t L, DMat* y, DMat* pre, DMat* x, cudaStream_t s);

struct BackwardIO {
    uint64_t L = 0;
    const DMat* y = nullptr;    // Y^(l), n x in_dim_l
    const DMat* pre = nullptr;  // pre-activations, n x dims[l]
    DMat top_grad;              // n x dims[L-1]
    const DMat* w = nullptr;    // W^(l), in_dim_l x dims[l]
    DMat* w_grads = nullptr;    // out: in_dim_l x dims[l]
    DMat* x_grads = nullptr;    // optional out, index L-1-l (layer L-1 first)
    uint64_t* edges = nullptr;  // optional out: backward_edges_per_layer
};
// engine.hpp:267-349 (gather_mode 0 = Local, 1 = Global)
void backward_epp(Groups* const* path_groups, Frontiers& F, const BackwardIO& io, int gather_mode,
                  uint64_t expected_fp, cudaStream_t s);
// engine.hpp:177-214
void backward_all_active(Groups& graph_groups, const BackwardIO& io, cudaStream_t s);
// engine.hpp:218-257
void backward_ifelse(Groups& graph_groups, Frontiers& F, const BackwardIO& io, cudaStream_t s);

}  // namespace pg
