// Execution-path preparation on device (bit-exact with the reference):
//   * compute_frontiers (frontier.cpp:7-26): direction-optimising bitmap
//     expansion — push (warp per frontier vertex, atomicOr into u32 words,
//     order independent) for small levels, pull (a vertex joins iff one of
//     its neighbours is in the level; valid since CsrGraph is symmetric,
//     csr_graph.hpp:15-18) for large ones — then popcount-scan compaction to
//     the sorted id array.
//   * extract_execution_path (execution_path.cpp:24-88): warp per destination,
//     __ballot_sync over parent-bitmap tests; kept counts -> u64 scan ->
//     ballot-compacted fill in parent-CSR order. Referenced sources are
//     found by a pull over the parent frontier and ranked by prefix popcount,
//     which yields the same sorted-unique order as the reference's sort+unique
//     and replaces its per-edge lower_bound with O(1) ranks.
//   * group_neighbors (grouping.cpp:7-27) and the cost-model group-size sweep
//     (group_cost.cpp:9-53) as closed-form integer reductions.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <vector>

#include "pg_internal.h"

namespace pg {

namespace {

constexpr int kThreads = 256;

// ---- frontiers -----------------------------------------------------------

__global__ void k_set_bits(const uint32_t* __restrict__ ids, uint64_t k, uint32_t* __restrict__ bits) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < k) atomicOr(bits + (ids[i] >> 5), 1u << (ids[i] & 31));
}

// push: warp per vertex of the current level
__global__ void k_expand_push(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                              const uint32_t* __restrict__ level, uint64_t k,
                              uint32_t* __restrict__ next_bits) {
    const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= k) return;
    const uint32_t v = level[w];
    const uint64_t b = offsets[v], e = offsets[v + 1];
    for (uint64_t j = b + lane_id(); j < e; j += 32) {
        const uint32_t u = nbrs[j];
        atomicOr(next_bits + (u >> 5), 1u << (u & 31));
    }
}

// pull: thread per vertex, early exit at the first neighbour in the level;
// each warp owns 32 consecutive vertices = one bitmap word (no atomics)
__global__ void k_expand_pull(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                              uint32_t n, const uint32_t* __restrict__ cur_bits,
                              uint32_t* __restrict__ next_bits) {
    const uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    bool hit = false;
    if (u < n) {
        const uint64_t e = offsets[u + 1];
        for (uint64_t j = offsets[u]; j < e && !hit; ++j) hit = bit_of(cur_bits, __ldg(nbrs + j));
    }
    const unsigned word = __ballot_sync(0xffffffffu, hit);
    if (lane_id() == 0 && (u >> 5) < (static_cast<uint64_t>(n) + 31) / 32) next_bits[u >> 5] = word;
}

__global__ void k_popc(const uint32_t* __restrict__ bits, uint32_t nw, uint32_t* __restrict__ cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nw) cnt[i] = __popc(bits[i]);
}

// bitmap -> ascending id array (one thread per word)
__global__ void k_bits_to_ids(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ prefix,
                              uint32_t nw, uint32_t* __restrict__ ids) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nw) return;
    uint32_t w = bits[i];
    uint32_t pos = prefix[i];
    while (w) {
        const int b = __ffs(w) - 1;
        ids[pos++] = i * 32 + b;
        w &= w - 1;
    }
}

void finish_level(Level& lv, uint32_t n, cudaStream_t s, bool want_ids) {
    const uint32_t nw = (n + 31) / 32;
    DevBuf<uint32_t> cnt(nw, s);
    lv.prefix = DevBuf<uint32_t>(static_cast<uint64_t>(nw) + 1, s);
    DevBuf<uint64_t> scratch(scan_scratch_elems(nw), s);
    if (nw) {
        k_popc<<<grid_for(nw, kThreads), kThreads, 0, s>>>(lv.bits.get(), nw, cnt.get());
        PG_LAUNCH("k_popc");
    }
    exclusive_scan(cnt.get(), nw, lv.prefix.get(), scratch.get(), s);
    uint32_t total = 0;
    PG_CUDA(cudaMemcpyAsync(&total, lv.prefix.get() + nw, 4, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    lv.size = total;
    if (want_ids) {
        lv.ids = DevBuf<uint32_t>(total, s);
        if (nw && total) {
            k_bits_to_ids<<<grid_for(nw, kThreads), kThreads, 0, s>>>(lv.bits.get(), lv.prefix.get(), nw,
                                                                    lv.ids.get());
            PG_LAUNCH("k_bits_to_ids");
        }
    }
}

// ---- execution path --------------------------------------------------------

__global__ void k_count_kept(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                             const uint32_t* __restrict__ dests, uint32_t D,
                             const uint32_t* __restrict__ parent_bits, uint64_t* __restrict__ kept) {
    const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= D) return;
    const uint32_t v = dests[w];
    const uint64_t b = offsets[v], e = offsets[v + 1];
    uint32_t c = 0;
    for (uint64_t j = b + lane_id(); j < e; j += 32) c += bit_of(parent_bits, __ldg(nbrs + j));
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane_id() == 0) kept[w] = c;
}

// referenced sources: u in parent with a neighbour in the destination set
// (pull over the parent frontier, warp per vertex, early exit)
__global__ void k_mark_sources(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                               const uint32_t* __restrict__ parent, uint32_t P,
                               const uint32_t* __restrict__ dest_bits, uint32_t* __restrict__ src_bits) {
    const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= P) return;
    const uint32_t u = parent[w];
    const uint64_t b = offsets[u], e = offsets[u + 1];
    bool hit = false;
    for (uint64_t j0 = b; j0 < e; j0 += 32) {
        const uint64_t j = j0 + lane_id();
        const bool h = j < e && bit_of(dest_bits, __ldg(nbrs + j));
        if (__any_sync(0xffffffffu, h)) {
            hit = true;
            break;
        }
    }
    if (hit && lane_id() == 0) atomicOr(src_bits + (u >> 5), 1u << (u & 31));
}

__global__ void k_fill_path(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                            const double* __restrict__ w64, const uint32_t* __restrict__ dests, uint32_t D,
                            const uint32_t* __restrict__ parent_bits, const uint32_t* __restrict__ parent_prefix,
                            const uint32_t* __restrict__ src_bits, const uint32_t* __restrict__ src_prefix,
                            const uint64_t* __restrict__ p_offsets, uint32_t* __restrict__ p_nbr_local,
                            double* __restrict__ p_w64, Edge* __restrict__ p_edges) {
    const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= D) return;
    const unsigned lane = lane_id();
    const uint32_t v = dests[w];
    const uint64_t b = offsets[v], e = offsets[v + 1];
    uint64_t pos = p_offsets[w];
    const unsigned lt = (1u << lane) - 1u;
    for (uint64_t j0 = b; j0 < e; j0 += 32) {
        const uint64_t j = j0 + lane;
        const uint32_t u = j < e ? __ldg(nbrs + j) : 0u;
        const bool keep = j < e && bit_of(parent_bits, u);
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const uint64_t k = pos + __popc(mask & lt);
            const double wt = w64[j];
            p_nbr_local[k] = rank_of(src_bits, src_prefix, u);
            p_w64[k] = wt;
            p_edges[k] = make_uint2(rank_of(parent_bits, parent_prefix, u),
                                    __float_as_uint(static_cast<float>(wt)));
        }
        pos += __popc(mask);
    }
}

__global__ void k_src_pos(const uint32_t* __restrict__ src, uint32_t S,
                          const uint32_t* __restrict__ parent_bits, const uint32_t* __restrict__ parent_prefix,
                          uint32_t* __restrict__ srcpos) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < S) srcpos[s] = rank_of(parent_bits, parent_prefix, src[s]);
}

__global__ void k_remap(const Edge* __restrict__ in, uint64_t E, const uint32_t* __restrict__ map,
                        Edge* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < E) {
        const Edge e = in[i];
        out[i] = make_uint2(map[e.x], e.y);
    }
}

__global__ void k_pack_local(const uint32_t* __restrict__ nl, const Edge* __restrict__ ep, uint64_t E,
                             Edge* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < E) out[i] = make_uint2(nl[i], ep[i].y);
}

// ---- degree-bucket schedule ---------------------------------------------------

__device__ __forceinline__ int deg_bucket(uint64_t deg) {
    return deg == 0 ? 0 : 64 - __clzll(static_cast<long long>(deg));  // 1..64
}

__global__ void k_bucket_hist(const uint64_t* __restrict__ offsets, uint32_t D,
                              unsigned long long* __restrict__ hist) {
    __shared__ unsigned long long h[65];
    for (int i = threadIdx.x; i < 65; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d < D) atomicAdd(&h[deg_bucket(offsets[d + 1] - offsets[d])], 1ull);
    __syncthreads();
    for (int i = threadIdx.x; i < 65; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void k_bucket_scatter(const uint64_t* __restrict__ offsets, uint32_t D,
                                 unsigned long long* __restrict__ cursor, uint32_t* __restrict__ order) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    const unsigned long long slot = atomicAdd(&cursor[deg_bucket(offsets[d + 1] - offsets[d])], 1ull);
    order[slot] = d;
}

// ---- groups -------------------------------------------------------------

__global__ void k_groups_per_dest(const uint64_t* __restrict__ offsets, uint32_t D, uint32_t gs,
                                  uint64_t* __restrict__ k) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d < D) k[d] = (offsets[d + 1] - offsets[d] + gs - 1) / gs;
}

// one thread per group; its destination by upper_bound over dest_groups
__global__ void k_emit_groups(const uint64_t* __restrict__ offsets, const uint64_t* __restrict__ dest_groups,
                              uint32_t D, uint64_t G, uint32_t gs, uint32_t* __restrict__ gdest,
                              uint64_t* __restrict__ gbegin, uint64_t* __restrict__ gend) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= G) return;
    uint32_t lo = 0, hi = D;  // first d with dest_groups[d+1] > i
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (dest_groups[mid + 1] <= i) lo = mid + 1;
        else hi = mid;
    }
    const uint32_t d = lo;
    const uint64_t b = offsets[d] + (i - dest_groups[d]) * gs;
    const uint64_t end = offsets[d + 1];
    gdest[i] = d;
    gbegin[i] = b;
    gend[i] = b + gs < end ? b + gs : end;
}

// group_cost.cpp:9-24 in closed form. Group sizes are gs except the last
// group r_v of each destination, so worker w's load is
//   dim * (gs * #{i < G : i mod W == w} - sum_{v : last_v mod W == w} (k_v*gs - deg_v))
// and atomic writes are dim * sum_v max(k_v - 1, 0). Exact u64 arithmetic.
__global__ void k_cost_deficits(const uint64_t* __restrict__ offsets, const uint64_t* __restrict__ dest_groups,
                                uint32_t D, uint32_t gs, uint64_t W, unsigned long long* __restrict__ deficit,
                                unsigned long long* __restrict__ extra_groups) {
    extern __shared__ unsigned long long sdef[];
    const bool use_smem = W <= 4096;
    if (use_smem)
        for (uint64_t i = threadIdx.x; i < W; i += blockDim.x) sdef[i] = 0;
    __syncthreads();
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long extra = 0;
    if (d < D) {
        const uint64_t deg = offsets[d + 1] - offsets[d];
        const uint64_t k = dest_groups[d + 1] - dest_groups[d];
        if (k > 0) {
            const uint64_t bin = (dest_groups[d + 1] - 1) % W;
            const unsigned long long def = k * gs - deg;
            if (def) {
                if (use_smem) atomicAdd(&sdef[bin], def);
                else atomicAdd(&deficit[bin], def);
            }
            extra = k - 1;
        }
    }
    extra = warp_sum(extra);
    if (lane_id() == 0 && extra) atomicAdd(extra_groups, extra);
    __syncthreads();
    if (use_smem)
        for (uint64_t i = threadIdx.x; i < W; i += blockDim.x)
            if (sdef[i]) atomicAdd(&deficit[i], sdef[i]);
}

}  // namespace

namespace {
// UINT64_MAX = width-dependent default (measured on B200, Reddit shape):
// narrow rows (<= 8 float4 columns) route destinations with >= 4096 edges to
// the heavy kernel (top layer 4.6 -> 1.2 ms); wide rows keep every
// destination on the main kernel, which already runs at the L2 cap.
std::atomic<uint64_t> g_heavy_min{[] {
    const char* e = std::getenv("PG_HEAVY_MIN_DEG");
    return e ? static_cast<uint64_t>(std::strtoull(e, nullptr, 10)) : UINT64_MAX;
}()};
}  // namespace

uint64_t heavy_min_degree(uint64_t dim, uint64_t range_edges) {
    const uint64_t v = g_heavy_min.load(std::memory_order_relaxed);
    if (v != UINT64_MAX) return v;
    // Measured on B200 (profiles/README.md, Reddit shape, 1/2/4/8 shards):
    // a destination is a tail once its serial chain outlasts the range's
    // bandwidth-bound time, which shrinks with the range's edge count.
    if ((dim + 3) / 4 <= 8) return range_edges > 20000000ull ? 4096 : 2048;
    const uint64_t t = range_edges / 7000;
    return t > 12288 ? 0 : std::max<uint64_t>(t, 2048);
}
void set_heavy_min_degree(uint64_t v) { g_heavy_min.store(v, std::memory_order_relaxed); }
bool heavy_min_forced() { return g_heavy_min.load(std::memory_order_relaxed) != UINT64_MAX; }

void degree_order(const uint64_t* offsets, uint32_t D, DevBuf<uint32_t>& order, cudaStream_t s, DegHist* out_hist) {
    order = DevBuf<uint32_t>(D, s);
    if (out_hist) *out_hist = DegHist{};
    if (D == 0) return;
    DevBuf<unsigned long long> hist(65, s);
    PG_CUDA(cudaMemsetAsync(hist.get(), 0, 65 * 8, s));
    k_bucket_hist<<<grid_for(D, kThreads), kThreads, 0, s>>>(offsets, D, hist.get());
    PG_LAUNCH("k_bucket_hist");
    unsigned long long h[65];
    PG_CUDA(cudaMemcpyAsync(h, hist.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    uint64_t ends[2] = {0, 0};
    PG_CUDA(cudaMemcpyAsync(&ends[0], offsets, 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaMemcpyAsync(&ends[1], offsets + D, 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    if (out_hist) {
        for (int b = 0; b < 65; ++b) out_hist->h[b] = h[b];
        out_hist->edges = ends[1] - ends[0];
    }
    unsigned long long cur[65];
    unsigned long long run = 0;
    for (int b = 64; b >= 0; --b) {  // descending degree bucket
        cur[b] = run;
        run += h[b];
    }
    PG_CUDA(cudaMemcpyAsync(hist.get(), cur, sizeof(cur), cudaMemcpyHostToDevice, s));
    k_bucket_scatter<<<grid_for(D, kThreads), kThreads, 0, s>>>(offsets, D, hist.get(), order.get());
    PG_LAUNCH("k_bucket_scatter");
    PG_CUDA(cudaStreamSynchronize(s));
}

std::unique_ptr<Frontiers> frontiers_compute(const Graph& g, const uint32_t* vt_host, uint64_t k,
                                             uint64_t L) {
    if (L < 1) fail(kConfig, "frontiers: layer count must be >= 1");
    if (k == 0) fail(kConfig, "frontiers: training set is empty");
    for (uint64_t i = 0; i < k; ++i) {
        if (vt_host[i] >= g.n) fail(kConfig, "frontiers: training vertex out of range");
        if (i && vt_host[i] <= vt_host[i - 1]) fail(kConfig, "frontiers: training set must be sorted and unique");
    }
    DeviceGuard dg(g.device);
    cudaStream_t s = lib_stream(g.device);
    auto f = std::make_unique<Frontiers>();
    f->device = g.device;
    f->n = g.n;
    f->L = L;
    f->graph = &g;
    f->levels.resize(L + 1);
    const uint32_t nw = (g.n + 31) / 32;
    const uint64_t avg_deg = g.n ? g.m / g.n : 0;
    {
        Level& l0 = f->levels[0];
        l0.ids = DevBuf<uint32_t>(k, s);
        PG_CUDA(cudaMemcpyAsync(l0.ids.get(), vt_host, k * 4, cudaMemcpyHostToDevice, s));
        l0.bits = DevBuf<uint32_t>(nw, s);
        PG_CUDA(cudaMemsetAsync(l0.bits.get(), 0, static_cast<uint64_t>(nw) * 4, s));
        k_set_bits<<<grid_for(k, kThreads), kThreads, 0, s>>>(l0.ids.get(), k, l0.bits.get());
        PG_LAUNCH("k_set_bits");
        finish_level(l0, g.n, s, false);
    }
    for (uint64_t lv = 0; lv < L; ++lv) {
        Level& cur = f->levels[lv];
        Level& nxt = f->levels[lv + 1];
        nxt.bits = DevBuf<uint32_t>(nw, s);
        PG_CUDA(cudaMemsetAsync(nxt.bits.get(), 0, static_cast<uint64_t>(nw) * 4, s));
        // direction optimisation: push touches sum(deg(level)) edges with
        // atomics, pull touches at most m with early exit
        const bool push = cur.size * std::max<uint64_t>(avg_deg, 1) * 8 < g.m || cur.size * 32 < g.n;
        if (g.m && cur.size) {
            if (push) {
                k_expand_push<<<grid_for(cur.size * 32, kThreads), kThreads, 0, s>>>(
                    g.offsets.get(), g.nbrs.get(), cur.ids.get(), cur.size, nxt.bits.get());
                PG_LAUNCH("k_expand_push");
            } else {
                k_expand_pull<<<grid_for(static_cast<uint64_t>(nw) * 32, kThreads), kThreads, 0, s>>>(
                    g.offsets.get(), g.nbrs.get(), g.n, cur.bits.get(), nxt.bits.get());
                PG_LAUNCH("k_expand_pull");
            }
        }
        finish_level(nxt, g.n, s, true);
    }
    PG_CUDA(cudaStreamSynchronize(s));
    return f;
}

std::unique_ptr<Path> path_extract(const Graph& g, const Frontiers& f, uint64_t layer) {
    const uint64_t L = f.L;
    if (layer >= L) fail(kConfig, "execution path: layer index out of range");
    if (f.graph != &g || f.n != g.n) fail(kConfig, "execution path: frontiers belong to another graph");
    DeviceGuard dg(g.device);
    cudaStream_t s = lib_stream(g.device);
    const Level& dl = f.levels[L - layer];
    const Level& pl = f.levels[L - layer - 1];
    auto p = std::make_unique<Path>();
    p->device = g.device;
    p->layer = layer;
    p->D = static_cast<uint32_t>(dl.size);
    p->P = static_cast<uint32_t>(pl.size);
    const uint32_t D = p->D, P = p->P;
    const uint32_t nw = (g.n + 31) / 32;

    p->dest = DevBuf<uint32_t>(D, s);
    if (D) PG_CUDA(cudaMemcpyAsync(p->dest.get(), dl.ids.get(), static_cast<uint64_t>(D) * 4,
                                   cudaMemcpyDeviceToDevice, s));
    // filtered degrees -> offsets
    DevBuf<uint64_t> kept(D, s);
    if (D) {
        k_count_kept<<<grid_for(static_cast<uint64_t>(D) * 32, kThreads), kThreads, 0, s>>>(
            g.offsets.get(), g.nbrs.get(), p->dest.get(), D, pl.bits.get(), kept.get());
        PG_LAUNCH("k_count_kept");
    }
    p->offsets = DevBuf<uint64_t>(static_cast<uint64_t>(D) + 1, s);
    {
        DevBuf<uint64_t> scratch(scan_scratch_elems(D), s);
        exclusive_scan(kept.get(), D, p->offsets.get(), scratch.get(), s);
    }
    PG_CUDA(cudaMemcpyAsync(&p->E, p->offsets.get() + D, 8, cudaMemcpyDeviceToHost, s));
    // referenced sources (sorted by construction) and their ranks
    Level srcl;
    srcl.bits = DevBuf<uint32_t>(nw, s);
    PG_CUDA(cudaMemsetAsync(srcl.bits.get(), 0, static_cast<uint64_t>(nw) * 4, s));
    if (P && D) {
        k_mark_sources<<<grid_for(static_cast<uint64_t>(P) * 32, kThreads), kThreads, 0, s>>>(
            g.offsets.get(), g.nbrs.get(), pl.ids.get(), P, dl.bits.get(), srcl.bits.get());
        PG_LAUNCH("k_mark_sources");
    }
    finish_level(srcl, g.n, s, true);  // syncs; p->E is now valid
    p->S = static_cast<uint32_t>(srcl.size);
    p->src = std::move(srcl.ids);
    p->srcpos = DevBuf<uint32_t>(p->S, s);
    if (p->S) {
        k_src_pos<<<grid_for(p->S, kThreads), kThreads, 0, s>>>(p->src.get(), p->S, pl.bits.get(),
                                                               pl.prefix.get(), p->srcpos.get());
        PG_LAUNCH("k_src_pos");
    }
    const uint64_t E = p->E;
    p->nbr_local = DevBuf<uint32_t>(E, s);
    p->w64 = DevBuf<double>(E, s);
    p->edges_parent = edge_buf(E, s);
    if (D && E) {
        k_fill_path<<<grid_for(static_cast<uint64_t>(D) * 32, kThreads), kThreads, 0, s>>>(
            g.offsets.get(), g.nbrs.get(), g.w64.get(), p->dest.get(), D, pl.bits.get(), pl.prefix.get(),
            srcl.bits.get(), srcl.prefix.get(), p->offsets.get(), p->nbr_local.get(), p->w64.get(),
            p->edges_parent.get());
        PG_LAUNCH("k_fill_path");
    }
    degree_order(p->offsets.get(), D, p->order, s, &p->hist);
    p->max_degree = max_degree_dev(p->offsets.get(), D, s);
    PG_CUDA(cudaStreamSynchronize(s));
    return p;
}

namespace {
__global__ void k_segment_bounds(const uint64_t* __restrict__ offsets, const Edge* __restrict__ edges, uint32_t D,
                                 const uint64_t* __restrict__ cuts, uint32_t K, uint64_t* __restrict__ bnd) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<uint64_t>(D) * (K + 1)) return;
    const uint32_t k = static_cast<uint32_t>(i / D), d = static_cast<uint32_t>(i % D);
    const uint64_t b = offsets[d], e = offsets[d + 1];
    if (k == K) {
        bnd[i] = e;
        return;
    }
    const uint64_t c = cuts[k];
    uint64_t lo = b, hi = e;  // first edge with source row >= c
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (edges[mid].x < c) lo = mid + 1;
        else hi = mid;
    }
    bnd[i] = lo;
}
}  // namespace

void segment_bounds(const uint64_t* offsets, const Edge* edges, uint32_t D, const uint64_t* cuts_host, uint32_t K,
                    DevBuf<uint64_t>& bnd, cudaStream_t s) {
    retire(bnd);  // the previous bounds may still be read on a caller stream
    bnd = DevBuf<uint64_t>(static_cast<uint64_t>(D) * (K + 1), s);
    if (!D) return;
    DevBuf<uint64_t> cuts(K + 1, s);
    PG_CUDA(cudaMemcpyAsync(cuts.get(), cuts_host, (K + 1) * 8, cudaMemcpyHostToDevice, s));
    k_segment_bounds<<<grid_for(static_cast<uint64_t>(D) * (K + 1), kThreads), kThreads, 0, s>>>(
        offsets, edges, D, cuts.get(), K, bnd.get());
    PG_LAUNCH("k_segment_bounds");
    PG_CUDA(cudaStreamSynchronize(s));
}

namespace {
__global__ void k_src_counts(const Edge* __restrict__ edges, uint64_t E, uint32_t* __restrict__ counts) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < E;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        atomicAdd(counts + edges[i].x, 1u);
}
}  // namespace

void source_edge_counts(const Edge* edges, uint64_t E, uint64_t P, uint32_t* counts, cudaStream_t s) {
    if (P) PG_CUDA(cudaMemsetAsync(counts, 0, P * 4, s));
    if (!E) return;
    k_src_counts<<<148 * 16, kThreads, 0, s>>>(edges, E, counts);
    PG_LAUNCH("k_src_counts");
}

void remap_edges(const Edge* in, uint64_t E, const uint32_t* map, Edge* out, cudaStream_t s) {
    if (E == 0) return;
    k_remap<<<grid_for(E, kThreads), kThreads, 0, s>>>(in, E, map, out);
    PG_LAUNCH("k_remap");
}

void path_pack_local(Path& p, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(p.mu);
    if (p.edges_local.get() || p.E == 0 || p.S == p.P) return;
    p.edges_local = edge_buf(p.E, s);
    k_pack_local<<<grid_for(p.E, kThreads), kThreads, 0, s>>>(p.nbr_local.get(), p.edges_parent.get(), p.E,
                                                            p.edges_local.get());
    PG_LAUNCH("k_pack_local");
}

std::unique_ptr<Groups> groups_build(uint32_t D, const uint64_t* offsets_dev, uint32_t gs, int device) {
    if (gs == 0) fail(kConfig, "group size must be at least 1");
    DeviceGuard dg(device);
    cudaStream_t s = lib_stream(device);
    auto G = std::make_unique<Groups>();
    G->device = device;
    G->gs = gs;
    DevBuf<uint64_t> k(D, s);
    if (D) {
        k_groups_per_dest<<<grid_for(D, kThreads), kThreads, 0, s>>>(offsets_dev, D, gs, k.get());
        PG_LAUNCH("k_groups_per_dest");
    }
    G->dest_groups = DevBuf<uint64_t>(static_cast<uint64_t>(D) + 1, s);
    DevBuf<uint64_t> scratch(scan_scratch_elems(D), s);
    exclusive_scan(k.get(), D, G->dest_groups.get(), scratch.get(), s);
    PG_CUDA(cudaMemcpyAsync(&G->G, G->dest_groups.get() + D, 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    G->gdest = DevBuf<uint32_t>(G->G, s);
    G->gbegin = DevBuf<uint64_t>(G->G, s);
    G->gend = DevBuf<uint64_t>(G->G, s);
    if (G->G) {
        k_emit_groups<<<grid_for(G->G, kThreads), kThreads, 0, s>>>(offsets_dev, G->dest_groups.get(), D, G->G,
                                                                   gs, G->gdest.get(), G->gbegin.get(),
                                                                   G->gend.get());
        PG_LAUNCH("k_emit_groups");
    }
    PG_CUDA(cudaStreamSynchronize(s));
    return G;
}

void grouping_cost_dev(uint32_t D, const uint64_t* offsets_dev, uint32_t gs, uint64_t dim, uint64_t workers,
                       uint64_t* max_load, uint64_t* atomic_writes, cudaStream_t s) {
    if (workers < 1) fail(kConfig, "cost model: worker count must be >= 1");
    if (gs == 0) fail(kConfig, "group size must be at least 1");
    DevBuf<uint64_t> k(D, s), dest_groups(static_cast<uint64_t>(D) + 1, s);
    if (D) {
        k_groups_per_dest<<<grid_for(D, kThreads), kThreads, 0, s>>>(offsets_dev, D, gs, k.get());
        PG_LAUNCH("k_groups_per_dest");
    }
    {
        DevBuf<uint64_t> scratch(scan_scratch_elems(D), s);
        exclusive_scan(k.get(), D, dest_groups.get(), scratch.get(), s);
    }
    DevBuf<unsigned long long> deficit(workers + 1, s);
    PG_CUDA(cudaMemsetAsync(deficit.get(), 0, (workers + 1) * 8, s));
    if (D) {
        const size_t smem = workers <= 4096 ? workers * 8 : 0;
        k_cost_deficits<<<grid_for(D, kThreads), kThreads, smem, s>>>(offsets_dev, dest_groups.get(), D, gs,
                                                                     workers, deficit.get(),
                                                                     deficit.get() + workers);
        PG_LAUNCH("k_cost_deficits");
    }
    std::vector<unsigned long long> h(workers + 1);
    uint64_t G = 0;
    PG_CUDA(cudaMemcpyAsync(h.data(), deficit.get(), (workers + 1) * 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaMemcpyAsync(&G, dest_groups.get() + D, 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    uint64_t best = 0;
    for (uint64_t w = 0; w < workers; ++w) {
        const uint64_t cnt = G / workers + (w < G % workers ? 1 : 0);
        const uint64_t load = (static_cast<uint64_t>(gs) * cnt - h[w]) * dim;
        best = std::max(best, load);
    }
    *max_load = best;
    *atomic_writes = h[workers] * dim;
}

}  // namespace pg
