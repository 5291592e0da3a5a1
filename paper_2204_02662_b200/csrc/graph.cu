// Graph load on device: the reference's build_undirected_csr +
// assign_edge_weights (csr_graph.cpp:33-77), bit-exact.
//   directed keys u<<32|v (self loops dropped) -> radix sort (CUB) -> unique
//   (flag + scan compaction) -> row offsets by binary search -> weights.
// Sym-norm weights are 1/sqrt(du*dv) in f64: CUDA's double sqrt and '/' are
// IEEE round-to-nearest, as on the host, so the weights are bit-identical.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <mutex>
#include <vector>

#include "pg_internal.h"

namespace pg {

__global__ void k_scan_sums(uint64_t* sums, uint64_t nb) {
    // one block of kScanThreads; in-place exclusive scan of the tile sums
    uint64_t carry = 0;
    for (uint64_t b0 = 0; b0 < nb; b0 += kScanTile) {
        const uint64_t base = b0 + threadIdx.x * kScanItems;
        uint64_t v[kScanItems];
        uint64_t loc = 0;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            v[i] = base + i < nb ? sums[base + i] : 0;
            loc += v[i];
        }
        uint64_t total;
        uint64_t run = carry + block_excl_scan(loc, total);
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            if (base + i < nb) sums[base + i] = run;
            run += v[i];
        }
        carry += total;
    }
}

namespace {

std::mutex g_stream_mu;
std::vector<cudaStream_t> g_streams;

__global__ void k_make_keys(const uint32_t* __restrict__ pairs, uint64_t np, uint32_t n,
                            uint64_t* __restrict__ keys) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= np) return;
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    // self loops sort after every real key (u < n) and are dropped
    const uint64_t sentinel = static_cast<uint64_t>(n) << 32;
    keys[2 * i] = u == v ? sentinel : (static_cast<uint64_t>(u) << 32) | v;
    keys[2 * i + 1] = u == v ? sentinel : (static_cast<uint64_t>(v) << 32) | u;
}

__global__ void k_max_id(const uint32_t* __restrict__ pairs, uint64_t np,
                         unsigned long long* __restrict__ out) {
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    uint32_t best = 0;
    unsigned any = 0;
    for (; i < np; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
        if (u != v) {
            any = 1;
            best = max(best, max(u, v));
        }
    }
    best = __reduce_max_sync(0xffffffffu, best);
    any = __reduce_or_sync(0xffffffffu, any);
    if (lane_id() == 0 && any) atomicMax(out, static_cast<unsigned long long>(best) + 1ull);
    if (lane_id() == 0 && any) atomicOr(out + 1, 1ull);
}

__global__ void k_unique_flags(const uint64_t* __restrict__ keys, uint64_t nk, uint64_t sentinel,
                               uint32_t* __restrict__ flags) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= nk) return;
    const uint64_t k = keys[i];
    flags[i] = (k < sentinel && (i == 0 || keys[i - 1] != k)) ? 1u : 0u;
}

__global__ void k_unique_scatter(const uint64_t* __restrict__ keys, uint64_t nk,
                                 const uint32_t* __restrict__ flags,
                                 const uint64_t* __restrict__ pos, uint64_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= nk || !flags[i]) return;
    out[pos[i]] = keys[i];
}

// offsets[u] = first index with key >= u<<32 (sorted unique keys)
__global__ void k_row_offsets(const uint64_t* __restrict__ keys, uint64_t m, uint32_t n,
                              uint64_t* __restrict__ offsets) {
    const uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (u > n) return;
    const uint64_t target = u << 32;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (keys[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    offsets[u] = lo;
}

__global__ void k_low_words(const uint64_t* __restrict__ keys, uint64_t m,
                            uint32_t* __restrict__ nbrs) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < m) nbrs[i] = static_cast<uint32_t>(keys[i]);
}

// csr_graph.cpp:65-77; warp per row
__global__ void k_weights(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                          uint32_t n, int symnorm, double* __restrict__ w) {
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (warp >= n) return;
    const uint32_t u = static_cast<uint32_t>(warp);
    const uint64_t b = offsets[u], e = offsets[u + 1];
    const double du = static_cast<double>(e - b);
    for (uint64_t j = b + lane_id(); j < e; j += 32) {
        if (!symnorm) {
            w[j] = 1.0;
            continue;
        }
        const uint32_t v = nbrs[j];
        const double dv = static_cast<double>(offsets[v + 1] - offsets[v]);
        w[j] = 1.0 / sqrt(du * dv);
    }
}

// CsrGraph invariants (csr_graph.hpp:15-18): rows sorted, duplicate free,
// ids < n, symmetric with equal weights. Warp per row; err bit set on failure.
__global__ void k_validate(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs,
                           const double* __restrict__ w, uint32_t n, unsigned* __restrict__ err) {
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (warp >= n) return;
    const uint32_t v = static_cast<uint32_t>(warp);
    const uint64_t b = offsets[v], e = offsets[v + 1];
    if (e < b) {
        if (lane_id() == 0) atomicOr(err, 1u);
        return;
    }
    for (uint64_t j = b + lane_id(); j < e; j += 32) {
        const uint32_t u = nbrs[j];
        unsigned bad = 0;
        if (u >= n) bad |= 2u;
        else if (j > b && nbrs[j - 1] >= u) bad |= 4u;
        else {
            // find v in N(u)
            uint64_t lo = offsets[u], hi = offsets[u + 1];
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (nbrs[mid] < v) lo = mid + 1;
                else hi = mid;
            }
            if (lo == offsets[u + 1] || nbrs[lo] != v) bad |= 8u;
            else if (__double_as_longlong(w[lo]) != __double_as_longlong(w[j])) bad |= 16u;
        }
        if (bad) atomicOr(err, bad);
    }
}

__global__ void k_pack_edges(const uint32_t* __restrict__ nbrs, const double* __restrict__ w,
                             uint64_t m, Edge* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < m) out[i] = make_uint2(nbrs[i], __float_as_uint(static_cast<float>(w[i])));
}

__global__ void k_max_degree(const uint64_t* __restrict__ offsets, uint32_t n,
                             unsigned* __restrict__ out) {
    uint32_t best = 0;
    for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        best = max(best, static_cast<uint32_t>(offsets[v + 1] - offsets[v]));
    best = __reduce_max_sync(0xffffffffu, best);
    if (lane_id() == 0) atomicMax(out, best);
}

}  // namespace

uint32_t max_degree_dev(const uint64_t* offsets, uint32_t n, cudaStream_t s) {
    if (n == 0) return 0;
    DevBuf<unsigned> d(1, s);
    PG_CUDA(cudaMemsetAsync(d.get(), 0, 4, s));
    k_max_degree<<<std::min<uint64_t>(grid_for(n, 256), 4096), 256, 0, s>>>(offsets, n, d.get());
    PG_LAUNCH("k_max_degree");
    unsigned h = 0;
    PG_CUDA(cudaMemcpyAsync(&h, d.get(), 4, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    return h;
}

uint64_t& launch_counter() {
    static uint64_t n = 0;
    return n;
}

cudaStream_t lib_stream(int device) {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    if (static_cast<int>(g_streams.size()) <= device) g_streams.resize(device + 1, nullptr);
    if (!g_streams[device]) {
        DeviceGuard dg(device);
        PG_CUDA(cudaStreamCreateWithFlags(&g_streams[device], cudaStreamNonBlocking));
        // keep freed stream-ordered allocations in the pool instead of
        // returning them to the driver at every synchronisation (the
        // host-buffer calls stage ~GBs per call)
        cudaMemPool_t pool;
        PG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        PG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    return g_streams[device];
}

void graph_assign_weights(Graph& g, int weight_mode, cudaStream_t s) {
    if (g.m == 0) return;
    k_weights<<<grid_for(static_cast<uint64_t>(g.n) * 32, 256), 256, 0, s>>>(
        g.offsets.get(), g.nbrs.get(), g.n, weight_mode ? 1 : 0, g.w64.get());
    PG_LAUNCH("k_weights");
    g.edges.reset();
}

void graph_pack_edges(Graph& g, cudaStream_t s) {
    if (g.edges.get() || g.m == 0) return;
    g.edges = edge_buf(g.m, s);
    k_pack_edges<<<grid_for(g.m, 256), 256, 0, s>>>(g.nbrs.get(), g.w64.get(), g.m, g.edges.get());
    PG_LAUNCH("k_pack_edges");
}

std::unique_ptr<Graph> graph_build(int device, int64_t n_hint, const uint32_t* pairs_host,
                                   uint64_t npairs, int weight_mode) {
    DeviceGuard dg(device);
    cudaStream_t s = lib_stream(device);
    auto g = std::make_unique<Graph>();
    g->device = device;

    DevBuf<uint32_t> pairs(2 * npairs, s);
    if (npairs)
        PG_CUDA(cudaMemcpyAsync(pairs.get(), pairs_host, 2 * npairs * 4, cudaMemcpyHostToDevice, s));
    // n = max(n_hint, 1 + max id over non-self-loop pairs) (csr_graph.cpp:34-40)
    unsigned long long mx[2] = {0, 0};
    if (npairs) {
        DevBuf<unsigned long long> dmx(2, s);
        PG_CUDA(cudaMemsetAsync(dmx.get(), 0, 16, s));
        k_max_id<<<std::min<uint64_t>(grid_for(npairs, 256), 8192), 256, 0, s>>>(pairs.get(), npairs, dmx.get());
        PG_LAUNCH("k_max_id");
        PG_CUDA(cudaMemcpyAsync(mx, dmx.get(), 16, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
    }
    const bool any = mx[1] != 0;
    if (!any && n_hint < 0)
        fail(kConfig, "cannot build a graph from an empty edge list without a vertex-count hint");
    uint64_t n64 = n_hint >= 0 ? static_cast<uint64_t>(n_hint) : 0;
    n64 = std::max<uint64_t>(n64, mx[0]);
    if (n64 >= 0xFFFFFFFFull) fail(kConfig, "graph: vertex count exceeds 32-bit ids");
    const uint32_t n = static_cast<uint32_t>(n64);
    g->n = n;

    const uint64_t nk = 2 * npairs;
    uint64_t m = 0;
    DevBuf<uint64_t> uniq;
    if (nk) {
        DevBuf<uint64_t> keys(nk, s), sorted(nk, s);
        k_make_keys<<<grid_for(npairs, 256), 256, 0, s>>>(pairs.get(), npairs, n, keys.get());
        PG_LAUNCH("k_make_keys");
        pairs.reset();
        int hi_bits = 1;
        while ((1ull << hi_bits) <= n64) ++hi_bits;
        const int end_bit = std::min(64, 32 + hi_bits);
        size_t tmp_bytes = 0;
        PG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.get(), sorted.get(), nk, 0,
                                               end_bit, s));
        {
            DevBuf<unsigned char> tmp(tmp_bytes, s);
            PG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tmp_bytes, keys.get(), sorted.get(),
                                                   nk, 0, end_bit, s));
        }
        keys.reset();
        DevBuf<uint32_t> flags(nk, s);
        DevBuf<uint64_t> pos(nk + 1, s);
        DevBuf<uint64_t> scratch(scan_scratch_elems(nk), s);
        const uint64_t sentinel = static_cast<uint64_t>(n) << 32;
        k_unique_flags<<<grid_for(nk, 256), 256, 0, s>>>(sorted.get(), nk, sentinel, flags.get());
        PG_LAUNCH("k_unique_flags");
        exclusive_scan(flags.get(), nk, pos.get(), scratch.get(), s);
        PG_CUDA(cudaMemcpyAsync(&m, pos.get() + nk, 8, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
        uniq = DevBuf<uint64_t>(m, s);
        k_unique_scatter<<<grid_for(nk, 256), 256, 0, s>>>(sorted.get(), nk, flags.get(), pos.get(),
                                                         uniq.get());
        PG_LAUNCH("k_unique_scatter");
    }
    g->m = m;
    g->offsets = DevBuf<uint64_t>(static_cast<uint64_t>(n) + 1, s);
    g->nbrs = DevBuf<uint32_t>(m, s);
    g->w64 = DevBuf<double>(m, s);
    k_row_offsets<<<grid_for(static_cast<uint64_t>(n) + 1, 256), 256, 0, s>>>(uniq.get(), m, n,
                                                                             g->offsets.get());
    PG_LAUNCH("k_row_offsets");
    if (m) {
        k_low_words<<<grid_for(m, 256), 256, 0, s>>>(uniq.get(), m, g->nbrs.get());
        PG_LAUNCH("k_low_words");
    }
    uniq.reset();
    graph_assign_weights(*g, weight_mode, s);
    g->max_degree = max_degree_dev(g->offsets.get(), n, s);
    PG_CUDA(cudaStreamSynchronize(s));
    return g;
}

std::unique_ptr<Graph> graph_upload(int device, uint32_t n, const uint64_t* offsets,
                                    const uint32_t* nbrs, const double* w, bool validate) {
    DeviceGuard dg(device);
    cudaStream_t s = lib_stream(device);
    auto g = std::make_unique<Graph>();
    g->device = device;
    g->n = n;
    if (offsets[0] != 0) fail(kConfig, "graph: offsets[0] must be 0");
    g->m = offsets[n];
    g->offsets = DevBuf<uint64_t>(static_cast<uint64_t>(n) + 1, s);
    g->nbrs = DevBuf<uint32_t>(g->m, s);
    g->w64 = DevBuf<double>(g->m, s);
    PG_CUDA(cudaMemcpyAsync(g->offsets.get(), offsets, (static_cast<uint64_t>(n) + 1) * 8,
                            cudaMemcpyHostToDevice, s));
    if (g->m) {
        PG_CUDA(cudaMemcpyAsync(g->nbrs.get(), nbrs, g->m * 4, cudaMemcpyHostToDevice, s));
        PG_CUDA(cudaMemcpyAsync(g->w64.get(), w, g->m * 8, cudaMemcpyHostToDevice, s));
    }
    if (validate && n) {
        DevBuf<unsigned> err(1, s);
        PG_CUDA(cudaMemsetAsync(err.get(), 0, 4, s));
        k_validate<<<grid_for(static_cast<uint64_t>(n) * 32, 256), 256, 0, s>>>(
            g->offsets.get(), g->nbrs.get(), g->w64.get(), n, err.get());
        PG_LAUNCH("k_validate");
        unsigned h = 0;
        PG_CUDA(cudaMemcpyAsync(&h, err.get(), 4, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
        if (h & 1u) fail(kConfig, "graph: offsets are not non-decreasing");
        if (h & 2u) fail(kConfig, "graph: neighbor id out of range");
        if (h & 4u) fail(kConfig, "graph: neighbor lists must be sorted and duplicate-free");
        if (h & 8u) fail(kConfig, "graph: adjacency is not symmetric");
        if (h & 16u) fail(kConfig, "graph: weight(u->v) != weight(v->u)");
    }
    g->max_degree = max_degree_dev(g->offsets.get(), n, s);
    PG_CUDA(cudaStreamSynchronize(s));
    return g;
}

}  // namespace pg
