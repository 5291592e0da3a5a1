// Shared device helpers for the pathgcn B200 path: error plumbing, warp/block
// scans, bitmap ranks and the device-wide exclusive scan used by every
// compaction (frontiers, path offsets, group offsets).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace pg {

// Status codes of the C ABI. 2/3/4 follow the reference's error taxonomy and
// CLI exit codes (error.hpp:10-47, main.cpp:383-406); 5 is new: a CUDA
// runtime/device failure.
enum Status : int { kOk = 0, kConfig = 2, kIo = 3, kNumeric = 4, kDevice = 5 };
// The reference exception type behind a status (error.hpp:10-47), carried
// across the ABI by pg_last_error_kind (PG_KIND_* in pathgcn_b200.h) so the
// C++ and Python wrappers rethrow the exact subtype instead of guessing it
// from the message.
enum Kind : int { kKindNone = 0, kKindConfig = 1, kKindShape = 2, kKindStaleness = 3, kKindParse = 4,
                  kKindIo = 5, kKindNumeric = 6, kKindDevice = 7 };

inline int kind_of_status(int code) {
    return code == kConfig ? kKindConfig : code == kIo ? kKindIo : code == kNumeric ? kKindNumeric
         : code == kDevice ? kKindDevice : kKindNone;
}

struct Error : std::runtime_error {
    int code;
    int kind;
    uint64_t line = 0;  // ParseError::line_number
    Error(int c, const std::string& m) : std::runtime_error(m), code(c), kind(kind_of_status(c)) {}
    Error(int c, int k, const std::string& m, uint64_t ln = 0) : std::runtime_error(m), code(c), kind(k), line(ln) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
// ShapeError / StalenessError / ParseError (status 2, error.hpp:18-31)
[[noreturn]] inline void fail_shape(const std::string& msg) { throw Error(kConfig, kKindShape, msg); }
[[noreturn]] inline void fail_stale(const std::string& msg) { throw Error(kConfig, kKindStaleness, msg); }
[[noreturn]] inline void fail_parse(const std::string& msg, uint64_t line) {
    throw Error(kConfig, kKindParse, msg + " (line " + std::to_string(line) + ")", line);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(kDevice, std::string(what) + ": " + cudaGetErrorString(e));
}
#define PG_CUDA(x) ::pg::cuda_check((x), #x)
// every kernel launch of the library goes through PG_LAUNCH: it checks the
// launch and counts it (pg_launch_count, the bench's gpu_launches)
uint64_t& launch_counter();
inline void launched(const char* what) {
    cuda_check(cudaGetLastError(), what);
    __atomic_fetch_add(&launch_counter(), 1, __ATOMIC_RELAXED);
}
#define PG_LAUNCH(what) ::pg::launched(what)

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, v, o);
        if (static_cast<int>(lane_id()) >= o) v += t;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive block scan of one value per thread (blockDim.x multiple of 32).
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t& total) {
    __shared__ uint64_t warp_tot[32];
    const unsigned lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t inc = warp_incl_scan(v);
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint64_t s = lane < nw ? warp_tot[lane] : 0;
        warp_tot[lane] = warp_incl_scan(s);
    }
    __syncthreads();
    const uint64_t base = wid ? warp_tot[wid - 1] : 0;
    total = warp_tot[nw - 1];
    __syncthreads();
    return base + inc - v;
}

// Membership bit and rank (number of set bits strictly below u).
__device__ __forceinline__ bool bit_of(const uint32_t* __restrict__ bits, uint32_t u) {
    return (__ldg(bits + (u >> 5)) >> (u & 31)) & 1u;
}
__device__ __forceinline__ uint32_t rank_of(const uint32_t* __restrict__ bits,
                                            const uint32_t* __restrict__ word_prefix, uint32_t u) {
    const uint32_t w = __ldg(bits + (u >> 5));
    return __ldg(word_prefix + (u >> 5)) + __popc(w & ((1u << (u & 31)) - 1u));
}

// ---- device-wide exclusive scan: out[0..n] with out[n] = total ----------
template <typename Tin>
__global__ void k_tile_sums(const Tin* __restrict__ in, uint64_t n, uint64_t* __restrict__ sums) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += static_cast<uint64_t>(in[base + i]);
    uint64_t total;
    block_excl_scan(s, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void k_scan_sums(uint64_t* sums, uint64_t nb);

template <typename Tin, typename Tout>
__global__ void k_scan_tiles(const Tin* __restrict__ in, uint64_t n,
                             const uint64_t* __restrict__ tile_off, Tout* __restrict__ out) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t loc = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? static_cast<uint64_t>(in[base + i]) : 0;
        loc += v[i];
    }
    uint64_t total;
    uint64_t run = tile_off[blockIdx.x] + block_excl_scan(loc, total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = static_cast<Tout>(run);
        run += v[i];
        if (base + i + 1 == n) out[n] = static_cast<Tout>(run);
    }
}

// Scratch sized for exclusive_scan over n elements.
inline uint64_t scan_scratch_elems(uint64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

// out[0..n]: exclusive prefix sums of in[0..n), out[n] = total. `scratch`
// holds scan_scratch_elems(n) u64. Stream-ordered.
template <typename Tin, typename Tout>
void exclusive_scan(const Tin* in, uint64_t n, Tout* out, uint64_t* scratch, cudaStream_t s) {
    if (n == 0) {
        PG_CUDA(cudaMemsetAsync(out, 0, sizeof(Tout), s));
        return;
    }
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    k_tile_sums<Tin><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, scratch);
    PG_LAUNCH("k_tile_sums");
    k_scan_sums<<<1, kScanThreads, 0, s>>>(scratch, nb);
    PG_LAUNCH("k_scan_sums");
    k_scan_tiles<Tin, Tout><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, scratch, out);
    PG_LAUNCH("k_scan_tiles");
}

// RAII device buffer (stream-ordered allocator).
template <typename T>
struct DevBuf {
    T* p = nullptr;
    uint64_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(uint64_t count, cudaStream_t st) : n(count), s(st) {
        if (count) PG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p; n = o.n; s = o.s;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// Cached device buffers (schedules, segment bounds, remapped edge streams)
// are read by kernels on CALLER streams but were allocated on the library
// stream, so a cudaFreeAsync on that idle stream is not ordered after those
// kernels. Replacing or destroying one therefore drains the device first
// (rare: a knob change, a remap, a handle destroy).
inline void drain_device() { PG_CUDA(cudaDeviceSynchronize()); }
template <typename T>
void retire(DevBuf<T>& b) {
    if (b.p) {
        drain_device();
        b.reset();
    }
}

inline unsigned grid_for(uint64_t work, unsigned per_block) {
    uint64_t g = (work + per_block - 1) / per_block;
    return static_cast<unsigned>(g ? g : 1);
}

}  // namespace pg
