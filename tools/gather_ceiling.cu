// Microbenchmark: the ceiling of the SpMM's access pattern on this GPU.
// A warp gathers 512-byte rows (one float4 per lane) at random row indices,
// U = 8 independent gathers in flight per lane, and sums them (so nothing is
// dead code). Measured over a source matrix that fits in L2 (the rate the
// layer-0 SpMM sees for L2-resident hub rows) and one that does not (random
// 512-B gathers from HBM), next to a plain streaming read. Bytes counted =
// rows x 512 B requested (the SpMM's "algorithmic" gather bytes).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_ceiling tools/gather_ceiling.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

template <int U>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ src, uint32_t rows_mask,
                                                const uint32_t* __restrict__ idx, uint64_t n_items, int per_item,
                                                float4* __restrict__ out) {
    const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= n_items) return;
    const unsigned lane = threadIdx.x & 31;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t* ix = idx + w * per_item;
    for (int e = 0; e < per_item; e += U) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t r = __ldg(ix + e + u) & rows_mask;
            x[u] = __ldg(src + static_cast<uint64_t>(r) * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc.x += x[u].x;
            acc.y += x[u].y;
            acc.z += x[u].z;
            acc.w += x[u].w;
        }
    }
    out[w * 32 + lane] = acc;
}

__global__ void k_stream(const float4* __restrict__ src, uint64_t n, float4* __restrict__ out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float4 v = __ldg(src + i);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    out[blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x] = acc;
}

int main() {
    const int per_item = 512;          // gathers per warp
    const uint64_t n_items = 148 * 64;  // warps
    const uint64_t n_idx = n_items * per_item;
    std::vector<uint32_t> h(n_idx);
    uint64_t s = 88172645463325252ull;
    for (auto& v : h) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        v = static_cast<uint32_t>(s >> 20);
    }
    uint32_t* idx;
    CK(cudaMalloc(&idx, n_idx * 4));
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    float4* out;
    CK(cudaMalloc(&out, n_items * 32 * 16));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint64_t big_rows = 1u << 22;  // 4M rows x 512 B = 2 GB
    float4* src;
    CK(cudaMalloc(&src, big_rows * 512));
    CK(cudaMemset(src, 0, big_rows * 512));
    for (uint32_t rows : {1u << 15, 1u << 16, 1u << 17, 1u << 18, 1u << 20, 1u << 22}) {  // 16 MB .. 2 GB
        const uint32_t mask = rows - 1;
        for (int rep = 0; rep < 2; ++rep) k_gather<8><<<n_items * 32 / 256, 256>>>(src, mask, idx, n_items, per_item, out);
        CK(cudaEventRecord(a));
        const int R = 10;
        for (int rep = 0; rep < R; ++rep) k_gather<8><<<n_items * 32 / 256, 256>>>(src, mask, idx, n_items, per_item, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = static_cast<double>(n_idx) * 512 * R;
        std::printf("gather 512B rows, source %6.0f MB: %8.1f GB/s\n", rows * 512.0 / 1e6, bytes / (ms * 1e-3) / 1e9);
    }
    {
        const uint64_t n = big_rows * 32;
        k_stream<<<148 * 8, 256>>>(src, n, out);
        CK(cudaEventRecord(a));
        for (int rep = 0; rep < 5; ++rep) k_stream<<<148 * 8, 256>>>(src, n, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("stream read 2 GB: %8.1f GB/s\n", n * 16.0 * 5 / (ms * 1e-3) / 1e9);
    }
    return 0;
}
