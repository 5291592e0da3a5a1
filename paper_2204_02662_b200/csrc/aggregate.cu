// Backward aggregation SpMM over an execution path, bit-exact with the
// reference's aggregate_pull<float> Deterministic (aggregate.hpp:69-83):
// every output element is accumulated in ascending edge order as
//   acc = fl(acc + fl(w_e * x))   (no FMA contraction, like the x86-64
// reference build), then acc = fl(acc + 0) to canonicalise -0.
//
// Work decomposition: a (sub-)warp owns one (destination, 32-float4 column
// chunk); lanes own float4 columns, so each edge costs one coalesced 128-bit
// gather per lane (512 B per warp). Rows of one destination never split
// across edges (that would change the fp32 summation order), so hubs are
// parallelised across column chunks and scheduled first: `order` lists
// destinations by descending degree bucket. Memory-level parallelism comes
// from U edges in flight per lane (U independent LDG.128 before the ordered
// adds). The gather of gradient rows (engine.hpp:334) is folded into the
// packed edge record (src_pos_in_parent composed at path build).
#include "pg_internal.h"

namespace pg {

namespace {

__device__ __forceinline__ float4 ldg4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ void acc4(float4& a, float w, const float4& x) {
    a.x = __fadd_rn(a.x, __fmul_rn(w, x.x));
    a.y = __fadd_rn(a.y, __fmul_rn(w, x.y));
    a.z = __fadd_rn(a.z, __fmul_rn(w, x.z));
    a.w = __fadd_rn(a.w, __fmul_rn(w, x.w));
}

// LPD lanes per (destination, chunk); each lane one float4 column.
template <int LPD, int U>
__global__ void __launch_bounds__(256) k_agg_vec4(const uint64_t* __restrict__ offsets,
                                                 const Edge* __restrict__ edges,
                                                 const uint32_t* __restrict__ order, uint32_t d_begin,
                                                 uint64_t n_items, uint32_t chunks,
                                                 const float* __restrict__ in, uint64_t ld_in,
                                                 float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                 int accumulate) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    if (item >= n_items) return;
    const uint32_t d = order[d_begin + item / chunks];
    const uint32_t q = static_cast<uint32_t>(item % chunks) * LPD + static_cast<uint32_t>(t % LPD);
    const uint32_t col = q * 4;
    const bool active = col < dim;
    uint64_t e = offsets[d];
    const uint64_t end = offsets[d + 1];
    float* orow = out + d * ld_out + col;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (accumulate && active) {
        if (col + 3 < dim) acc = *reinterpret_cast<const float4*>(orow);
        else {
            acc.x = orow[0];
            if (col + 1 < dim) acc.y = orow[1];
            if (col + 2 < dim) acc.z = orow[2];
        }
    }
    const float* icol = in + col;
    for (; e + U <= end; e += U) {
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = __ldg(edges + e + u);
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            x[u] = active ? ldg4(icol + ed[u].x * ld_in) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) acc4(acc, __uint_as_float(ed[u].y), x[u]);
    }
    for (; e < end; ++e) {
        const Edge ed = __ldg(edges + e);
        const float4 x = active ? ldg4(icol + ed.x * ld_in) : make_float4(0.f, 0.f, 0.f, 0.f);
        acc4(acc, __uint_as_float(ed.y), x);
    }
    if (!active) return;
    acc.x = __fadd_rn(acc.x, 0.f);
    acc.y = __fadd_rn(acc.y, 0.f);
    acc.z = __fadd_rn(acc.z, 0.f);
    acc.w = __fadd_rn(acc.w, 0.f);
    if (col + 3 < dim) {
        __stcs(reinterpret_cast<float4*>(orow), acc);
    } else {
        orow[0] = acc.x;
        if (col + 1 < dim) orow[1] = acc.y;
        if (col + 2 < dim) orow[2] = acc.z;
    }
}

// Scalar fallback for unaligned rows (ld or base not 16-byte aligned).
template <int U>
__global__ void __launch_bounds__(256) k_agg_scalar(const uint64_t* __restrict__ offsets,
                                                   const Edge* __restrict__ edges,
                                                   const uint32_t* __restrict__ order, uint32_t d_begin,
                                                   uint64_t n_items, uint32_t chunks,
                                                   const float* __restrict__ in, uint64_t ld_in,
                                                   float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                   int accumulate) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / 32;
    if (item >= n_items) return;
    const uint32_t d = order[d_begin + item / chunks];
    const uint32_t col = static_cast<uint32_t>(item % chunks) * 32 + lane_id();
    const bool active = col < dim;
    uint64_t e = offsets[d];
    const uint64_t end = offsets[d + 1];
    float acc = (accumulate && active) ? out[d * ld_out + col] : 0.f;
    for (; e + U <= end; e += U) {
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = __ldg(edges + e + u);
        float x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = active ? __ldg(in + ed[u].x * ld_in + col) : 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __fadd_rn(acc, __fmul_rn(__uint_as_float(ed[u].y), x[u]));
    }
    for (; e < end; ++e) {
        const Edge ed = __ldg(edges + e);
        const float x = active ? __ldg(in + ed.x * ld_in + col) : 0.f;
        acc = __fadd_rn(acc, __fmul_rn(__uint_as_float(ed.y), x));
    }
    if (active) out[d * ld_out + col] = __fadd_rn(acc, 0.f);
}

template <int LPD, int U>
void launch_vec4(const uint64_t* offsets, const Edge* edges, const uint32_t* order, uint32_t d_begin,
                 uint32_t nd, uint32_t chunks, const float* in, uint64_t ld_in, float* out, uint64_t ld_out,
                 uint32_t dim, bool accumulate, cudaStream_t s) {
    const uint64_t items = static_cast<uint64_t>(nd) * chunks;
    k_agg_vec4<LPD, U><<<grid_for(items * LPD, 256), 256, 0, s>>>(offsets, edges, order, d_begin, items, chunks,
                                                                 in, ld_in, out, ld_out, dim, accumulate);
    PG_LAUNCH("k_agg_vec4");
}

// dense_matrix.hpp:78-95: out[i][j] = sum_k a[i][k] * b[j][k] in ascending
// k with separately rounded mul/add, then + 0. Block: 128 columns j x 32 rows
// i; b^T chunk and the a-row tile staged in shared memory, k in chunks of 32.
constexpr int kGemmJ = 128, kGemmI = 32, kGemmK = 32;

__global__ void __launch_bounds__(kGemmJ) k_gemm_a_bt(const float* __restrict__ a, uint64_t lda,
                                                     const float* __restrict__ b, uint64_t ldb,
                                                     float* __restrict__ out, uint64_t ldo, uint64_t n,
                                                     uint64_t m, uint64_t K) {
    __shared__ float bt[kGemmK][kGemmJ];
    __shared__ float at[kGemmI][kGemmK + 1];
    const uint64_t j = blockIdx.x * static_cast<uint64_t>(kGemmJ) + threadIdx.x;
    const uint64_t i0 = blockIdx.y * static_cast<uint64_t>(kGemmI);
    float acc[kGemmI];
#pragma unroll
    for (int r = 0; r < kGemmI; ++r) acc[r] = 0.f;
    for (uint64_t k0 = 0; k0 < K; k0 += kGemmK) {
        const int kc = static_cast<int>(K - k0 < kGemmK ? K - k0 : kGemmK);
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) bt[kk][threadIdx.x] = j < m ? b[j * ldb + k0 + kk] : 0.f;
        for (int idx = threadIdx.x; idx < kGemmI * kGemmK; idx += kGemmJ) {
            const int r = idx / kGemmK, kk = idx % kGemmK;
            at[r][kk] = (i0 + r < n && kk < kc) ? a[(i0 + r) * lda + k0 + kk] : 0.f;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            const float bv = bt[kk][threadIdx.x];
#pragma unroll
            for (int r = 0; r < kGemmI; ++r) acc[r] = __fadd_rn(acc[r], __fmul_rn(at[r][kk], bv));
        }
    }
    if (j >= m) return;
#pragma unroll
    for (int r = 0; r < kGemmI; ++r)
        if (i0 + r < n) out[(i0 + r) * ldo + j] = __fadd_rn(acc[r], 0.f);
}

__global__ void k_relu_backward(const float* __restrict__ g, uint64_t ldg, const float* __restrict__ pre,
                                uint64_t ldp, float* __restrict__ out, uint64_t ldo, uint64_t rows,
                                uint64_t cols) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= rows * cols) return;
    const uint64_t r = i / cols, c = i % cols;
    out[r * ldo + c] = pre[r * ldp + c] > 0.f ? g[r * ldg + c] : 0.f;
}

__global__ void k_gather_rows(const float* __restrict__ src, uint64_t lds, const uint32_t* __restrict__ ids,
                              uint64_t k, float* __restrict__ out, uint64_t ldo, uint64_t cols) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= k * cols) return;
    const uint64_t r = i / cols, c = i % cols;
    out[r * ldo + c] = src[static_cast<uint64_t>(ids[r]) * lds + c];
}

}  // namespace

void aggregate_det(const uint64_t* offsets, const Edge* edges, const uint32_t* order, uint32_t D,
                   uint32_t d_begin, uint32_t d_end, const float* in, uint64_t ld_in, float* out,
                   uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s) {
    (void)D;
    if (d_end <= d_begin || dim == 0) return;
    const uint32_t nd = d_end - d_begin;
    const uint32_t dim32 = static_cast<uint32_t>(dim);
    const bool vec = (ld_in % 4 == 0) && (ld_out % 4 == 0) &&
                     (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0) && ld_in >= ((dim + 3) & ~3ull);
    if (!vec) {
        const uint32_t chunks = (dim32 + 31) / 32;
        const uint64_t items = static_cast<uint64_t>(nd) * chunks;
        k_agg_scalar<8><<<grid_for(items * 32, 256), 256, 0, s>>>(offsets, edges, order, d_begin, items, chunks,
                                                                 in, ld_in, out, ld_out, dim32, accumulate);
        PG_LAUNCH("k_agg_scalar");
        return;
    }
    const uint32_t nq = (dim32 + 3) / 4;
    if (nq > 16) {
        launch_vec4<32, 8>(offsets, edges, order, d_begin, nd, (nq + 31) / 32, in, ld_in, out, ld_out, dim32,
                           accumulate, s);
    } else if (nq > 8) {
        launch_vec4<16, 8>(offsets, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s);
    } else if (nq > 4) {
        launch_vec4<8, 8>(offsets, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s);
    } else {
        launch_vec4<4, 8>(offsets, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s);
    }
}

void gemm_a_bt(const float* a, uint64_t lda, const float* b, uint64_t ldb, float* out, uint64_t ldo,
               uint64_t n, uint64_t m, uint64_t k, cudaStream_t s) {
    if (n == 0 || m == 0) return;
    dim3 grid(static_cast<unsigned>((m + kGemmJ - 1) / kGemmJ), static_cast<unsigned>((n + kGemmI - 1) / kGemmI));
    k_gemm_a_bt<<<grid, kGemmJ, 0, s>>>(a, lda, b, ldb, out, ldo, n, m, k);
    PG_LAUNCH("k_gemm_a_bt");
}

void relu_backward(const float* grad, uint64_t ldg, const float* pre, uint64_t ldp, float* out, uint64_t ldo,
                   uint64_t rows, uint64_t cols, cudaStream_t s) {
    if (rows * cols == 0) return;
    k_relu_backward<<<grid_for(rows * cols, 256), 256, 0, s>>>(grad, ldg, pre, ldp, out, ldo, rows, cols);
    PG_LAUNCH("k_relu_backward");
}

void gather_rows(const float* src, uint64_t lds, const uint32_t* ids, uint64_t k, float* out, uint64_t ldo,
                 uint64_t cols, cudaStream_t s) {
    if (k * cols == 0) return;
    k_gather_rows<<<grid_for(k * cols, 256), 256, 0, s>>>(src, lds, ids, k, out, ldo, cols);
    PG_LAUNCH("k_gather_rows");
}

}  // namespace pg
