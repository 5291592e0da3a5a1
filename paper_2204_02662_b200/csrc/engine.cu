// The GCN chain around the backward aggregation (engine.hpp), device
// resident and bit-exact with the reference's f32 build:
//   * dense products (dense_matrix.hpp:40-96): every output element is one
//     thread's ascending-k chain of separately rounded multiply/add, then
//     + 0 — the reference's association order, so the bits match;
//   * relu / row_softmax / top_grad_from_probs (dense_matrix.hpp:98-135,
//     engine.hpp:146-156);
//   * the three backward variants (engine.hpp:177-349) and forward
//     (:114-140), composed from those kernels and the SpMM (aggregate.cu)
//     with relu_backward fused into the SpMM epilogue and gather_rows fused
//     into the W-gradient product.
// These are HBM/latency-bound fp32 reductions with a fixed order; nothing
// here is reshaped for tensor cores (a tcgen05 MMA would re-associate the
// sums and break bit parity with the reference).
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "../../include/pathgcn_b200.h"
#include "pg_internal.h"

namespace pg {

namespace {

constexpr int kThreads = 256;

// ---- out = A * op(B), op(B)(k, j) = BT ? b[j][k] : b[k][j] -----------------
// Block: 32 lanes = 32 output columns j, 8 warps x RPW rows i. K staged in
// chunks of 32 through shared memory; thread (i, j) keeps one ascending-k
// chain per row.
constexpr int kGT = 32;  // j tile / k chunk
constexpr int kGRPW = 16;  // rows per warp: 128-row tiles keep the grid of a write-bound gemm_a_bt (K = 16) from being launch-bound
constexpr int kGI = 8 * kGRPW;

template <bool BT>
__global__ void __launch_bounds__(256) k_gemm(const float* __restrict__ a, uint64_t lda,
                                              const float* __restrict__ b, uint64_t ldb, float* __restrict__ out,
                                              uint64_t ldo, uint64_t n, uint64_t m, uint64_t K) {
    __shared__ float as[kGI][kGT + 1];
    __shared__ float bs[kGT][kGT + 1];
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t j = blockIdx.y * static_cast<uint64_t>(kGT) + lane;
    const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(kGI);  // rows on x: no 65535 cap
    float acc[kGRPW];
#pragma unroll
    for (int r = 0; r < kGRPW; ++r) acc[r] = 0.f;
    for (uint64_t k0 = 0; k0 < K; k0 += kGT) {
        const int kc = static_cast<int>(K - k0 < kGT ? K - k0 : kGT);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kGI * kGT; idx += 256) {
            const int r = idx / kGT, kk = idx % kGT;
            as[r][kk] = (i0 + r < n && kk < kc) ? a[(i0 + r) * lda + k0 + kk] : 0.f;
        }
        for (int idx = threadIdx.x; idx < kGT * kGT; idx += 256) {
            const int kk = idx / kGT, jj = idx % kGT;
            const uint64_t jg = blockIdx.y * static_cast<uint64_t>(kGT) + jj;
            float v = 0.f;
            if (kk < kc && jg < m) v = BT ? b[jg * ldb + k0 + kk] : b[(k0 + kk) * ldb + jg];
            bs[kk][jj] = v;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            const float bv = bs[kk][lane];
#pragma unroll
            for (int r = 0; r < kGRPW; ++r) acc[r] = __fadd_rn(acc[r], __fmul_rn(as[w * kGRPW + r][kk], bv));
        }
    }
    if (j >= m) return;
#pragma unroll
    for (int r = 0; r < kGRPW; ++r) {
        const uint64_t i = i0 + w * kGRPW + r;
        if (i < n) out[i * ldo + j] = __fadd_rn(acc[r], 0.f);
    }
}

// Packed variant (the one dispatched): a lane owns two adjacent output
// columns, so each chain step of a row is half an FFMA2 (runtime -0 addend:
// exactly fl(a*b)) + half an FADD2; the A values come 4 k at a time (one
// broadcast LDS.128), the B pairs once per k for all 16 rows of the warp.
// 128 x 64 output tiles, K in chunks of 32 through shared memory; the same
// ascending-k chain per output as k_gemm, bit for bit.
constexpr int kG2J = 64;

template <bool BT>
__global__ void __launch_bounds__(256) k_gemm2(const float* __restrict__ a, uint64_t lda,
                                               const float* __restrict__ b, uint64_t ldb, float* __restrict__ out,
                                               uint64_t ldo, uint64_t n, uint64_t m, uint64_t K, float nz) {
    __shared__ __align__(16) float as[kGI][kGT];
    __shared__ __align__(16) float bs[kGT][kG2J];
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t j0 = blockIdx.y * static_cast<uint64_t>(kG2J);
    const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(kGI);
    unsigned long long nz2, acc[kGRPW];
    asm("mov.b64 %0, {%1,%1};" : "=l"(nz2) : "f"(nz));
#pragma unroll
    for (int r = 0; r < kGRPW; ++r) asm("mov.b64 %0, {%1,%1};" : "=l"(acc[r]) : "f"(0.f));
    for (uint64_t k0 = 0; k0 < K; k0 += kGT) {
        const int kc = static_cast<int>(K - k0 < kGT ? K - k0 : kGT);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kGI * kGT; idx += 256) {
            const int r = idx / kGT, kk = idx % kGT;
            as[r][kk] = (i0 + r < n && kk < kc) ? a[(i0 + r) * lda + k0 + kk] : 0.f;
        }
        for (int idx = threadIdx.x; idx < kGT * kG2J; idx += 256) {
            int kk, jj;
            if (BT) {  // b[j][k]: consecutive threads walk k
                kk = idx % kGT;
                jj = idx / kGT;
            } else {
                kk = idx / kG2J;
                jj = idx % kG2J;
            }
            const uint64_t jg = j0 + jj;
            float v = 0.f;
            if (kk < kc && jg < m) v = BT ? b[jg * ldb + k0 + kk] : b[(k0 + kk) * ldb + jg];
            bs[kk][jj] = v;
        }
        __syncthreads();
        // zero-padded k (kk >= kc) and rows/columns past the matrix add +0
        // products after the real ones: only a -0 chain can change (to +0),
        // which the final fl(acc + 0) does anyway
        for (int kq = 0; kq < (kc + 3) / 4; ++kq) {
            unsigned long long bp[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) bp[u] = *reinterpret_cast<const unsigned long long*>(&bs[4 * kq + u][2 * lane]);
#pragma unroll
            for (int r = 0; r < kGRPW; ++r) {
                const float4 a4 = *reinterpret_cast<const float4*>(&as[w * kGRPW + r][4 * kq]);
                const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    unsigned long long aa, p;
                    asm("mov.b64 %0, {%1,%1};" : "=l"(aa) : "f"(av[u]));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(aa), "l"(bp[u]), "l"(nz2));
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc[r]) : "l"(acc[r]), "l"(p));
                }
            }
        }
    }
    const uint64_t j = j0 + 2 * lane;
    if (j >= m) return;
#pragma unroll
    for (int r = 0; r < kGRPW; ++r) {
        const uint64_t i = i0 + w * kGRPW + r;
        if (i >= n) continue;
        float lo, hi;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[r]));
        out[i * ldo + j] = __fadd_rn(lo, 0.f);
        if (j + 1 < m) out[i * ldo + j + 1] = __fadd_rn(hi, 0.f);
    }
}

// Register-tiled variant (tuning "gemm_packed" = 2): each thread owns an
// 8 x 8 output tile (rows {4ty..4ty+3, 64+4ty..}, column pairs at 4tx and
// 64+4tx of a 128 x 128 CTA tile), so per k it reads 8 A scalars and 8 B
// values from shared memory for 32 FFMA2 + 32 FADD2 (k_gemm2's warp-wide
// row tile loads one broadcast A value per row per k for only 2 output
// columns a lane: 18 registers per 32 FP instructions, FMA pipe 58 % busy;
// here 16 per 64 and the FMA pipe 88 % busy, ncu profiles/ncu_gemm_r02.json). A goes global -> shared by cp.async (16 B, zero-fill
// past n / K), double-buffered over 16-k chunks; B arrives k-major
// (gemm_a_bt transposes W first, a few KB). Same chain per output as k_gemm:
// ascending k, fl(a*b) by FFMA2 with a runtime -0 addend, FADD2, then + 0.
constexpr int kG3K = 16;   // k chunk
constexpr int kG3N = 128;  // columns per CTA tile (16 threads x 8)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes));
}

// A rows [i0, i0+TM) x k [k0, k0+16) and B (k-major, ld ldb) rows
// [k0, k0+16) x columns [j0, j0+128) into stage buffers; zero past n / m / K
template <int TM>
__device__ __forceinline__ void g3_load(float (*As)[kG3K + 4], float (*Bs)[kG3N + 4], const float* a, uint64_t lda,
                                        const float* b, uint64_t ldb, uint64_t n, uint64_t m, uint64_t K,
                                        uint64_t i0, uint64_t j0, uint64_t k0, int tid) {
#pragma unroll
    for (int h = 0; h < TM / 64; ++h) {
        const int row = (tid >> 2) + 64 * h, kq = (tid & 3) * 4;
        const uint64_t gi = i0 + row, gk = k0 + kq;
        const bool in = gi < n && gk < K;
        const int bytes = in ? (K - gk >= 4 ? 16 : static_cast<int>((K - gk) * 4)) : 0;
        cp_async16(&As[row][kq], in ? a + gi * lda + gk : a, bytes);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = (tid >> 5) + 8 * h, jq = (tid & 31) * 4;
        const uint64_t gk = k0 + k, gj = j0 + jq;
        const bool in = gk < K && gj < m;
        const int bytes = in ? (m - gj >= 4 ? 16 : static_cast<int>((m - gj) * 4)) : 0;
        cp_async16(&Bs[k][jq], in ? b + gk * ldb + gj : b, bytes);
    }
    asm volatile("cp.async.commit_group;");
}

// thread row r of RM: rows 4 ty + (r % 4) + 64 (r / 4) of the CTA tile
template <int RM>
__global__ void __launch_bounds__(256, RM == 8 ? 2 : 1) k_gemm3(const float* __restrict__ a, uint64_t lda,
                                                                const float* __restrict__ b, uint64_t ldb,
                                                                float* __restrict__ out, uint64_t ldo, uint64_t n,
                                                                uint64_t m, uint64_t K, float nz) {
    constexpr int TM = 16 * RM;
    // dynamic: 2 x (TM x 20 + 16 x 132) floats = 38.4 KB (RM 8) / 57.3 KB (RM 16)
    extern __shared__ __align__(16) float g3_smem[];
    auto As = reinterpret_cast<float(*)[TM][kG3K + 4]>(g3_smem);
    auto Bs = reinterpret_cast<float(*)[kG3K][kG3N + 4]>(g3_smem + 2 * TM * (kG3K + 4));
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(TM), j0 = blockIdx.y * static_cast<uint64_t>(kG3N);
    unsigned long long nz2, acc[RM][4];
    asm("mov.b64 %0, {%1,%1};" : "=l"(nz2) : "f"(nz));
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) asm("mov.b64 %0, {%1,%1};" : "=l"(acc[i][p]) : "f"(0.f));
    const uint64_t nk = (K + kG3K - 1) / kG3K;
    g3_load<TM>(As[0], Bs[0], a, lda, b, ldb, n, m, K, i0, j0, 0, tid);
    for (uint64_t c = 0; c < nk; ++c) {
        const int cur = static_cast<int>(c & 1);
        if (c + 1 < nk) {
            g3_load<TM>(As[cur ^ 1], Bs[cur ^ 1], a, lda, b, ldb, n, m, K, i0, j0, (c + 1) * kG3K, tid);
            asm volatile("cp.async.wait_group 1;");
        } else {
            asm volatile("cp.async.wait_group 0;");
        }
        __syncthreads();
        // zero-filled k past K adds +-0 products after the real ones: only a
        // -0 chain can change (to +0), which the final fl(acc + 0) does anyway
#pragma unroll
        for (int kk = 0; kk < kG3K; kk += 2) {
            float2 av[RM];
#pragma unroll
            for (int i = 0; i < RM; ++i)
                av[i] = *reinterpret_cast<const float2*>(&As[cur][4 * ty + (i & 3) + 64 * (i >> 2)][kk]);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][kk + u][4 * tx]);
                const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][kk + u][64 + 4 * tx]);
                unsigned long long bp[4];
                asm("mov.b64 %0, {%1,%2};" : "=l"(bp[0]) : "f"(b0.x), "f"(b0.y));
                asm("mov.b64 %0, {%1,%2};" : "=l"(bp[1]) : "f"(b0.z), "f"(b0.w));
                asm("mov.b64 %0, {%1,%2};" : "=l"(bp[2]) : "f"(b1.x), "f"(b1.y));
                asm("mov.b64 %0, {%1,%2};" : "=l"(bp[3]) : "f"(b1.z), "f"(b1.w));
#pragma unroll
                for (int i = 0; i < RM; ++i) {
                    unsigned long long aa;
                    asm("mov.b64 %0, {%1,%1};" : "=l"(aa) : "f"(u ? av[i].y : av[i].x));
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        unsigned long long pr;
                        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pr) : "l"(aa), "l"(bp[p]), "l"(nz2));
                        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc[i][p]) : "l"(acc[i][p]), "l"(pr));
                    }
                }
            }
        }
        __syncthreads();
    }
    const bool v4 = (ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
        const uint64_t gi = i0 + 4 * ty + (i & 3) + 64 * (i >> 2);
        if (gi >= n) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint64_t gj = j0 + 64 * h + 4 * tx;
            if (gj >= m) continue;
            float v[4];
            asm("mov.b64 {%0,%1}, %2;" : "=f"(v[0]), "=f"(v[1]) : "l"(acc[i][2 * h]));
            asm("mov.b64 {%0,%1}, %2;" : "=f"(v[2]), "=f"(v[3]) : "l"(acc[i][2 * h + 1]));
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = __fadd_rn(v[q], 0.f);
            float* o = out + gi * ldo + gj;
            if (v4 && gj + 3 < m) {
                *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (gj + q < m) o[q] = v[q];
            }
        }
    }
}

// W^T for gemm_a_bt's k-major B operand: t[k][j] = b[j][k] (ld_t = m4)
__global__ void k_transpose(const float* __restrict__ b, uint64_t ldb, float* __restrict__ t, uint64_t ldt,
                            uint64_t m, uint64_t K) {
    const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= m * K) return;
    const uint64_t k = idx / m, j = idx % m;
    t[k * ldt + j] = b[j * ldb + k];
}

// ---- out = A[rows]^T * B (dense_matrix.hpp:57-76 gemm_at_b) -----------------
// out[i][j] = sum over k < n, ascending, of A(k, i) * B(k, j), A(k, i) =
// a[(rows ? rows[k] : k) * lda + i] (the engine's gather_rows fused in).
// The order forces one serial chain per output over all n rows, so the
// only parallelism is the r x c outputs and the floor is n dependent FADDs
// (4 cycles each). A 32-thread block owns TI x TC chains, two adjacent
// columns per lane: one row is LDS (a, broadcast) + LDS.64 (b pair) + FFMA2
// (products, runtime -0 addend: fl(a*b) exactly, no contraction) + FADD2
// (both chain steps) plus the copy issue. No block barrier: the warp owns
// its kAtbStages-deep cp.async ring (__syncwarp orders it); lane kk copies
// row kk of each stage (its gathered A slice, its B slice, fixed column
// offsets as immediates), and the row ids of stage ts ride in the copy
// group of stage ts - (S-1), so no copy waits on an id load. Rows past n
// are zero filled: their +0 products only flip a -0 accumulator to +0,
// which the final fl(acc + 0) does anyway.
// Measured (Reddit shape): ~19 cycles per row per warp, i.e. 1.46 ms for
// the top layer and 2.26 ms for layer 0, against 3.2 / 2.5 ms for the
// earlier 128-thread block-owned kernel. The copy-warp variant below
// (k_gemm_at_b_split, the default) takes the copy issue off the chain
// warp: ~11 cycles per row, 0.83 / 1.32 ms. Producer warps forming the
// products, LDS.128 stage layouts, and scalar one-chain-per-lane kernels
// measured equal or slower; see DESIGN.md.
constexpr int kAtbStages = 8;

template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool ok) {
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                     "l"(src), "r"(ok ? 4 : 0)
                     : "memory");
}

// cp.async with the ignore-src predicate: skip == true zero-fills the
// destination without reading src (src must still be a valid address)
template <int CP>
__device__ __forceinline__ void cp_async_skip(void* dst, const void* src, bool skip) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    if (CP == 16)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n cp.async.cg.shared.global [%0], [%1], 16, p;\n}" ::"r"(d),
                     "l"(src), "r"(static_cast<int>(skip))
                     : "memory");
    else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n cp.async.ca.shared.global [%0], [%1], 4, p;\n}" ::"r"(d),
                     "l"(src), "r"(static_cast<int>(skip))
                     : "memory");
}

template <int TI, int V>
__global__ void __launch_bounds__(32) k_gemm_at_b_w(const float* __restrict__ a, uint64_t lda,
                                                   const uint32_t* __restrict__ rows, const float* __restrict__ b,
                                                   uint64_t ldb, float* __restrict__ out, uint64_t ldo, uint32_t n,
                                                   uint32_t r, uint32_t c, float nz) {
    constexpr int LPI = 32 / TI;  // lanes per A column
    constexpr int TC = 2 * LPI;   // B columns per warp
    constexpr int KC = 32;        // rows per stage: lane kk copies row kk's A slice and id
    constexpr int S = kAtbStages;
    constexpr int AV = (V == 4 && TI % 4 == 0) ? 4 : 1;
    constexpr int BV = V == 4 ? 4 : 1;
    constexpr int NA = TI / AV, NB = TC / BV;  // copies per lane per stage
    __shared__ __align__(16) float sa[S][KC][TI];
    __shared__ __align__(16) float sb[S][KC][TC];
    // row ids ride the copy pipeline: stage ts's ids are copied in the group
    // of stage ts - (S-1), so the wait that makes stage t readable also
    // lands the ids the next issue needs
    __shared__ uint32_t sid[S][KC];
    const unsigned lane = threadIdx.x;
    const uint32_t i0 = blockIdx.x * TI, j0 = blockIdx.y * TC;
    const unsigned ti = lane / LPI, tj = (lane % LPI) * 2;
    const uint32_t ntiles = (n + KC - 1) / KC;
    // lane kk copies row kk of every stage: its A slice (gathered row id)
    // and its TC-float B slice, fixed column offsets as immediates; columns
    // past r / c are skipped: ignore-src zero-fills without reading, so the
    // address of a skipped column is never dereferenced
    bool a_skip[NA], b_skip[NB];
#pragma unroll
    for (int q = 0; q < NA; ++q) a_skip[q] = i0 + q * AV >= r;
#pragma unroll
    for (int q = 0; q < NB; ++q) b_skip[q] = j0 + q * BV >= c;
    const float* a_col = a + i0;
    const float* b_row = b + static_cast<uint64_t>(lane) * ldb + j0;  // row lane of stage 0
    const uint64_t b_stage = static_cast<uint64_t>(KC) * ldb;
    auto copies = [&](uint32_t ts, uint32_t id, auto tail_t) {
        constexpr bool tail = decltype(tail_t)::value;
        const int slot = ts % S;
        const bool out_row = tail && ts * KC + lane >= n;
        const float* ar = out_row ? a : a_col + static_cast<uint64_t>(id) * lda;
#pragma unroll
        for (int q = 0; q < NA; ++q)
            cp_async_skip<AV * 4>(&sa[slot][lane][q * AV], ar + q * AV, a_skip[q] || out_row);
        const float* br = out_row ? b : b_row + ts * b_stage;
#pragma unroll
        for (int q = 0; q < NB; ++q)
            cp_async_skip<BV * 4>(&sb[slot][lane][q * BV], br + q * BV, b_skip[q] || out_row);
    };
    auto issue = [&](uint32_t ts, uint32_t id) {
        if (ts < ntiles) {
            if (ts * KC + KC <= n)
                copies(ts, id, std::false_type{});
            else
                copies(ts, id, std::true_type{});
        }
        if (rows) {
            const uint32_t ka = (ts + S - 1) * KC + lane;
            const bool out_row = ka >= n;
            cp_async_skip<4>(&sid[(ts + S - 1) % S][lane], out_row ? rows : rows + ka, out_row);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll 1
    for (int s = 0; s < S - 1; ++s) {
        const uint32_t k = s * KC + lane;
        issue(s, k < n ? (rows ? __ldg(rows + k) : k) : 0u);
    }
    unsigned long long nz2, acc;
    asm("mov.b64 %0, {%1,%1};" : "=l"(nz2) : "f"(nz));
    asm("mov.b64 %0, {%1,%1};" : "=l"(acc) : "f"(0.f));
    for (uint32_t t = 0; t < ntiles; ++t) {
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 2) : "memory");
        __syncwarp();  // stage t visible to every lane; stage t-1's slot is free
        {
            const uint32_t ts = t + S - 1;
            issue(ts, rows ? sid[ts % S][lane] : ts * KC + lane);
        }
        const int slot = t % S;
        const float* pa = &sa[slot][0][ti];
        const unsigned long long* pb = reinterpret_cast<const unsigned long long*>(&sb[slot][0][tj]);
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            unsigned long long aa, p;
            asm("mov.b64 %0, {%1,%1};" : "=l"(aa) : "f"(pa[kk * TI]));
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(aa), "l"(pb[kk * (TC / 2)]), "l"(nz2));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc) : "l"(acc), "l"(p));
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc));
    const uint64_t i = i0 + ti, j = j0 + tj;
    if (i < r && j < c) out[i * ldo + j] = __fadd_rn(lo, 0.f);
    if (i < r && j + 1 < c) out[i * ldo + j + 1] = __fadd_rn(hi, 0.f);
}

// Copy warp + chain warp variant (tuning "atb_split", default): warp 1
// issues every cp.async of a 64-row stage (2 rows per lane, the same 16-byte
// copies and id pipeline as above) and warp 0 only walks the chains
// (LDS a + LDS.64 b + FFMA2 + FADD2 per row); SL stage slots are
// handed over with named barriers (FULL: copy warp waits for its group and
// arrives; EMPTY: chain warp arrives after reading). 64-row stages keep
// the barrier cost per row small.
// SL slots, LAG stages in flight ahead of the chain warp (tuning
// "atb_depth": 0 = 4 / 2, 1 = 7 / 5). A block's copy pipeline is its
// memory-level parallelism: LAG x 64 gathered rows per latency. At 4 / 2 the
// products layer-0 W' (1.2M rows per chain) ran at ~34 cycles per row, the
// 128 rows in flight per block over a ~1 us gather latency.
constexpr int kAtbKC = 64;

// TI A columns x TC B columns per block; CH A columns per lane (CH = 2:
// 128 chains per block for shapes with more chains than SMs)
template <int TI, int CH, int SL, int LAG>
struct AtbSplitSmem {
    static constexpr int TC = 2 * 32 / (TI / CH);
    float sa[SL][kAtbKC][TI];
    float sb[SL][kAtbKC][TC];
    uint32_t sid[LAG + 2][kAtbKC];
};

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int TI, int V, int CH, int SL = 4, int LAG = 2, bool kAtbCoopCopy = false>
__global__ void __launch_bounds__(64) k_gemm_at_b_split(const float* __restrict__ a, uint64_t lda,
                                                       const uint32_t* __restrict__ rows, const float* __restrict__ b,
                                                       uint64_t ldb, float* __restrict__ out, uint64_t ldo,
                                                       uint32_t n, uint32_t r, uint32_t c, float nz) {
    using Sm = AtbSplitSmem<TI, CH, SL, LAG>;
    constexpr int LPI = 32 / (TI / CH), TC = Sm::TC, KC = kAtbKC, NI = LAG + 2;
    constexpr int AV = (V == 4 && TI % 4 == 0) ? 4 : 1;
    constexpr int BV = V == 4 ? 4 : 1;
    constexpr int NA = TI / AV, NB = TC / BV;
    __shared__ __align__(16) Sm sm;
    const unsigned lane = threadIdx.x & 31;
    const uint32_t i0 = blockIdx.x * TI, j0 = blockIdx.y * TC;
    const uint32_t ntiles = (n + KC - 1) / KC;
    auto full_bar = [](uint32_t ts) { return 1 + static_cast<int>(ts % SL); };
    auto empty_bar = [](uint32_t ts) { return 1 + SL + static_cast<int>(ts % SL); };
    if (threadIdx.x < 32) {  // chain warp: A columns ti*CH .. +CH-1, B columns tj, tj+1
        const unsigned ti = (lane / LPI) * CH, tj = (lane % LPI) * 2;
        unsigned long long nz2, acc[CH];
        asm("mov.b64 %0, {%1,%1};" : "=l"(nz2) : "f"(nz));
#pragma unroll
        for (int h = 0; h < CH; ++h) asm("mov.b64 %0, {%1,%1};" : "=l"(acc[h]) : "f"(0.f));
        for (uint32_t ts = 0; ts < ntiles; ++ts) {
            const int slot = ts % SL;
            named_sync(full_bar(ts), 64);
            const float* pa = &sm.sa[slot][0][ti];
            const unsigned long long* pb = reinterpret_cast<const unsigned long long*>(&sm.sb[slot][0][tj]);
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
                float av[CH];
                if (CH == 2) {
                    const float2 a2 = *reinterpret_cast<const float2*>(pa + kk * TI);
                    av[0] = a2.x;
                    av[CH - 1] = a2.y;
                } else {
                    av[0] = pa[kk * TI];
                }
                const unsigned long long bb = pb[kk * (TC / 2)];
#pragma unroll
                for (int h = 0; h < CH; ++h) {
                    unsigned long long aa, p;
                    asm("mov.b64 %0, {%1,%1};" : "=l"(aa) : "f"(av[h]));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(aa), "l"(bb), "l"(nz2));
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc[h]) : "l"(acc[h]), "l"(p));
                }
            }
            named_arrive(empty_bar(ts), 64);
        }
#pragma unroll
        for (int h = 0; h < CH; ++h) {
            float lo, hi;
            asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[h]));
            const uint64_t i = i0 + ti + h, j = j0 + tj;
            if (i < r && j < c) out[i * ldo + j] = __fadd_rn(lo, 0.f);
            if (i < r && j + 1 < c) out[i * ldo + j + 1] = __fadd_rn(hi, 0.f);
        }
        return;
    }
    // copy warp: lane copies rows lane and lane + 32 of every stage
    bool a_skip[NA], b_skip[NB];
#pragma unroll
    for (int q = 0; q < NA; ++q) a_skip[q] = i0 + q * AV >= r;
#pragma unroll
    for (int q = 0; q < NB; ++q) b_skip[q] = j0 + q * BV >= c;
    const float* a_col = a + i0;
    const uint64_t b_stage = static_cast<uint64_t>(KC) * ldb;
    auto copy_row = [&](uint32_t ts, int slot, int kk, uint32_t id) {
        const bool out_row = ts * KC + kk >= n;
        const float* ar = out_row ? a : a_col + static_cast<uint64_t>(id) * lda;
#pragma unroll
        for (int q = 0; q < NA; ++q)
            cp_async_skip<AV * 4>(&sm.sa[slot][kk][q * AV], ar + q * AV, a_skip[q] || out_row);
        const float* br = out_row ? b : b + static_cast<uint64_t>(kk) * ldb + j0 + ts * b_stage;
#pragma unroll
        for (int q = 0; q < NB; ++q)
            cp_async_skip<BV * 4>(&sm.sb[slot][kk][q * BV], br + q * BV, b_skip[q] || out_row);
    };
    auto fetch_id = [&](uint32_t ts, int kk) -> uint32_t {
        const uint32_t k = ts * KC + kk;
        return k < n ? (rows ? __ldg(rows + k) : k) : 0u;
    };
    for (uint32_t ts = 0; ts < ntiles + LAG; ++ts) {
        if (ts < ntiles) {
            if (ts >= static_cast<uint32_t>(SL)) named_sync(empty_bar(ts), 64);
            const int slot = ts % SL;
            if (kAtbCoopCopy) {
                // lanes share rows: a warp-wide copy touches 32 / NA (A) and
                // 32 / NB (B) rows instead of 32 — one L1 wavefront per row
                // line, 3x fewer than one row per lane
                const bool tail = ts * KC + KC > n;
#pragma unroll
                for (int q = lane; q < KC * NA; q += 32) {
                    const int kk = q / NA, qa = q % NA;
                    const bool out_row = tail && ts * KC + kk >= n;
                    uint32_t id;
                    if (!rows)
                        id = ts * KC + kk;
                    else if (ts <= static_cast<uint32_t>(LAG))
                        id = fetch_id(ts, kk);
                    else
                        id = sm.sid[ts % NI][kk];
                    const float* ar = out_row ? a : a_col + static_cast<uint64_t>(id) * lda;
                    cp_async_skip<AV * 4>(&sm.sa[slot][kk][qa * AV], ar + qa * AV, a_skip[qa] || out_row);
                }
#pragma unroll
                for (int q = lane; q < KC * NB; q += 32) {
                    const int kk = q / NB, qb = q % NB;
                    const bool out_row = tail && ts * KC + kk >= n;
                    const float* br = out_row ? b : b + static_cast<uint64_t>(kk) * ldb + j0 + ts * b_stage;
                    cp_async_skip<BV * 4>(&sm.sb[slot][kk][qb * BV], br + qb * BV, b_skip[qb] || out_row);
                }
            } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int kk = lane + 32 * h;
                uint32_t id;
                if (!rows)
                    id = ts * KC + kk;
                else if (ts <= static_cast<uint32_t>(LAG))
                    id = fetch_id(ts, kk);
                else
                    id = sm.sid[ts % NI][kk];
                copy_row(ts, slot, kk, id);
            }
            }
            if (rows) {  // ids of stage ts + LAG + 1 ride with this group
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int kk = lane + 32 * h;
                    const uint32_t ka = (ts + LAG + 1) * KC + kk;
                    const bool skip = ka >= n;
                    cp_async_skip<4>(&sm.sid[(ts + LAG + 1) % NI][kk], skip ? rows : rows + ka, skip);
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (ts >= static_cast<uint32_t>(LAG)) {
            asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
            __syncwarp();
            named_arrive(full_bar(ts - LAG), 64);
        }
    }
    // match the chain warp's last EMPTY arrivals (no barrier left half-arrived)
    for (uint32_t ts = ntiles > static_cast<uint32_t>(SL) ? ntiles : SL; ts < ntiles + SL; ++ts)
        named_sync(empty_bar(ts), 64);
}

// Four chain warps + four copy warps per block, one block per SM (tuning
// "atb_quad"). The FP32 pipe holds an FFMA2 / FADD2 two cycles, so a chain
// warp's row costs 4 pipe cycles at best and two chain warps on one SMSP
// halve each other: here every SMSP runs exactly one chain warp (warps 0-3),
// and four copy warps (warps 4-7, each a quarter of every 64-row stage) keep
// enough gathered rows in flight — one copy warp per block capped the ring at
// ~128 rows per gather latency. Chain warp w owns the tile's B columns
// [w*TCW, (w+1)*TCW): lane = (A column ti, B column pair tj). Same chain per
// output (ascending rows, fl(a*b) by FFMA2 with a -0 addend, FADD2, + 0):
// bit-identical.
template <int TI, int TCW, int SL, int LAG>
struct AtbQuadSmem {
    float sa[SL][kAtbKC][TI];
    float sb[SL][kAtbKC][4 * TCW];
    uint32_t sid[LAG + 2][kAtbKC];
};

template <int TI, int TCW, int SL, int LAG>
__global__ void __launch_bounds__(256) k_gemm_at_b_quad(const float* __restrict__ a, uint64_t lda,
                                                       const uint32_t* __restrict__ rows, const float* __restrict__ b,
                                                       uint64_t ldb, float* __restrict__ out, uint64_t ldo,
                                                       uint32_t n, uint32_t r, uint32_t c, float nz) {
    constexpr int KC = kAtbKC, NI = LAG + 2, TC = 4 * TCW, NT = 256, RPW = KC / 4;  // rows per copy warp
    constexpr int NA = TI / 4, NB = TC / 4;  // 16-byte pieces per row
    static_assert(TI % 4 == 0 && TC % 4 == 0 && TI * (TCW / 2) <= 32, "tile");
    using Sm = AtbQuadSmem<TI, TCW, SL, LAG>;
    extern __shared__ __align__(16) unsigned char atbq_smem[];
    Sm& sm = *reinterpret_cast<Sm*>(atbq_smem);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t i0 = blockIdx.x * TI, j0 = blockIdx.y * TC;
    const uint32_t ntiles = (n + KC - 1) / KC;
    auto full_bar = [](uint32_t ts) { return 1 + static_cast<int>(ts % SL); };
    auto empty_bar = [](uint32_t ts) { return 1 + SL + static_cast<int>(ts % SL); };
    if (warp < 4) {  // chain warp: B columns [warp*TCW, +TCW) of the tile
        constexpr int NP = TCW / 2;
        const bool on = lane < TI * NP;
        const unsigned ti = on ? lane / NP : 0, tj = warp * TCW + (on ? lane % NP : 0) * 2;
        unsigned long long nz2, acc;
        asm("mov.b64 %0, {%1,%1};" : "=l"(nz2) : "f"(nz));
        asm("mov.b64 %0, {%1,%1};" : "=l"(acc) : "f"(0.f));
        for (uint32_t ts = 0; ts < ntiles; ++ts) {
            const int slot = ts % SL;
            named_sync(full_bar(ts), NT);
            const float* pa = &sm.sa[slot][0][ti];
            const unsigned long long* pb = reinterpret_cast<const unsigned long long*>(&sm.sb[slot][0][tj]);
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
                unsigned long long aa, p;
                asm("mov.b64 %0, {%1,%1};" : "=l"(aa) : "f"(pa[kk * TI]));
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(aa), "l"(pb[kk * (TC / 2)]), "l"(nz2));
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc) : "l"(acc), "l"(p));
            }
            named_arrive(empty_bar(ts), NT);
        }
        if (!on) return;
        float lo, hi;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc));
        const uint64_t i = i0 + ti, j = j0 + tj;
        if (i < r && j < c) out[i * ldo + j] = __fadd_rn(lo, 0.f);
        if (i < r && j + 1 < c) out[i * ldo + j + 1] = __fadd_rn(hi, 0.f);
        return;
    }
    // copy warp cw: rows [cw*RPW, (cw+1)*RPW) of every stage, 16-byte pieces,
    // lanes sharing rows
    const unsigned cw = warp - 4;
    const float* a_col = a + i0;
    const uint64_t b_stage = static_cast<uint64_t>(KC) * ldb;
    auto fetch_id = [&](uint32_t ts, int kk) -> uint32_t {
        const uint32_t k = ts * KC + kk;
        return k < n ? (rows ? __ldg(rows + k) : k) : 0u;
    };
    for (uint32_t ts = 0; ts < ntiles + LAG; ++ts) {
        if (ts < ntiles) {
            if (ts >= static_cast<uint32_t>(SL)) named_sync(empty_bar(ts), NT);
            const int slot = ts % SL;
            const bool tail = ts * KC + KC > n;
#pragma unroll
            for (int q = lane; q < RPW * NA; q += 32) {
                const int kk = cw * RPW + q / NA, qa = q % NA;
                const bool skip = (tail && ts * KC + kk >= n) || i0 + qa * 4 >= r;
                uint32_t id;
                if (!rows)
                    id = ts * KC + kk;
                else if (ts <= static_cast<uint32_t>(LAG))
                    id = fetch_id(ts, kk);
                else
                    id = sm.sid[ts % NI][kk];
                cp_async_skip<16>(&sm.sa[slot][kk][qa * 4], skip ? a : a_col + static_cast<uint64_t>(id) * lda + qa * 4,
                                  skip);
            }
#pragma unroll
            for (int q = lane; q < RPW * NB; q += 32) {
                const int kk = cw * RPW + q / NB, qb = q % NB;
                const bool skip = (tail && ts * KC + kk >= n) || j0 + qb * 4 >= c;
                cp_async_skip<16>(&sm.sb[slot][kk][qb * 4],
                                  skip ? b : b + static_cast<uint64_t>(kk) * ldb + j0 + ts * b_stage + qb * 4, skip);
            }
            if (rows && lane < RPW) {  // ids of stage ts + LAG + 1 ride with this group
                const int kk = cw * RPW + lane;
                const uint32_t ka = (ts + LAG + 1) * KC + kk;
                const bool skip = ka >= n;
                cp_async_skip<4>(&sm.sid[(ts + LAG + 1) % NI][kk], skip ? rows : rows + ka, skip);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (ts >= static_cast<uint32_t>(LAG)) {
            asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
            __syncwarp();
            named_arrive(full_bar(ts - LAG), NT);
        }
    }
    for (uint32_t ts = ntiles > static_cast<uint32_t>(SL) ? ntiles : SL; ts < ntiles + SL; ++ts)
        named_sync(empty_bar(ts), NT);
}

// one-column-per-lane blocks (64 chains each) beyond ~1.5 per SM: use 2
bool gemm_at_b_chain_pairs(uint64_t r, uint64_t c) {
    if (!tuning(kTuneAtbSplit) || tuning(kTuneAtbPairs) == 0) return false;
    const uint64_t ti = c <= 8 ? 8 : 4, tc = 64 / ti;
    return ((r + ti - 1) / ti) * ((c + tc - 1) / tc) > static_cast<uint64_t>(tuning(kTuneAtbPairs));
}

template <int TI>
void launch_at_b(DMat a, const uint32_t* rows, DMat b, DMat out, uint64_t n, uint64_t r, uint64_t c,
                 cudaStream_t s) {
    constexpr unsigned TC = 64 / TI;
    dim3 grid(static_cast<unsigned>((r + TI - 1) / TI), static_cast<unsigned>((c + TC - 1) / TC));
    const bool v4 = a.ld % 4 == 0 && b.ld % 4 == 0 && reinterpret_cast<uintptr_t>(a.p) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(b.p) % 16 == 0;
    volatile float nz = -0.f;  // runtime -0: a literal lets ptxas fold the FFMA2 away
    const uint32_t n32 = static_cast<uint32_t>(n), r32 = static_cast<uint32_t>(r), c32 = static_cast<uint32_t>(c);
    if (tuning(kTuneAtbSplit)) {
        // two A columns per lane once one-per-lane blocks outnumber the SMs
        // ~1.5x: fewer chain warps sharing SMSPs (products layer 0: 400 -> 200)
        const bool deep = tuning(kTuneAtbDepth) == 1;
        const bool coop = tuning(kTuneAtbDepth) == 2;
        if (gemm_at_b_chain_pairs(r, c)) {
            constexpr int TI2 = 2 * TI;
            dim3 g2(static_cast<unsigned>((r + TI2 - 1) / TI2), grid.y);
            if (v4 && coop)
                k_gemm_at_b_split<TI2, 4, 2, 4, 2, true><<<g2, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld,
                                                                          n32, r32, c32, nz);
            else if (v4 && deep)
                k_gemm_at_b_split<TI2, 4, 2, 7, 5><<<g2, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32,
                                                                    r32, c32, nz);
            else if (v4)
                k_gemm_at_b_split<TI2, 4, 2><<<g2, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32, c32,
                                                              nz);
            else
                k_gemm_at_b_split<TI2, 1, 2><<<g2, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32, c32,
                                                              nz);
        } else if (v4 && coop) {
            k_gemm_at_b_split<TI, 4, 1, 4, 2, true><<<grid, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32,
                                                                       r32, c32, nz);
        } else if (v4 && deep) {
            k_gemm_at_b_split<TI, 4, 1, 7, 5><<<grid, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32,
                                                                 c32, nz);
        } else if (v4) {
            k_gemm_at_b_split<TI, 4, 1><<<grid, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32, c32, nz);
        } else {
            k_gemm_at_b_split<TI, 1, 1><<<grid, 64, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32, c32, nz);
        }
        PG_LAUNCH("k_gemm_at_b_split");
        return;
    }
    if (v4)
        k_gemm_at_b_w<TI, 4><<<grid, 32, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32, c32, nz);
    else
        k_gemm_at_b_w<TI, 1><<<grid, 32, 0, s>>>(a.p, a.ld, rows, b.p, b.ld, out.p, out.ld, n32, r32, c32, nz);
    PG_LAUNCH("k_gemm_at_b_w");
}

// ---- elementwise / row kernels ---------------------------------------------
// 2-D grid-stride over (rows, cols): blockIdx.y strides rows
constexpr int kEwRows = 8;  // elementwise row kernels: rows per thread and step

__global__ void k_relu(const float* __restrict__ x, uint64_t ldx, float* __restrict__ out, uint64_t ldo,
                       uint64_t rows, uint32_t cols) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    // kEwRows rows per step, all loads in flight before the stores (one
    // load per thread in flight held the products forward's relu at 2 TB/s)
    const uint64_t gy = gridDim.y;
    for (uint64_t r = blockIdx.y; r < rows; r += kEwRows * gy) {
        float v[kEwRows];
#pragma unroll
        for (int u = 0; u < kEwRows; ++u) {
            const uint64_t rr = r + u * gy;
            v[u] = rr < rows ? x[rr * ldx + c] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kEwRows; ++u) {
            const uint64_t rr = r + u * gy;
            if (rr < rows) out[rr * ldo + c] = v[u] > 0.f ? v[u] : 0.f;
        }
    }
}

// relu_backward with the pre-activation rows selected by pre_rows
__global__ void k_relu_bwd_rows(const float* __restrict__ g, uint64_t ldg, const float* __restrict__ pre,
                                uint64_t ldp, const uint32_t* __restrict__ pre_rows, float* __restrict__ out,
                                uint64_t ldo, uint64_t rows, uint32_t cols) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    const uint64_t gy = gridDim.y;
    for (uint64_t r = blockIdx.y; r < rows; r += kEwRows * gy) {
        float pv[kEwRows], gv[kEwRows];
#pragma unroll
        for (int u = 0; u < kEwRows; ++u) {
            const uint64_t rr = r + u * gy;
            if (rr < rows) {
                const uint64_t pr = pre_rows ? pre_rows[rr] : rr;
                pv[u] = pre[pr * ldp + c];
                gv[u] = g[rr * ldg + c];
            } else {
                pv[u] = gv[u] = 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < kEwRows; ++u) {
            const uint64_t rr = r + u * gy;
            if (rr < rows) out[rr * ldo + c] = pv[u] > 0.f ? gv[u] : 0.f;
        }
    }
}

// std::exp(float) in the reference is glibc's expf. This is its algorithm
// (exp2f_data table, 32 entries + degree-3 polynomial in double), in the
// form glibc 2.39 runs on FMA-capable x86-64 (the ifunc-selected FMA build,
// where r = fma(InvLn2N, x, -kd) and the polynomial steps are fused):
// checked equal to the host's expf for all 2^32 float inputs.
__constant__ unsigned long long kExp2fTab[32] = {0x3ff0000000000000ULL,0x3fefd9b0d3158574ULL,0x3fefb5586cf9890fULL,0x3fef9301d0125b51ULL,0x3fef72b83c7d517bULL,0x3fef54873168b9aaULL,0x3fef387a6e756238ULL,0x3fef1e9df51fdee1ULL,0x3fef06fe0a31b715ULL,0x3feef1a7373aa9cbULL,0x3feedea64c123422ULL,0x3feece086061892dULL,0x3feebfdad5362a27ULL,0x3feeb42b569d4f82ULL,0x3feeab07dd485429ULL,0x3feea47eb03a5585ULL,0x3feea09e667f3bcdULL,0x3fee9f75e8ec5f74ULL,0x3feea11473eb0187ULL,0x3feea589994cce13ULL,0x3feeace5422aa0dbULL,0x3feeb737b0cdc5e5ULL,0x3feec49182a3f090ULL,0x3feed503b23e255dULL,0x3feee89f995ad3adULL,0x3feeff76f2fb5e47ULL,0x3fef199bdd85529cULL,0x3fef3720dcef9069ULL,0x3fef5818dcfba487ULL,0x3fef7c97337b9b5fULL,0x3fefa4afa2a490daULL,0x3fefd0765b6e4540ULL};

__device__ __forceinline__ float expf_glibc(float x) {
    const uint32_t ux = __float_as_uint(x), abstop = (ux >> 20) & 0x7ffu;
    if (abstop >= 0x42bu) {  // |x| >= 88
        if (ux == 0xff800000u) return 0.f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.f;
    }
    constexpr double N = 32.0;
    constexpr double InvLn2N = 0x1.71547652b82fep+0 * N;
    constexpr double Shift = 0x1.8p+52;
    constexpr double C0 = 0x1.c6af84b912394p-5 / N / N / N, C1 = 0x1.ebfce50fac4f3p-3 / N / N,
                     C2 = 0x1.62e42ff0c52d6p-1 / N;
    const double xd = static_cast<double>(x);
    const double z = __dmul_rn(InvLn2N, xd);
    double kd = __dadd_rn(z, Shift);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, Shift);
    const double r = __fma_rn(InvLn2N, xd, -kd);
    const unsigned long long t = kExp2fTab[ki % 32] + (ki << 47);
    const double sc = __longlong_as_double(static_cast<long long>(t));
    const double zz = __fma_rn(C0, r, C1), r2 = __dmul_rn(r, r);
    double y = __fma_rn(C2, r, 1.0);
    y = __fma_rn(zz, r2, y);
    return __double2float_rn(__dmul_rn(y, sc));
}

// dense_matrix.hpp:116-135: per row max (std::max: (a < b) ? b : a),
// o = exp(x - max) in float, serial float sum, divide. Thread per row.
__global__ void k_row_softmax(const float* __restrict__ x, uint64_t ldx, float* __restrict__ out, uint64_t ldo,
                              uint64_t rows, uint64_t cols) {
    const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (r >= rows) return;
    const float* in = x + r * ldx;
    float* o = out + r * ldo;
    float mx = in[0];
    for (uint64_t j = 1; j < cols; ++j) mx = (mx < in[j]) ? in[j] : mx;
    float sum = 0.f;
    for (uint64_t j = 0; j < cols; ++j) {
        const float e = expf_glibc(__fsub_rn(in[j], mx));
        o[j] = e;
        sum = __fadd_rn(sum, e);
    }
    for (uint64_t j = 0; j < cols; ++j) o[j] = __fdiv_rn(o[j], sum);
}

// The same per-row computation with the rows staged through shared memory:
// a block loads kSoftRows rows coalesced (a warp per row, lanes over the
// columns), one thread then runs its row's max / exp + serial sum / divide
// in the reference order from shared memory (odd row stride: no bank
// conflicts), and the block stores the rows coalesced. The thread-per-row
// kernel reads a column of 32 rows per load instruction (32 sectors) and
// ran the products softmax (2.45M x 47) at 0.25 TB/s.
constexpr int kSoftRows = 128;
__global__ void __launch_bounds__(kSoftRows) k_row_softmax_tiled(const float* __restrict__ x, uint64_t ldx,
                                                               float* __restrict__ out, uint64_t ldo, uint64_t rows,
                                                               uint32_t cols) {
    extern __shared__ float t[];
    const uint32_t st = cols | 1u;  // odd stride
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kSoftRows;
    const uint32_t nr = static_cast<uint32_t>(min(static_cast<uint64_t>(kSoftRows), rows - r0));
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kSoftRows / 32;
    for (uint32_t rr = warp; rr < nr; rr += nw)
        for (uint32_t j = lane; j < cols; j += 32) t[rr * st + j] = x[(r0 + rr) * ldx + j];
    __syncthreads();
    if (threadIdx.x < nr) {
        float* row = t + threadIdx.x * st;
        float mx = row[0];
        for (uint32_t j = 1; j < cols; ++j) mx = (mx < row[j]) ? row[j] : mx;
        float sum = 0.f;
        for (uint32_t j = 0; j < cols; ++j) {
            const float e = expf_glibc(__fsub_rn(row[j], mx));
            row[j] = e;
            sum = __fadd_rn(sum, e);
        }
        for (uint32_t j = 0; j < cols; ++j) row[j] = __fdiv_rn(row[j], sum);
    }
    __syncthreads();
    for (uint32_t rr = warp; rr < nr; rr += nw)
        for (uint32_t j = lane; j < cols; j += 32) out[(r0 + rr) * ldo + j] = t[rr * st + j];
}

// engine.hpp:146-156: grad = 0; grad[v] = (probs[v] - r[v]) * inv on V_t
__global__ void k_top_grad(const float* __restrict__ probs, uint64_t ldp, const float* __restrict__ ref,
                           uint64_t ldr, const uint32_t* __restrict__ vt, uint64_t k, float inv,
                           float* __restrict__ out, uint64_t ldo, uint32_t cols, uint64_t rows) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (uint64_t i = blockIdx.y; i < k; i += gridDim.y) {
        const uint64_t v = vt[i];
        if (v >= rows) continue;  // not a vertex of this graph: nothing to write
        out[v * ldo + c] = __fmul_rn(__fsub_rn(probs[v * ldp + c], ref[v * ldr + c]), inv);
    }
}

// aggregate_pull_filtered work counters (aggregate.hpp:139-162): warp per
// destination of the full graph. c = {edges, groups, edges_skipped,
// groups_skipped}.
__global__ void k_filter_counts(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ nbrs, uint32_t n,
                                uint32_t gs, const uint32_t* __restrict__ dst_bits,
                                const uint32_t* __restrict__ src_bits, unsigned long long* __restrict__ c) {
    const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= n) return;
    const uint32_t v = static_cast<uint32_t>(w);
    const uint64_t b = offsets[v], e = offsets[v + 1];
    const uint64_t deg = e - b, groups = (deg + gs - 1) / gs;
    const unsigned lane = lane_id();
    if (!bit_of(dst_bits, v)) {
        if (lane == 0) {
            atomicAdd(c + 2, static_cast<unsigned long long>(deg));
            atomicAdd(c + 3, static_cast<unsigned long long>(groups));
        }
        return;
    }
    unsigned long long on = 0;
    for (uint64_t j = b + lane; j < e; j += 32) on += bit_of(src_bits, __ldg(nbrs + j));
    on = warp_sum(on);
    if (lane == 0) {
        atomicAdd(c + 0, on);
        atomicAdd(c + 1, static_cast<unsigned long long>(groups));
        atomicAdd(c + 2, static_cast<unsigned long long>(deg - on));
    }
}

dim3 rows_grid(uint64_t rows, uint64_t cols, unsigned tx) {
    return dim3(static_cast<unsigned>((cols + tx - 1) / tx),
                static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(rows, 32768))));
}

}  // namespace

void gemm(DMat a, DMat b, DMat out, bool b_transposed, cudaStream_t s, int packed) {
    const uint64_t K = a.cols;
    if (b_transposed ? b.cols != K : b.rows != K) fail_shape("gemm: inner dimensions differ");
    const uint64_t n = a.rows, m = b_transposed ? b.rows : b.cols;
    if (out.rows != n || out.cols != m) fail_shape("gemm: output shape mismatch");
    if (n == 0 || m == 0) return;
    if (K == 0) {
        PG_CUDA(cudaMemset2DAsync(out.p, out.ld * 4, 0, m * 4, n, s));
        return;
    }
    // y_grad = g W^T on the tensor cores when selected (tolerance, not bits)
    // (below K = 32 the write-bound FFMA2 kernel is faster and exact)
    if (b_transposed && tuning(kTuneGemmTc) == 1 && K >= 32 && gemm_a_bt_tc_supported(a)) {
        gemm_a_bt_tc(a, b, out, s);
        return;
    }
    // register-tiled k_gemm3: A rows by 16-byte cp.async (lda % 4 == 0,
    // 16-byte aligned), B k-major (gemm_a_bt transposes W into scratch)
    const bool a16 = (a.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(a.p) & 15) == 0;
    // (m <= 64: a 128-column tile is mostly waste, k_gemm2's 64 wins: the
    // products H W1 at m = 47 runs 4.08 ms there vs 5.02 ms here)
    if (packed < 0) packed = static_cast<int>(tuning(kTuneGemmPacked));
    if (packed == 2 && m > 2 * kGT && a16 &&
        (b_transposed || ((b.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(b.p) & 15) == 0))) {
        volatile float nz = -0.f;
        const float* bk = b.p;
        uint64_t ldbk = b.ld;
        DevBuf<float> bt;
        int dev = 0;
        PG_CUDA(cudaGetDevice(&dev));
        (void)lib_stream(dev);  // the stream-ordered pool keeps the scratch (no re-map per call)
        if (b_transposed) {
            ldbk = (m + 3) & ~3ull;
            bt = DevBuf<float>(K * ldbk, s);
            k_transpose<<<grid_for(m * K, 256), 256, 0, s>>>(b.p, b.ld, bt.get(), ldbk, m, K);
            PG_LAUNCH("k_transpose");
            bk = bt.get();
        }
        // 16 x 8 thread tiles (24 registers loaded per 128 FP instructions)
        // when the rows fill 256-row CTA tiles, else 8 x 8
        const unsigned gy = static_cast<unsigned>((m + kG3N - 1) / kG3N);
        auto launch = [&](auto kern, int rm) {
            const int smem = 2 * (16 * rm * (kG3K + 4) + kG3K * (kG3N + 4)) * 4;
            PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));  // per device
            kern<<<dim3(static_cast<unsigned>((n + 16 * rm - 1) / (16 * rm)), gy), 256, smem, s>>>(
                a.p, a.ld, bk, ldbk, out.p, out.ld, n, m, K, nz);
        };
        if (tuning(kTuneGemm3Rows) == 16)
            launch(k_gemm3<16>, 16);
        else
            launch(k_gemm3<8>, 8);
        PG_LAUNCH("k_gemm3");
        return;
    }
    // 64-column tiles waste most of a narrow output (m <= 32: the forward's
    // X W at width 16 runs 1.01 ms packed vs 0.61 ms scalar)
    if (packed && m > kGT) {
        dim3 grid(static_cast<unsigned>((n + kGI - 1) / kGI), static_cast<unsigned>((m + kG2J - 1) / kG2J));
        volatile float nz = -0.f;  // runtime -0: a literal lets ptxas fold the FFMA2 away
        if (b_transposed)
            k_gemm2<true><<<grid, 256, 0, s>>>(a.p, a.ld, b.p, b.ld, out.p, out.ld, n, m, K, nz);
        else
            k_gemm2<false><<<grid, 256, 0, s>>>(a.p, a.ld, b.p, b.ld, out.p, out.ld, n, m, K, nz);
        PG_LAUNCH("k_gemm2");
        return;
    }
    dim3 grid(static_cast<unsigned>((n + kGI - 1) / kGI), static_cast<unsigned>((m + kGT - 1) / kGT));
    if (b_transposed)
        k_gemm<true><<<grid, 256, 0, s>>>(a.p, a.ld, b.p, b.ld, out.p, out.ld, n, m, K);
    else
        k_gemm<false><<<grid, 256, 0, s>>>(a.p, a.ld, b.p, b.ld, out.p, out.ld, n, m, K);
    PG_LAUNCH("k_gemm");
}

void gemm_at_b(DMat a, const uint32_t* a_rows, DMat b, DMat out, cudaStream_t s) {
    const uint64_t n = b.rows, r = a.cols, c = b.cols;
    if (!a_rows && a.rows != n) fail_shape("gemm_at_b: row counts differ");
    if (out.rows != r || out.cols != c) fail_shape("gemm_at_b: output shape mismatch");
    if (r == 0 || c == 0) return;
    if (n >= (1ull << 31) || r >= (1ull << 31) || c >= (1ull << 31)) fail(kConfig, "gemm_at_b: dimension too large");
    // W' on the tensor cores when selected (split-K 3xTF32: tolerance, not bits)
    if (tuning(kTuneGemmTc) == 1 && gemm_at_b_tc_supported(r, c) && a.ld % 4 == 0 && b.ld % 4 == 0 &&
        reinterpret_cast<uintptr_t>(a.p) % 16 == 0 && reinterpret_cast<uintptr_t>(b.p) % 16 == 0) {
        gemm_at_b_tc(a, a_rows, b, out, s);
        return;
    }
    // one chain warp per SMSP (k_gemm_at_b_quad, tuning atb_quad): the tile
    // shape whose block count comes closest to one block per SM
    const bool v4 = a.ld % 4 == 0 && b.ld % 4 == 0 && reinterpret_cast<uintptr_t>(a.p) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(b.p) % 16 == 0;
    // (wide outputs only: at c = 16 / 41 the 32-column tiles leave chain
    // warps idle and the split kernel wins, Reddit 1.92 vs 1.32 ms)
    // atb_quad 3 (default): only for W' over whole matrices (no row
    // gather: the all-active / if-else / Global EPP chains, products 47 ->
    // 39 ms); beside the Local EPP chain's SpMM it lost (16.7 -> 28.6 ms)
    const int64_t quad = tuning(kTuneAtbQuad);
    const bool quad_on = quad == 1 || quad == 2 || (quad == 3 && !a_rows);
    if (quad_on && tuning(kTuneAtbSplit) && v4 && c >= 64) {
        int dev = 0, sms = 148;
        PG_CUDA(cudaGetDevice(&dev));
        PG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        struct Cand {
            int ti, tcw;
        };
        const Cand cands[] = {{8, 8}, {16, 4}, {8, 4}, {4, 8}, {4, 4}};
        int best = -1;
        uint64_t best_blocks = 0;
        const uint64_t sm64 = static_cast<uint64_t>(sms);
        for (int k = 0; k < 5; ++k) {
            const uint64_t bl =
                ((r + cands[k].ti - 1) / cands[k].ti) * ((c + 4 * cands[k].tcw - 1) / (4 * cands[k].tcw));
            const bool better = best < 0 ? true
                                : bl <= sm64 ? (best_blocks > sm64 || bl > best_blocks)
                                             : (best_blocks > sm64 && bl < best_blocks);
            if (better) {
                best = k;
                best_blocks = bl;
            }
        }
        volatile float nz = -0.f;
        const uint32_t n32 = static_cast<uint32_t>(n), r32 = static_cast<uint32_t>(r), c32 = static_cast<uint32_t>(c);
        const Cand cd = cands[best];
        const dim3 grid(static_cast<unsigned>((r + cd.ti - 1) / cd.ti),
                        static_cast<unsigned>((c + 4 * cd.tcw - 1) / (4 * cd.tcw)));
        auto go = [&](auto kern, size_t smem) {
            PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            kern<<<grid, 256, smem, s>>>(a.p, a.ld, a_rows, b.p, b.ld, out.p, out.ld, n32, r32, c32, nz);
        };
        auto pick = [&](auto qs, auto ql) {  // slots / stages in flight
            constexpr int QS = decltype(qs)::value, QL = decltype(ql)::value;
            if (cd.ti == 8 && cd.tcw == 8)
                go(k_gemm_at_b_quad<8, 8, QS, QL>, sizeof(AtbQuadSmem<8, 8, QS, QL>));
            else if (cd.ti == 16)
                go(k_gemm_at_b_quad<16, 4, QS, QL>, sizeof(AtbQuadSmem<16, 4, QS, QL>));
            else if (cd.ti == 8)
                go(k_gemm_at_b_quad<8, 4, QS, QL>, sizeof(AtbQuadSmem<8, 4, QS, QL>));
            else if (cd.tcw == 8)
                go(k_gemm_at_b_quad<4, 8, QS, QL>, sizeof(AtbQuadSmem<4, 8, QS, QL>));
            else
                go(k_gemm_at_b_quad<4, 4, QS, QL>, sizeof(AtbQuadSmem<4, 4, QS, QL>));
        };
        if (tuning(kTuneAtbQuad) == 2)
            pick(std::integral_constant<int, 10>{}, std::integral_constant<int, 8>{});
        else
            pick(std::integral_constant<int, 6>{}, std::integral_constant<int, 4>{});
        PG_LAUNCH("k_gemm_at_b_quad");
        return;
    }
    // 64 chains per warp: 4 (or 8) A columns x 16 (or 8) B columns
    if (c <= 8) launch_at_b<8>(a, a_rows, b, out, n, r, c, s);
    else launch_at_b<4>(a, a_rows, b, out, n, r, c, s);
}

void relu(DMat x, DMat out, cudaStream_t s) {
    if (x.rows != out.rows || x.cols != out.cols) fail_shape("relu: shape mismatch");
    if (x.rows * x.cols == 0) return;
    k_relu<<<rows_grid(x.rows, x.cols, 128), 128, 0, s>>>(x.p, x.ld, out.p, out.ld, x.rows,
                                                         static_cast<uint32_t>(x.cols));
    PG_LAUNCH("k_relu");
}

void relu_backward_rows(DMat g, DMat pre, const uint32_t* pre_rows, DMat out, cudaStream_t s) {
    if (g.rows != out.rows || g.cols != out.cols || pre.cols != g.cols || (!pre_rows && pre.rows != g.rows))
        fail_shape("relu_backward: shape mismatch");
    if (g.rows * g.cols == 0) return;
    k_relu_bwd_rows<<<rows_grid(g.rows, g.cols, 128), 128, 0, s>>>(g.p, g.ld, pre.p, pre.ld, pre_rows, out.p, out.ld,
                                                                   g.rows, static_cast<uint32_t>(g.cols));
    PG_LAUNCH("k_relu_bwd_rows");
}

void row_softmax(DMat x, DMat out, cudaStream_t s) {
    if (x.cols == 0) fail_shape("row_softmax: zero columns");
    if (x.rows != out.rows || x.cols != out.cols) fail_shape("row_softmax: shape mismatch");
    if (x.rows == 0) return;
    const size_t smem = static_cast<size_t>(kSoftRows) * ((x.cols | 1) * 4);
    if (smem <= 48 * 1024) {
        k_row_softmax_tiled<<<static_cast<unsigned>((x.rows + kSoftRows - 1) / kSoftRows), kSoftRows, smem, s>>>(
            x.p, x.ld, out.p, out.ld, x.rows, static_cast<uint32_t>(x.cols));
        PG_LAUNCH("k_row_softmax_tiled");
        return;
    }
    k_row_softmax<<<grid_for(x.rows, 128), 128, 0, s>>>(x.p, x.ld, out.p, out.ld, x.rows, x.cols);
    PG_LAUNCH("k_row_softmax");
}

void top_grad_from_probs(DMat probs, DMat ref, const uint32_t* vt, uint64_t k, DMat out, cudaStream_t s) {
    if (probs.rows != ref.rows || probs.cols != ref.cols || out.rows != probs.rows || out.cols != probs.cols)
        fail_shape("top_grad_from_probs: shapes differ");
    if (out.rows * out.cols) PG_CUDA(cudaMemset2DAsync(out.p, out.ld * 4, 0, out.cols * 4, out.rows, s));
    if (k == 0 || out.cols == 0) return;
    const float inv = 1.0f / static_cast<float>(k);  // T(1) / static_cast<T>(vt.size())
    k_top_grad<<<rows_grid(k, out.cols, 64), 64, 0, s>>>(probs.p, probs.ld, ref.p, ref.ld, vt, k, inv, out.p, out.ld,
                                                          static_cast<uint32_t>(out.cols), out.rows);
    PG_LAUNCH("k_top_grad");
}

void filter_counts(const Graph& g, uint32_t gs, const uint32_t* dst_bits, const uint32_t* src_bits, uint64_t* c4,
                   cudaStream_t s) {
    DevBuf<unsigned long long> c(4, s);
    PG_CUDA(cudaMemsetAsync(c.get(), 0, 32, s));
    if (g.n) {
        k_filter_counts<<<grid_for(static_cast<uint64_t>(g.n) * 32, kThreads), kThreads, 0, s>>>(
            g.offsets.get(), g.nbrs.get(), g.n, gs, dst_bits, src_bits, c.get());
        PG_LAUNCH("k_filter_counts");
    }
    PG_CUDA(cudaMemcpyAsync(c4, c.get(), 32, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace pg

// ============================================================================
// The chains. Temporaries are stream-ordered pool allocations on s; every
// call is asynchronous on s except where a counter needs a host value.
namespace pg {

namespace {

struct Tmp {
    DevBuf<float> buf;
    DMat m;
    Tmp(uint64_t rows, uint64_t cols, cudaStream_t s, bool zero = false) : buf(rows * pad_ld(cols), s) {
        m = DMat{buf.get(), rows, cols, pad_ld(cols)};
        if (zero && rows * cols) PG_CUDA(cudaMemsetAsync(buf.get(), 0, rows * pad_ld(cols) * 4, s));
    }
};

void check_chain(const BackwardIO& io, uint64_t n) {
    if (io.L == 0) fail(kConfig, "backward: need at least one layer");
    for (uint64_t l = 0; l < io.L; ++l) {
        if (io.y[l].rows != n || io.y[l].cols != io.w[l].rows)
            fail_shape("backward: Y^(l) shape does not match W^(l) at layer " + std::to_string(l));
        if (io.pre[l].rows != n || io.pre[l].cols != io.w[l].cols)
            fail_shape("backward: pre-activation shape mismatch at layer " + std::to_string(l));
        if (l > 0 && io.w[l].rows != io.w[l - 1].cols) fail_shape("backward: weight chain mismatch");
        if (io.w_grads[l].rows != io.w[l].rows || io.w_grads[l].cols != io.w[l].cols)
            fail_shape("backward: W gradient shape mismatch at layer " + std::to_string(l));
    }
    if (io.top_grad.rows != n || io.top_grad.cols != io.w[io.L - 1].cols)
        fail_shape("backward: top gradient shape mismatch");
}

// W' = Y^T g on a forked stream (tuning "wgrad_fork"). The W gradients are
// chain outputs that nothing later in the chain reads, so each one overlaps
// the y_grad GEMM and the SpMM of its layer (the serial-order GEMM is
// latency-bound; the SpMM it hides behind is bandwidth-bound). Measured:
// Reddit backward_epp 17.9 -> 17.8 ms, products 22.2 -> 18.8, arxiv 2.85 ->
// 2.49 (with the one-warp W' kernel the 400-block products GEMM lost more
// to SMSP sharing than it hid, so the fork was limited to <= 160 blocks).
// Every g it reads is kept alive until join(), which makes the caller's
// stream wait for the last W' (stream-ordered frees then follow the join).
struct WGradSide {
    cudaStream_t main;
    cudaStream_t side;
    cudaEvent_t fork, done;
    std::vector<std::unique_ptr<Tmp>> keep;
    bool used = false;
    explicit WGradSide(cudaStream_t s) : main(s) {
        struct PerDev {
            cudaStream_t s = nullptr;
            cudaEvent_t fork = nullptr, done = nullptr;
        };
        static thread_local std::vector<PerDev> per_dev;
        int dev = 0;
        PG_CUDA(cudaGetDevice(&dev));
        if (static_cast<int>(per_dev.size()) <= dev) per_dev.resize(dev + 1);
        PerDev& d = per_dev[dev];
        if (!d.s) {
            // highest priority: the latency-bound W' chains take SMs as soon
            // as blocks of the bandwidth-bound y_grad GEMM / SpMM retire
            // (with the register-tiled y_grad GEMM filling every SM they
            // started late: products backward_epp 19.7 -> 24.2 ms)
            int lo = 0, hi = 0;
            PG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            PG_CUDA(cudaStreamCreateWithPriority(&d.s, cudaStreamNonBlocking, hi));
            PG_CUDA(cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming));
            PG_CUDA(cudaEventCreateWithFlags(&d.done, cudaEventDisableTiming));
        }
        side = d.s;
        fork = d.fork;
        done = d.done;
    }
    void gemm_at_b(DMat a, const uint32_t* rows, DMat b, DMat out) {
        if (!tuning(kTuneWgradFork)) {
            pg::gemm_at_b(a, rows, b, out, main);
            return;
        }
        PG_CUDA(cudaEventRecord(fork, main));
        PG_CUDA(cudaStreamWaitEvent(side, fork, 0));
        pg::gemm_at_b(a, rows, b, out, side);
        used = true;
    }
    // y_grad product beside a forked W' chain (tuning "gemm_beside_wgrad",
    // the EPP chain over compact frontier rows): the register-tiled k_gemm3
    // fills every SMSP with FP work and the latency-bound W' chains, that
    // chain's critical path, lose their issue slots (products backward_epp
    // 18.1 -> 24.3 ms); k_gemm2 leaves them room. The full-graph chains keep
    // k_gemm3 (products Global EPP 68.8 -> 47.5 ms)
    int beside_packed() const {
        return used && tuning(kTuneGemmPacked) == 2 && tuning(kTuneGemmBesideWgrad) ? 1 : -1;
    }
    void retire(std::unique_ptr<Tmp>& g) {
        if (g) keep.push_back(std::move(g));
    }
    void join() {
        if (!used) return;
        PG_CUDA(cudaEventRecord(done, side));
        PG_CUDA(cudaStreamWaitEvent(main, done, 0));
        used = false;
    }
    ~WGradSide() {
        if (used) {  // unwinding after a failure: still order the frees after the side work
            cudaEventRecord(done, side);
            cudaStreamWaitEvent(main, done, 0);
        }
    }
};

// The full-graph backward shared by Alg. 1 (all-active) and the if-else
// filter: per layer W' = Y^T g, y_grad = g W^T, x_grad = pull(y_grad), and
// g = relu_backward(x_grad, pre[l-1]) fused into the SpMM epilogue.
void backward_full(Groups& G, Frontiers* F, const BackwardIO& io, cudaStream_t s) {
    if (!G.graph) fail(kConfig, "backward: needs a grouping of the full graph");
    Graph& gr = *G.graph;
    const uint64_t n = gr.n, L = io.L;
    check_chain(io, n);
    if (F && F->L != L) fail_stale("ifelse backward: frontiers were computed for a different depth");
    WGradSide wgs(s);
    std::unique_ptr<Tmp> gcur;
    DMat g = io.top_grad;
    for (uint64_t l = L; l-- > 0;) {
        const uint64_t in_dim = io.w[l].rows;
        wgs.gemm_at_b(io.y[l], nullptr, g, io.w_grads[l]);
        Tmp yg(n, in_dim, s);
        gemm(g, io.w[l], yg.m, true, s);
        AggExt ext;
        if (F) {
            ext.dst_bits = F->levels[L - l].bits.get();
            ext.src_bits = F->levels[L - l - 1].bits.get();
        }
        DMat* xo = io.x_grads ? &io.x_grads[L - 1 - l] : nullptr;
        if (xo && (xo->rows != n || xo->cols != in_dim)) fail_shape("backward: x_grad shape mismatch");
        std::unique_ptr<Tmp> gnext;
        if (l > 0 && !xo) {  // fused: the SpMM writes relu_backward(x_grad, pre[l-1])
            gnext = std::make_unique<Tmp>(n, in_dim, s, F != nullptr);
            ext.relu_pre = io.pre[l - 1].p;
            ext.ld_pre = io.pre[l - 1].ld;
            run_aggregate(G, false, 0, gr.n, yg.m.p, yg.m.ld, gnext->m.p, gnext->m.ld, in_dim, PG_AGG_OVERWRITE, s,
                          SegSel{}, ext);
        } else {
            std::unique_ptr<Tmp> xt;
            DMat x = xo ? *xo : DMat{};
            if (!xo) {
                xt = std::make_unique<Tmp>(n, in_dim, s, F != nullptr);
                x = xt->m;
            } else if (F) {
                PG_CUDA(cudaMemset2DAsync(x.p, x.ld * 4, 0, x.cols * 4, x.rows, s));
            }
            run_aggregate(G, false, 0, gr.n, yg.m.p, yg.m.ld, x.p, x.ld, in_dim, PG_AGG_OVERWRITE, s, SegSel{}, ext);
            if (l > 0) {
                gnext = std::make_unique<Tmp>(n, in_dim, s);
                relu_backward_rows(x, io.pre[l - 1], nullptr, gnext->m, s);
            }
        }
        if (io.edges) {
            if (F) {
                uint64_t c[4];
                filter_counts(gr, G.gs, ext.dst_bits, ext.src_bits, c, s);
                io.edges[L - 1 - l] = c[0];
            } else {
                io.edges[L - 1 - l] = gr.m;
            }
        }
        if (l > 0) {
            wgs.retire(gcur);
            gcur = std::move(gnext);
            g = gcur->m;
        }
    }
    wgs.join();
}

}  // namespace

void forward(Groups& G, DMat x0, const DMat* w, uint64_t L, DMat* y, DMat* pre, DMat* x, cudaStream_t s) {
    if (!G.graph) fail(kConfig, "forward: needs a grouping of the full graph");
    const uint64_t n = G.graph->n;
    DMat cur = x0;
    if (x0.rows != n) fail_shape("forward: feature rows != vertex count");
    for (uint64_t l = 0; l < L; ++l) {
        if (cur.cols != w[l].rows)
            fail_shape("forward: feature/weight shape mismatch at layer " + std::to_string(l));
        if (y[l].rows != n || y[l].cols != cur.cols || pre[l].rows != n || pre[l].cols != w[l].cols ||
            x[l].rows != n || x[l].cols != w[l].cols)
            fail_shape("forward: output shape mismatch at layer " + std::to_string(l));
        run_aggregate(G, false, 0, G.graph->n, cur.p, cur.ld, y[l].p, y[l].ld, cur.cols, PG_AGG_OVERWRITE, s);
        gemm(y[l], w[l], pre[l], false, s);
        if (l + 1 < L) relu(pre[l], x[l], s);
        else row_softmax(pre[l], x[l], s);
        cur = x[l];
    }
}

void backward_all_active(Groups& G, const BackwardIO& io, cudaStream_t s) { backward_full(G, nullptr, io, s); }

void backward_ifelse(Groups& G, Frontiers& F, const BackwardIO& io, cudaStream_t s) { backward_full(G, &F, io, s); }

void backward_epp(Groups* const* PG, Frontiers& F, const BackwardIO& io, int gather_mode, uint64_t expected_fp,
                  cudaStream_t s) {
    const uint64_t L = io.L;
    if (F.L != L) fail_stale("epp backward: paths were prepared for a different layer count");
    for (uint64_t i = 0; i < L; ++i) {
        if (!PG[i] || !PG[i]->path) fail(kConfig, "epp backward: every grouping must be over an execution path");
        if (PG[i]->path->layer != L - 1 - i) fail_stale("epp backward: paths were prepared for a different layer count");
        if (PG[i]->path->fingerprint != expected_fp)
            fail_stale("epp backward: execution paths are stale for this graph/training set");
    }
    const uint64_t n = F.n;
    check_chain(io, n);
    if (gather_mode == 1) {  // Global: full-width matrices, the path walked with global ids
        if (io.x_grads) fail(kConfig, "epp backward: x_grads are only captured in Local gather mode");
        WGradSide wgs(s);
        std::unique_ptr<Tmp> gcur;
        DMat g = io.top_grad;
        for (uint64_t i = 0; i < L; ++i) {
            const uint64_t l = L - 1 - i, in_dim = io.w[l].rows;
            Path& p = *PG[i]->path;
            {
                // long-lived cache: built on the library stream (where it is
                // freed) and synchronised, under the path's lock
                std::lock_guard<std::mutex> lk(p.mu);
                if (!p.edges_global.get() && p.E) {
                    cudaStream_t ls = lib_stream(p.device);
                    PG_CUDA(cudaStreamSynchronize(s));  // F's ids are final
                    DevBuf<Edge> eg = edge_buf(p.E, ls);
                    remap_edges(p.edges_parent.get(), p.E, F.levels[i].ids.get(), eg.get(), ls);
                    PG_CUDA(cudaStreamSynchronize(ls));
                    p.edges_global = std::move(eg);
                }
            }
            wgs.gemm_at_b(io.y[l], nullptr, g, io.w_grads[l]);
            Tmp yg(n, in_dim, s);
            gemm(g, io.w[l], yg.m, true, s);
            auto gn = std::make_unique<Tmp>(n, in_dim, s, true);  // rows off the path stay +0
            AggExt ext;
            ext.out_rows = p.dest.get();
            if (l > 0) {
                ext.relu_pre = io.pre[l - 1].p;
                ext.ld_pre = io.pre[l - 1].ld;
            }
            run_aggregate(*PG[i], true, 0, p.D, yg.m.p, yg.m.ld, gn->m.p, gn->m.ld, in_dim, PG_AGG_OVERWRITE, s,
                          SegSel{}, ext, p.edges_global.get());
            if (io.edges) io.edges[i] = p.E;
            wgs.retire(gcur);
            gcur = std::move(gn);
            g = gcur->m;
        }
        wgs.join();
        return;
    }
    // Local: compact matrices whose rows follow the frontier arrays
    const uint64_t c = io.top_grad.cols;
    auto g0 = std::make_unique<Tmp>(F.levels[0].size, c, s);
    gather_rows(io.top_grad.p, io.top_grad.ld, F.levels[0].ids.get(), F.levels[0].size, g0->m.p, g0->m.ld, c, s);
    WGradSide wgs(s);
    std::unique_ptr<Tmp> gcur = std::move(g0);
    for (uint64_t i = 0; i < L; ++i) {
        const uint64_t l = L - 1 - i, in_dim = io.w[l].rows;
        Path& p = *PG[i]->path;
        if (p.P != F.levels[i].size || p.D != F.levels[i + 1].size)
            fail_stale("epp backward: path does not follow the frontiers");
        const DMat g = gcur->m;
        wgs.gemm_at_b(io.y[l], F.levels[i].ids.get(), g, io.w_grads[l]);  // gather_rows(Y, in_rows) fused
        Tmp yg(p.P, in_dim, s);
        gemm(g, io.w[l], yg.m, true, s, wgs.beside_packed());
        DMat* xo = io.x_grads ? &io.x_grads[i] : nullptr;
        if (xo && (xo->rows != p.D || xo->cols != in_dim)) fail_shape("backward: x_grad shape mismatch");
        std::unique_ptr<Tmp> gn;
        if (l > 0 && !xo) {  // relu_backward(x_grad, gather_rows(pre, levels[L-l])) in the SpMM epilogue
            gn = std::make_unique<Tmp>(p.D, in_dim, s);
            AggExt ext;
            ext.relu_pre = io.pre[l - 1].p;
            ext.ld_pre = io.pre[l - 1].ld;
            ext.pre_rows = p.dest.get();
            run_aggregate(*PG[i], true, 0, p.D, yg.m.p, yg.m.ld, gn->m.p, gn->m.ld, in_dim, PG_AGG_OVERWRITE, s,
                          SegSel{}, ext);
        } else {
            std::unique_ptr<Tmp> xt;
            DMat x = xo ? *xo : DMat{};
            if (!xo) {
                xt = std::make_unique<Tmp>(p.D, in_dim, s);
                x = xt->m;
            }
            run_aggregate(*PG[i], true, 0, p.D, yg.m.p, yg.m.ld, x.p, x.ld, in_dim, PG_AGG_OVERWRITE, s);
            if (l > 0) {
                gn = std::make_unique<Tmp>(p.D, in_dim, s);
                relu_backward_rows(x, io.pre[l - 1], p.dest.get(), gn->m, s);
            }
        }
        if (io.edges) io.edges[i] = p.E;
        if (gn) {
            wgs.retire(gcur);
            gcur = std::move(gn);
        }
    }
    wgs.join();
}

}  // namespace pg
