// Tensor-core gemm_a_bt (dense_matrix.hpp:78-95: out[n x m] = a[n x K] *
// b[m x K]^T) on the 5th-generation tensor cores: tcgen05.mma kind::tf32
// with the fp32 operands split 3 ways (3xTF32) so the product keeps ~fp32
// accuracy: a = ah + al with ah = a with its low 13 mantissa bits cleared
// (exactly a TF32 value) and al = a - ah (exact in fp32), likewise b, and
//   a.b ~= ah.bh + ah.bl + al.bh        (the al.bl term is below 2^-22 |a||b|)
// accumulated in fp32 in TMEM. This re-associates the K sum, so it is NOT
// bit-exact with the reference's serial chain: it is selected explicitly
// (PG_GEMM_TF32X3 / tuning "gemm_tc") and gated by the 1e-5 relative /
// 1e-6 absolute tolerance against the f64 product (tests/test_gpu_gemm_tc.py).
// The default gemm_a_bt stays the bit-exact FFMA2 kernel (engine.cu).
//
// Persistent, warp-specialised CTA (one per SM, 320 threads):
//   warp 0      TMA producer: per stage, the raw fp32 A tile(s) [128 x 32]
//               (cp.async.bulk.tensor, SWIZZLE_128B, out-of-bounds rows and
//               K columns zero-filled) and the pre-split B image of this
//               (N tile, k block) (one cp.async.bulk of hi + lo);
//   warp 1      TMEM allocation + the single MMA-issuing thread: per stage
//               3 x 4 tcgen05.mma (K = 8 each) per 128-row sub-tile into a
//               double-buffered TMEM accumulator, tcgen05.commit frees the
//               stage and, after the last k block, hands the tile to ...
//   warps 2-5   splitters: ah in place, al into its own buffer (the same
//               swizzled position: the split is element-wise), then
//               fence.proxy.async so the tensor core sees the generic writes;
//   warps 6-9   epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes
//               32*(w%4)..), streaming 128-bit stores of the fp32 rows,
//               overlapped with the next tile's MMAs (second accumulator).
#include <cuda.h>

#include <cstring>
#include <type_traits>
#include <mutex>
#include <vector>

#include "../../include/pathgcn_b200.h"
#include "pg_internal.h"

namespace pg {

namespace {

constexpr int kTcThreads = 320;
constexpr int kKB = 32;             // fp32 elements per k block = one 128-byte swizzle row
constexpr int kTileBytesA = 128 * 128;  // one 128-row x 32-float sub-tile
constexpr int kMaxN = 256;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TC_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra.uni TC_DONE;\n\t"
        "bra.uni TC_WAIT;\n"
        "TC_DONE:\n\t}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// SWIZZLE_128B, K-major shared-memory matrix descriptor (tcgen05 format):
// start address >> 4, LBO = 1 (unused for swizzled K-major), SBO = 1024 B
// between 8-row groups, version 1 (bits 46-47), layout type 2 = 128B swizzle.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// instruction descriptor, kind::tf32: D f32 (bits 4-5 = 1), A/B TF32 (bits
// 7-9, 10-12 = 2), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
__host__ __device__ constexpr uint32_t tf32_idesc(uint32_t M, uint32_t N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ uint32_t tf32_hi(uint32_t x) { return x & 0xFFFFE000u; }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

template <int MT>
struct TcShape {
    static constexpr int kABytes = MT * kTileBytesA;  // raw (-> hi) A of one stage; lo the same again
};

// B image of one (N tile, k block): hi then lo, each N rows x 128 bytes,
// K-major SWIZZLE_128B (16-byte chunk c of row r at chunk c ^ (r & 7)).
__global__ void k_tc_pack_b(const float* __restrict__ b, uint64_t ldb, uint32_t m, uint32_t K, uint32_t N,
                            uint32_t NT, uint32_t KB, float* __restrict__ img) {
    const uint64_t total = static_cast<uint64_t>(NT) * KB * N * kKB;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t k = static_cast<uint32_t>(i % kKB);
        const uint32_t r = static_cast<uint32_t>((i / kKB) % N);
        const uint32_t kb = static_cast<uint32_t>((i / (kKB * static_cast<uint64_t>(N))) % KB);
        const uint32_t nt = static_cast<uint32_t>(i / (kKB * static_cast<uint64_t>(N) * KB));
        const uint32_t row = nt * N + r, col = kb * kKB + k;
        const float v = (row < m && col < K) ? b[row * ldb + col] : 0.f;
        const uint32_t hb = tf32_hi(__float_as_uint(v));
        const float hi = __uint_as_float(hb), lo = __fsub_rn(v, hi);
        const uint64_t stage = (static_cast<uint64_t>(nt) * KB + kb) * (2ull * N * kKB);
        const uint32_t pos = r * kKB + (((k >> 2) ^ (r & 7)) << 2) + (k & 3);
        img[stage + pos] = hi;
        img[stage + static_cast<uint64_t>(N) * kKB + pos] = lo;
    }
}

struct TcParams {
    float* out;
    uint64_t ldo;
    uint64_t n, m;
    uint32_t N;         // N tile (multiple of 8, <= 256)
    uint32_t NT, KB;    // N tiles, k blocks
    uint32_t stages;
    uint32_t acc_stride;  // TMEM columns per accumulator (>= N, multiple of 32)
    uint64_t row_tiles;
    const float* bimg;
    int vec_out;
};

template <int MT>
__global__ void __launch_bounds__(kTcThreads, 1) k_gemm_abt_tc(const __grid_constant__ CUtensorMap amap, TcParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle atoms
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t N = P.N, S = P.stages;
    const uint32_t bbytes = 2u * N * 128u;
    const uint32_t stage_bytes = 2u * TcShape<MT>::kABytes + bbytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* full = bars;            // [S] TMA landed
    uint64_t* split = bars + S;       // [S] hi/lo written
    uint64_t* empty = bars + 2 * S;   // [S] MMAs done reading
    uint64_t* tfull = bars + 3 * S;   // [2] accumulator ready
    uint64_t* tempty = bars + 3 * S + 2;  // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&split[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // 512 TMEM columns: two accumulators of MT x acc_stride
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    const uint64_t tiles = P.row_tiles * P.NT;
    if (warp == 0) {
        if (lane == 0) {
            uint32_t q = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                const uint32_t nt = static_cast<uint32_t>(t % P.NT);
                const uint64_t rt = t / P.NT;
                for (uint32_t kb = 0; kb < P.KB; ++kb, ++q) {
                    const uint32_t s = q % S, ph = (q / S) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    unsigned char* st = smem + s * stage_bytes;
                    mbar_arrive_tx(&full[s], TcShape<MT>::kABytes + bbytes);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
                        tma_load_2d(st + mt * kTileBytesA, &amap, static_cast<int>(kb * kKB),
                                    static_cast<int>(rt * 128 * MT + mt * 128), &full[s]);
                    bulk_load(st + 2 * TcShape<MT>::kABytes,
                              P.bimg + (static_cast<uint64_t>(nt) * P.KB + kb) * (2ull * N * kKB), bbytes, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tf32_idesc(128, N);
            uint32_t q = 0, it = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
                const uint32_t buf = it & 1, bph = (it >> 1) & 1;
                mbar_wait(&tempty[buf], bph ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (uint32_t kb = 0; kb < P.KB; ++kb, ++q) {
                    const uint32_t s = q % S, ph = (q / S) & 1;
                    mbar_wait(&split[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned char* st = smem + s * stage_bytes;
                    const uint32_t a_hi = smem_addr(st), a_lo = a_hi + TcShape<MT>::kABytes;
                    const uint32_t b_hi = a_hi + 2 * TcShape<MT>::kABytes, b_lo = b_hi + N * 128;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const uint32_t d = tmem + (buf * MT + mt) * P.acc_stride;
#pragma unroll
                        for (int k = 0; k < kKB / 8; ++k) {  // K = 8 per MMA: 32 bytes along the swizzled row
                            const uint32_t ko = k * 32;
                            const uint32_t acc0 = (kb | k) ? 1u : 0u;
                            const uint64_t ah = sw128_desc(a_hi + mt * kTileBytesA + ko);
                            const uint64_t al = sw128_desc(a_lo + mt * kTileBytesA + ko);
                            const uint64_t bh = sw128_desc(b_hi + ko), bl = sw128_desc(b_lo + ko);
                            mma_tf32(d, ah, bh, idesc, acc0);
                            mma_tf32(d, ah, bl, idesc, 1u);
                            mma_tf32(d, al, bh, idesc, 1u);
                        }
                    }
                    mma_commit(&empty[s]);  // stage s free once these MMAs have read it
                }
                mma_commit(&tfull[buf]);  // accumulator complete
            }
        }
    } else if (warp < 6) {
        // splitters: 128 threads, 16-byte chunks of the stage's A tile(s)
        const uint32_t tid = threadIdx.x - 64;
        uint32_t q = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            for (uint32_t kb = 0; kb < P.KB; ++kb, ++q) {
                const uint32_t s = q % S, ph = (q / S) & 1;
                mbar_wait(&full[s], ph);
                // shared-window addresses (LDS/STS, not generic LD/ST)
                const uint32_t hi = smem_addr(smem + s * stage_bytes);
                const uint32_t lo = hi + TcShape<MT>::kABytes;
#pragma unroll 4
                for (uint32_t c = tid; c < TcShape<MT>::kABytes / 16; c += 128) {
                    uint32_t v0, v1, v2, v3;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                                 : "r"(hi + c * 16));
                    const uint32_t h0 = tf32_hi(v0), h1 = tf32_hi(v1), h2 = tf32_hi(v2), h3 = tf32_hi(v3);
                    const uint32_t l0 = __float_as_uint(__fsub_rn(__uint_as_float(v0), __uint_as_float(h0)));
                    const uint32_t l1 = __float_as_uint(__fsub_rn(__uint_as_float(v1), __uint_as_float(h1)));
                    const uint32_t l2 = __float_as_uint(__fsub_rn(__uint_as_float(v2), __uint_as_float(h2)));
                    const uint32_t l3 = __float_as_uint(__fsub_rn(__uint_as_float(v3), __uint_as_float(h3)));
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(hi + c * 16), "r"(h0), "r"(h1),
                                 "r"(h2), "r"(h3)
                                 : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(lo + c * 16), "r"(l0), "r"(l1),
                                 "r"(l2), "r"(l3)
                                 : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (tid == 0) mbar_arrive(&split[s]);
            }
        }
    } else {
        // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 = rows of the sub-tile
        const uint32_t quarter = warp & 3;
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            const uint32_t buf = it & 1, bph = (it >> 1) & 1;
            const uint32_t nt = static_cast<uint32_t>(t % P.NT);
            const uint64_t rt = t / P.NT;
            mbar_wait(&tfull[buf], bph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t col0 = static_cast<uint64_t>(nt) * N;
            for (int mt = 0; mt < MT; ++mt) {
                const uint64_t row = rt * 128 * MT + mt * 128 + quarter * 32 + lane;
                const uint32_t tbase = tmem + ((quarter * 32) << 16) + (buf * MT + mt) * P.acc_stride;
                float* orow = P.out + row * P.ldo + col0;
                for (uint32_t c = 0; c < N; c += 32) {
                    uint32_t v[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
                        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
                        "%30, %31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(tbase + c));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (row >= P.n) continue;
                    const uint64_t cg = col0 + c;
                    if (P.vec_out && c + 32 <= N && cg + 32 <= P.m) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            __stcs(reinterpret_cast<float4*>(orow + c + j),
                                   make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                               __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])));
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c + j < N && cg + j < P.m) orow[c + j] = __uint_as_float(v[j]);
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---- gemm_at_b on the tensor cores: W' = gather_rows(Y, rows)^T g -----------
// dense_matrix.hpp:57-76 (+ engine.hpp:323-324's gather folded in):
//   out[i][j] = sum_r Y[row(r)][i] * g[r][j],  i < in_dim (M), j < out_dim (N),
// the reduction over the n rows. Split-K: each persistent CTA owns a
// contiguous row range and accumulates the whole (in_dim x out_dim) tile in
// TMEM (MT 128-row M tiles x N columns, 3xTF32: ah.bh + ah.bl + al.bh), then
// writes its partial; k_atb_reduce adds the CTA partials in CTA order
// (deterministic run to run, re-associated vs the reference's serial chain:
// fp32 tolerance, not bit-exact).
// Operands are MN-major (a row of Y / g is contiguous along M / N). For
// 32-bit (tf32) MN-major operands tcgen05 takes the SWIZZLE_128B_BASE32B
// layout (descriptor layout type 1; CUTLASS Layout_MN_SW128_32B_Atom): atoms
// of 4 K rows x 32 MN elements (512 B), the 32-byte granule g of row k at
// g ^ (k & 3), atoms along MN at LBO = 512 B, 4-row K groups at SBO. (The
// 8-row SWIZZLE_128B MN-major form reads as zeros for tf32 — measured,
// tools/probes/umma_mn_probe.cu.) Producers (8 warps) gather the rows with
// coalesced 128-bit loads (one prefetched K tile ahead), split hi/lo in
// registers and store both straight into the swizzled slots.
constexpr int kAtbProducers = 8;
constexpr int kAtbThreads = 32 * (2 + kAtbProducers);  // MMA/TMEM warp, epilogue-lead, producers
constexpr int kAtbKT = 16;  // rows per K tile (two 8-row K groups)

__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(512 >> 4) << 16;             // LBO: next 32-element MN atom
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;  // SBO: next 4-row K group
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(1) << 61;                    // SWIZZLE_128B_BASE32B
    return d;
}
// kind::tf32, D f32, A and B MN-major (bits 15, 16)
__host__ __device__ constexpr uint32_t tf32_idesc_mn(uint32_t M, uint32_t N) {
    return tf32_idesc(M, N) | (1u << 15) | (1u << 16);
}

struct AtbParams {
    const float* a;
    uint64_t lda;
    const uint32_t* a_rows;  // nullable
    const float* b;
    uint64_t ldb;
    uint64_t n;              // rows (the K extent)
    uint32_t in_dim, out_dim;
    uint32_t Npad;           // out_dim rounded up to 32
    uint32_t stages;
    uint64_t rows_per_cta;
    float* part;             // [gridDim.x][in_dim][out_dim]
};

template <int MT>
__global__ void __launch_bounds__(kAtbThreads, 1) k_gemm_atb_tc(AtbParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t kAtile = 128u * kAtbKT * 4u;  // one M tile of one K tile, bytes
    const uint32_t Np = P.Npad, S = P.stages;
    const uint32_t bbytes = Np * kAtbKT * 4u;
    const uint32_t stage_bytes = 2u * MT * kAtile + 2u * bbytes;
    const uint32_t sbo_a = 4u * 512u, sbo_b = (Np / 32u) * 512u;  // K-group strides
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* done = bars + 2 * S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 1);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            mbar_init(&full[s], kAtbProducers);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * P.rows_per_cta;
    const uint64_t r1 = min(P.n, r0 + P.rows_per_cta);
    const uint32_t ntiles = r1 > r0 ? static_cast<uint32_t>((r1 - r0 + kAtbKT - 1) / kAtbKT) : 0u;

    if (warp == 0) {  // the MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tf32_idesc_mn(128, Np);
            for (uint32_t t = 0; t < ntiles; ++t) {
                const uint32_t s = t % S, ph = (t / S) & 1;
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = smem_addr(smem + s * stage_bytes);
                const uint32_t a_hi = st, a_lo = st + MT * kAtile, b_hi = st + 2 * MT * kAtile, b_lo = b_hi + bbytes;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const uint32_t d = tmem + mt * Np;
#pragma unroll
                    for (int g = 0; g < kAtbKT / 8; ++g) {  // K = 8 per MMA: two 4-row K groups
                        const uint32_t acc0 = (t | g) ? 1u : 0u;
                        const uint64_t ah = sw128_mn_desc(a_hi + mt * kAtile + 2 * g * sbo_a, sbo_a);
                        const uint64_t al = sw128_mn_desc(a_lo + mt * kAtile + 2 * g * sbo_a, sbo_a);
                        const uint64_t bh = sw128_mn_desc(b_hi + 2 * g * sbo_b, sbo_b);
                        const uint64_t bl = sw128_mn_desc(b_lo + 2 * g * sbo_b, sbo_b);
                        mma_tf32(d, ah, bh, idesc, acc0);
                        mma_tf32(d, ah, bl, idesc, 1u);
                        mma_tf32(d, al, bh, idesc, 1u);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(done);
        }
    } else if (warp >= 2) {  // producers: gather + split + swizzled store
        const uint32_t pw = warp - 2;
        constexpr int RPW = kAtbKT / kAtbProducers;  // rows per producer warp per K tile
        // register ring of DEPTH K tiles in flight per producer warp (a
        // runtime ring index would put it in local memory, so the loop below
        // is unrolled by DEPTH); the gathered rows' ids are loaded one tile
        // ahead of the rows, so no id -> row round trip is exposed
        constexpr int DEPTH = MT <= 2 ? 4 : 2;
        const uint32_t nq = Np / 4;  // float4 per B row (padded)
        float4 ra[DEPTH][RPW][MT], rb[DEPTH][RPW][2];
        uint64_t nid[RPW];  // Y row ids of the next tile to load
        auto load_ids = [&](uint32_t t) {
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const uint64_t r = r0 + static_cast<uint64_t>(t) * kAtbKT + pw * RPW + i;
                nid[i] = r < r1 ? (P.a_rows ? __ldg(P.a_rows + r) : r) : 0;
            }
        };
        auto load = [&](uint32_t t, auto bufc) {
            constexpr int buf = decltype(bufc)::value;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const uint64_t r = r0 + static_cast<uint64_t>(t) * kAtbKT + pw * RPW + i;
                const bool ok = r < r1;
                const uint64_t ar = nid[i];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const uint32_t col = mt * 128 + lane * 4;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ok && col < P.in_dim) {
                        const float* p = P.a + ar * P.lda + col;
                        if (col + 3 < P.in_dim) v = ldg4(p);
                        else {
                            v.x = __ldg(p);
                            if (col + 1 < P.in_dim) v.y = __ldg(p + 1);
                            if (col + 2 < P.in_dim) v.z = __ldg(p + 2);
                        }
                    }
                    ra[buf][i][mt] = v;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t q = lane + 32 * h;
                    const uint32_t col = q * 4;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ok && q < nq && col < P.out_dim) {
                        const float* p = P.b + r * P.ldb + col;
                        if (col + 3 < P.out_dim) v = ldg4(p);
                        else {
                            v.x = __ldg(p);
                            if (col + 1 < P.out_dim) v.y = __ldg(p + 1);
                            if (col + 2 < P.out_dim) v.z = __ldg(p + 2);
                        }
                    }
                    rb[buf][i][h] = v;
                }
            }
        };
        auto put = [&](uint32_t hi_addr, uint32_t lo_addr, float4 v) {
            const uint32_t h0 = tf32_hi(__float_as_uint(v.x)), h1 = tf32_hi(__float_as_uint(v.y));
            const uint32_t h2 = tf32_hi(__float_as_uint(v.z)), h3 = tf32_hi(__float_as_uint(v.w));
            const uint32_t l0 = __float_as_uint(__fsub_rn(v.x, __uint_as_float(h0)));
            const uint32_t l1 = __float_as_uint(__fsub_rn(v.y, __uint_as_float(h1)));
            const uint32_t l2 = __float_as_uint(__fsub_rn(v.z, __uint_as_float(h2)));
            const uint32_t l3 = __float_as_uint(__fsub_rn(v.w, __uint_as_float(h3)));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(hi_addr), "r"(h0), "r"(h1), "r"(h2), "r"(h3)
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(lo_addr), "r"(l0), "r"(l1), "r"(l2), "r"(l3)
                         : "memory");
        };
        auto step = [&](uint32_t t, auto bufc) {
            constexpr int cb = decltype(bufc)::value;
            if (t + DEPTH - 1 < ntiles) {  // keep DEPTH - 1 tiles in flight beyond this one
                load(t + DEPTH - 1, std::integral_constant<int, (cb + DEPTH - 1) % DEPTH>{});
                load_ids(t + DEPTH);
            }
            const uint32_t s = t % S, ph = (t / S) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            const uint32_t st = smem_addr(smem + s * stage_bytes);
            const uint32_t a_hi = st, a_lo = st + MT * kAtile, b_hi = st + 2 * MT * kAtile, b_lo = b_hi + bbytes;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                // float4 q of a row (MN elements 4q..4q+3): atom q / 8, 32-byte
                // granule ((q % 8) / 2) ^ (k % 4), half q % 2
                const uint32_t k = pw * RPW + i, g = k >> 2, kr = k & 3;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const uint32_t off = mt * kAtile + g * sbo_a + (lane >> 3) * 512u + kr * 128u +
                                         ((((lane & 7u) >> 1) ^ kr) << 5) + ((lane & 1u) << 4);
                    put(a_hi + off, a_lo + off, ra[cb][i][mt]);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t q = lane + 32 * h;
                    if (q < nq) {
                        const uint32_t off = g * sbo_b + (q >> 3) * 512u + kr * 128u + ((((q & 7u) >> 1) ^ kr) << 5) +
                                             ((q & 1u) << 4);
                        put(b_hi + off, b_lo + off, rb[cb][i][h]);
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        };
        // prologue: tiles 0 .. DEPTH-2 in flight, the ids of tile DEPTH-1 loaded
        load_ids(0);
        if (0 < ntiles) load(0, std::integral_constant<int, 0>{});
        load_ids(1);
        if (DEPTH > 2) {
            if (1 < ntiles) load(1, std::integral_constant<int, 1 % DEPTH>{});
            load_ids(2);
        }
        if (DEPTH > 3) {
            if (2 < ntiles) load(2, std::integral_constant<int, 2 % DEPTH>{});
            load_ids(3);
        }
        for (uint32_t t = 0; t < ntiles; t += DEPTH) {
            step(t, std::integral_constant<int, 0>{});
            if (t + 1 < ntiles) step(t + 1, std::integral_constant<int, 1 % DEPTH>{});
            if (DEPTH > 2 && t + 2 < ntiles) step(t + 2, std::integral_constant<int, 2 % DEPTH>{});
            if (DEPTH > 3 && t + 3 < ntiles) step(t + 3, std::integral_constant<int, 3 % DEPTH>{});
        }
    }
    // epilogue: warps 0-3 read TMEM lane quarters (warp w: lanes 32w..) — the
    // MMA warp joins after issuing; warps 2-3 after producing
    if (warp < 4) {
        mbar_wait(done, 0);
        __syncwarp();  // warp 0's issuing lane rejoins: tcgen05.ld is .sync.aligned
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float* part = P.part + static_cast<uint64_t>(blockIdx.x) * P.in_dim * P.out_dim;
        for (int mt = 0; mt < MT; ++mt) {
            const uint32_t i = mt * 128 + warp * 32 + lane;
            for (uint32_t c = 0; c < Np; c += 32) {
                uint32_t v[32];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
                    "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
                    "%30, %31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                      "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                      "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(tmem + ((warp * 32) << 16) + mt * Np + c));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (i < P.in_dim) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (c + j < P.out_dim) part[static_cast<uint64_t>(i) * P.out_dim + c + j] = __uint_as_float(v[j]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// out[i][j] = sum over CTAs c (ascending) of part[c][i][j]
__global__ void k_atb_reduce(const float* __restrict__ part, uint32_t nparts, uint32_t in_dim, uint32_t out_dim,
                             float* __restrict__ out, uint64_t ldo) {
    const uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t tot = static_cast<uint64_t>(in_dim) * out_dim;
    if (e >= tot) return;
    float acc = 0.f;
    for (uint32_t c = 0; c < nparts; ++c) acc = __fadd_rn(acc, part[c * tot + e]);
    out[(e / out_dim) * ldo + e % out_dim] = __fadd_rn(acc, 0.f);
}

template <int MT>
void launch_atb(const AtbParams& p, size_t smem, unsigned grid, cudaStream_t s) {
    static std::vector<char> attr;
    static std::mutex mu;
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        if (static_cast<int>(attr.size()) <= dev) attr.resize(dev + 1, 0);
        if (!attr[dev]) {
            PG_CUDA(cudaFuncSetAttribute(k_gemm_atb_tc<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            attr[dev] = 1;
        }
    }
    k_gemm_atb_tc<MT><<<grid, kAtbThreads, smem, s>>>(p);
    PG_LAUNCH("k_gemm_atb_tc");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

template <int MT>
void launch_tc(const CUtensorMap& amap, const TcParams& p, size_t smem, unsigned grid, cudaStream_t s) {
    static std::vector<char> attr;  // per device
    static std::mutex mu;
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        if (static_cast<int>(attr.size()) <= dev) attr.resize(dev + 1, 0);
        if (!attr[dev]) {
            PG_CUDA(cudaFuncSetAttribute(k_gemm_abt_tc<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            attr[dev] = 1;
        }
    }
    k_gemm_abt_tc<MT><<<grid, kTcThreads, smem, s>>>(amap, p);
    PG_LAUNCH("k_gemm_abt_tc");
}

}  // namespace

bool gemm_a_bt_tc_supported(DMat a) {
    return encode_fn() != nullptr && a.ld % 4 == 0 && reinterpret_cast<uintptr_t>(a.p) % 16 == 0 && a.cols > 0 &&
           a.rows < (1ull << 31) && a.cols < (1ull << 31) && a.ld * 4 < (1ull << 40);
}

void gemm_a_bt_tc(DMat a, DMat b, DMat out, cudaStream_t s) {
    const uint64_t n = a.rows, K = a.cols, m = b.rows;
    if (b.cols != K) fail_shape("gemm_a_bt: column counts differ");
    if (out.rows != n || out.cols != m) fail_shape("gemm_a_bt: output shape mismatch");
    if (n == 0 || m == 0) return;
    if (!gemm_a_bt_tc_supported(a))
        fail(kConfig, "gemm_a_bt (tensor cores): A needs a 16-byte aligned base and ld % 4 == 0");
    // N tile: the whole output width when it fits one MMA (<= 256), else
    // balanced 8-multiples
    const uint32_t NT = static_cast<uint32_t>((m + kMaxN - 1) / kMaxN);
    const uint32_t N = static_cast<uint32_t>(((m + NT - 1) / NT + 7) / 8 * 8);
    const uint32_t KB = static_cast<uint32_t>((K + kKB - 1) / kKB);
    const uint32_t acc_stride = (N + 31) / 32 * 32;
    const int MT = acc_stride <= 128 ? 2 : 1;  // two 128-row sub-tiles share each B stage when N is narrow
    const size_t stage = 2ull * MT * kTileBytesA + 2ull * N * 128;
    const size_t budget = 232448 - 1024 - 256;
    const uint32_t S = static_cast<uint32_t>(std::min<size_t>(4, budget / stage));
    if (S < 2) fail(kConfig, "gemm_a_bt (tensor cores): tile does not fit shared memory");
    const size_t smem = 1024 + S * stage + (3 * S + 4) * 8 + 16;

    // the pre-split B image (hi, lo), one stage per (N tile, k block)
    DevBuf<float> img(static_cast<uint64_t>(NT) * KB * 2 * N * kKB, s);
    {
        const uint64_t total = static_cast<uint64_t>(NT) * KB * N * kKB;
        k_tc_pack_b<<<grid_for(total, 256), 256, 0, s>>>(b.p, b.ld, static_cast<uint32_t>(m), static_cast<uint32_t>(K),
                                                      N, NT, KB, img.get());
        PG_LAUNCH("k_tc_pack_b");
    }
    CUtensorMap amap;
    std::memset(&amap, 0, sizeof(amap));
    const cuuint64_t gdim[2] = {K, n};
    const cuuint64_t gstride[1] = {a.ld * 4};
    const cuuint32_t box[2] = {kKB, 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a.p, gdim, gstride, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(kDevice, "gemm_a_bt (tensor cores): cuTensorMapEncodeTiled failed");
    TcParams p{};
    p.out = out.p;
    p.ldo = out.ld;
    p.n = n;
    p.m = m;
    p.N = N;
    p.NT = NT;
    p.KB = KB;
    p.stages = S;
    p.acc_stride = acc_stride;
    p.row_tiles = (n + 128ull * MT - 1) / (128ull * MT);
    p.bimg = img.get();
    p.vec_out = (out.ld % 4 == 0 && reinterpret_cast<uintptr_t>(out.p) % 16 == 0) ? 1 : 0;
    int dev = 0, sms = 148;
    PG_CUDA(cudaGetDevice(&dev));
    (void)lib_stream(dev);  // the stream-ordered pool keeps freed temporaries (no re-map per call)
    PG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t tiles = p.row_tiles * NT;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sms)));
    if (MT == 2)
        launch_tc<2>(amap, p, smem, grid, s);
    else
        launch_tc<1>(amap, p, smem, grid, s);
}

bool gemm_at_b_tc_supported(uint64_t in_dim, uint64_t out_dim) {
    // any shape: blocks of <= 640 x 256 outputs per launch (gemm_at_b_tc)
    return in_dim > 0 && out_dim > 0 && in_dim < (1ull << 31) && out_dim < (1ull << 31);
}

// one launch over output block [i0, i0 + bi) x [j0, j0 + bj) (bi <= 640,
// MT x Npad <= 512 TMEM columns): sub-views of the same pitched matrices
void gemm_at_b_tc_block(DMat a, const uint32_t* a_rows, DMat b, DMat out, uint64_t i0, uint64_t bi, uint64_t j0,
                        uint64_t bj, int sms, cudaStream_t s) {
    const uint64_t n = b.rows;
    const uint32_t Np = static_cast<uint32_t>((bj + 31) / 32 * 32);
    const int MT = static_cast<int>((bi + 127) / 128);
    const size_t stage = 2ull * MT * 128 * kAtbKT * 4 + 2ull * Np * kAtbKT * 4;
    const size_t budget = 232448 - 1024 - 256;
    const uint32_t S = static_cast<uint32_t>(std::min<size_t>(6, budget / stage));
    if (S < 2) fail(kConfig, "gemm_at_b (tensor cores): tile does not fit shared memory");
    const size_t smem = 1024 + S * stage + (2 * S + 2) * 8 + 16;
    const uint64_t tiles = (n + kAtbKT - 1) / kAtbKT;
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sms)));
    const uint64_t per = (tiles + grid - 1) / grid * kAtbKT;
    const uint32_t nparts = static_cast<uint32_t>((n + per - 1) / per);
    DevBuf<float> part(static_cast<uint64_t>(nparts) * bi * bj, s);
    AtbParams p{};
    p.a = a.p + i0;
    p.lda = a.ld;
    p.a_rows = a_rows;
    p.b = b.p + j0;
    p.ldb = b.ld;
    p.n = n;
    p.in_dim = static_cast<uint32_t>(bi);
    p.out_dim = static_cast<uint32_t>(bj);
    p.Npad = Np;
    p.stages = S;
    p.rows_per_cta = per;
    p.part = part.get();
    switch (MT) {
        case 1: launch_atb<1>(p, smem, nparts, s); break;
        case 2: launch_atb<2>(p, smem, nparts, s); break;
        case 3: launch_atb<3>(p, smem, nparts, s); break;
        case 4: launch_atb<4>(p, smem, nparts, s); break;
        default: launch_atb<5>(p, smem, nparts, s); break;
    }
    const uint64_t tot = bi * bj;
    k_atb_reduce<<<grid_for(tot, 256), 256, 0, s>>>(part.get(), nparts, p.in_dim, p.out_dim, out.p + i0 * out.ld + j0,
                                                 out.ld);
    PG_LAUNCH("k_atb_reduce");
}

void gemm_at_b_tc(DMat a, const uint32_t* a_rows, DMat b, DMat out, cudaStream_t s) {
    const uint64_t n = b.rows, in_dim = a.cols, out_dim = b.cols;
    if (!a_rows && a.rows != n) fail_shape("gemm_at_b: row counts differ");
    if (out.rows != in_dim || out.cols != out_dim) fail_shape("gemm_at_b: output shape mismatch");
    if (in_dim == 0 || out_dim == 0) return;
    if (a.ld % 4 || b.ld % 4 || reinterpret_cast<uintptr_t>(a.p) % 16 || reinterpret_cast<uintptr_t>(b.p) % 16)
        fail(kConfig, "gemm_at_b (tensor cores): Y and g need 16-byte aligned rows (ld % 4 == 0)");
    if (n == 0) {
        PG_CUDA(cudaMemset2DAsync(out.p, out.ld * 4, 0, out_dim * 4, in_dim, s));
        return;
    }
    int dev = 0, sms = 148;
    PG_CUDA(cudaGetDevice(&dev));
    (void)lib_stream(dev);  // the stream-ordered pool keeps freed temporaries (no re-map per call)
    PG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // output blocks: up to 5 M tiles (640 rows) x as many 32-column groups as
    // the 512 TMEM columns allow (<= 256)
    for (uint64_t i0 = 0; i0 < in_dim; i0 += 640) {
        const uint64_t bi = std::min<uint64_t>(640, in_dim - i0);
        const uint64_t MT = (bi + 127) / 128;
        const uint64_t nmax = std::min<uint64_t>(256, 512 / MT / 32 * 32);
        for (uint64_t j0 = 0; j0 < out_dim; j0 += nmax)
            gemm_at_b_tc_block(a, a_rows, b, out, i0, bi, j0, std::min<uint64_t>(nmax, out_dim - j0), sms, s);
    }
}

}  // namespace pg
