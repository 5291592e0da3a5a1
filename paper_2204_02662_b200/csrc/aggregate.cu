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
#include <deque>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "pg_internal.h"

namespace pg {

// Scheduling knobs (pg_set_tuning / $PG_<KEY>); none changes a result bit.
namespace {
struct TuneKey {
    const char* name;
    const char* env;
    int64_t def;
};
// order = enum TuneKeyId (pg_internal.h)
constexpr TuneKey kTuneKeys[] = {
    {"heavy_tma", "PG_HEAVY_TMA", 0},      // heavy narrow rows: 1 = TMA bulk-copy mbarrier ring (k_agg_heavy)
    {"vec_u", "PG_VEC_U", 0},              // edges per gather batch in k_agg_vec4 (4, 8, 16; 0 = by average degree)
    {"chunk_major", "PG_CHUNK_MAJOR", 1},  // k_agg_vec4 item order for multi-chunk rows
    {"host_segs", "PG_HOST_SEGS", 3},      // host drop-in: source-row segments (H2D overlap)
    {"host_chunks", "PG_HOST_CHUNKS", 8},  // host drop-in: row chunks of the last pass (D2H overlap)
    {"host_trace", "PG_HOST_TRACE", 0},    // host drop-in: print phase times to stderr
    {"heavy_narrow", "PG_HEAVY_NARROW", 0},  // heavy rows <= 64 floats: 1 = k_agg_narrow_lat, 0 = coop tiles
    {"wide_lpd", "PG_WIDE_LPD", 32},       // wide rows: lanes per (destination, chunk) item, 32 or 16
    {"src_segs", "PG_SRC_SEGS", 0},        // whole-path SpMM source segments: 0 = auto (L2-sized), K = forced
    {"ld_cg", "PG_LD_CG", 0},              // row gathers: 0/1 nc, 2 cg, 3 nc.L1::no_allocate, 4 plain, 5 nc.L1::evict_last, 6 records no_allocate, 7 records L2 evict_first, 9 rows L2 evict_last
    {"host_chunk_order", "PG_HOST_CHUNK_ORDER", 1},  // host drop-in last pass: 1 = last row chunk first
    {"grouped_seg", "PG_GROUPED_SEG", 0},  // grouped Fast: 0 = atomic-free k_agg_grp, 1 = CTA-segmented + atomics at CTA edges, 2 = an atomic per extra group
    // heavy wide rows: software-pipelined k_agg_wide_pipe with hub items
    // destination-major (1) or chunk-major (2); 3 = whole-row TMA ring
    // (k_agg_hub_ring: measured slower, its ~80 KB ring holds only 32 rows in
    // flight per hub, profiles/e2e_hub_ring_sweep_r02.log); 4 = cooperative
    // 64-row tiles (k_agg_heavy_coop<32>: slower still, 64 KB + 256 threads
    // per hub chunk, profiles/e2e_hub_coop_sweep_r02.log); 5 = float2 lanes,
    // 64 rows in flight per chain (k_agg_wide_pipe2: e2e 23.2-23.5 vs 23.0-23.2
    // ms, profiles/hub_pipe2_sweep_r02.log); 0 = k_agg_wide_lat
    {"heavy_wide_pipe", "PG_HEAVY_WIDE_PIPE", 1},
    {"host_final_segs", "PG_HOST_FINAL_SEGS", 1},  // host drop-in: trailing source segments of the chunked last pass
    {"host_pitch2d", "PG_HOST_PITCH2D", 0},  // host drop-in: odd widths by 2-D DMA (1) or flat DMA + repack kernel (0)
    {"host_copy_prio", "PG_HOST_COPY_PRIO", 1},  // host drop-in: copy/repack streams at the highest priority (read once)
    {"host_seg_balance", "PG_HOST_SEG_BALANCE", 1},  // host drop-in: source segments of equal rows (0) or equal edges (1)
    {"host_chunk_balance", "PG_HOST_CHUNK_BALANCE", 30},  // host drop-in: last-pass chunk cuts, % weight of edges vs rows
    {"atb_split", "PG_ATB_SPLIT", 1},  // W' GEMM: 1 = copy warp + chain warp, 0 = one warp does both
    {"atb_pairs", "PG_ATB_PAIRS", 224},  // W' split GEMM: 2 A columns per lane above this many 64-chain blocks (0 = never)
    {"gemm_packed", "PG_GEMM_PACKED", 2},  // gemm / gemm_a_bt: 2 = k_gemm3 register tiles (m > 64), 1 = k_gemm2 FFMA2 column pairs, 0 = k_gemm
    {"host_last_seg_pct", "PG_HOST_LAST_SEG_PCT", 45},  // host drop-in: % of the edges in the last (chunked) segment, 0 = 1/K
    {"wgrad_fork", "PG_WGRAD_FORK", 1},  // backward chains: W' GEMMs on a forked stream (1) or in order (0)
    // chain y_grad = g W^T (gemm_a_bt): 0 = bit-exact FFMA2 kernel, 1 = tcgen05
    // 3xTF32 tensor-core kernel (fp32 tolerance, not bit-exact)
    {"gemm_tc", "PG_GEMM_TC", 0},
    // k_agg_vec4 wide rows: 1 = coalesced record window + shuffles, 2 = the
    // window handed out by REDUX into uniform registers, 0 = a broadcast
    // record load per edge (measured fastest on the Reddit layer-0 path:
    // 15.65 vs 15.92 (1) / 15.93 (2) ms, so off)
    {"rec_window", "PG_REC_WINDOW", 0},
    // whole-path L2-sized source segments: cuts by rows (0) .. by edges (100)
    {"src_seg_balance", "PG_SRC_SEG_BALANCE", 0},
    // host drop-in: output size (MB) from which the copy/compute pipeline is used
    {"host_min_mb", "PG_HOST_MIN_MB", 32},
    // rows of 129..768 floats: 1 = whole-row warps (k_agg_row), 0 = 128-column
    // chunk items (k_agg_vec4)
    {"row_kernel", "PG_ROW_KERNEL", 0},
    {"row_u", "PG_ROW_U", 2},            // k_agg_row: edges per gather batch (2, 3, 4)
    {"row_seg_mb", "PG_ROW_SEG_MB", 56},  // k_agg_row: per-pass source working set (MB) of the L2-sized segments
    {"row_heavy", "PG_ROW_HEAVY", 0},    // k_agg_row: hub degree threshold (0 = the default rule)
    {"vec_block", "PG_VEC_BLOCK", 256},  // k_agg_vec4 wide rows: threads per CTA (256, 512, 1024)
    // wide-row hubs: 1 = destination-major front of the main kernel (every
    // hub chunk starts with the pass, no concurrent side kernel; Reddit
    // layer 0 16.5 -> 15.8 ms), 0 = k_agg_wide_pipe on a forked stream
    {"hub_inline", "PG_HUB_INLINE", 1},
    {"hub_front_min", "PG_HUB_FRONT_MIN", 0},  // hub_inline: degree threshold of the front (0 = the hub rule)
    {"gemm3_rows", "PG_GEMM3_ROWS", 8},  // k_gemm3 (gemm_packed 2): output rows per thread, 8 or 16
    {"gemm_beside_wgrad", "PG_GEMM_BESIDE_WGRAD", 1},  // backward chains: y_grad on k_gemm2 while a W' fork runs
    // host drop-in last pass: 1 = the hub rows (degree >= host_hub_min) of
    // every chunk first on their own stream, 2 = the whole hub chunk on its
    // own stream, 0 = off. Measured (profiles/e2e_hub_split_sweep_r02.log):
    // 27.2 / 25.7 vs 23.2 ms — latency-bound hub chains run 2.5x slower
    // beside the other chunks than alone, so the split costs more than the
    // 0.9 ms of D2H idle it was to remove
    {"host_hub_chunk_side", "PG_HOST_HUB_CHUNK_SIDE", 0},
    // k_agg_vec4 wide rows: > 0 = source-window lockstep CTAs (k_agg_vec4w),
    // the value = edges per warp per window
    {"vec_window", "PG_VEC_WINDOW", 0},
    {"host_hub_min", "PG_HOST_HUB_MIN", 16384},  // host_hub_chunk_side 1: degree of the hub rows split off
    {"grouped_src_segs", "PG_GROUPED_SRC_SEGS", 1},  // grouped Fast (k_agg_grp): L2-sized source segments for wide rows
    {"narrow_u", "PG_NARROW_U", 8},  // rows <= 16 floats: edges per gather batch of a 4-lane destination (8, 16)
    // W' split GEMM copy warp: 0 = a row per lane, 4 slots / 2 in flight;
    // 1 = the same 7 / 5; 2 = lanes sharing rows (fewer L1 wavefronts)
    {"atb_depth", "PG_ATB_DEPTH", 0},
    {"host_first_chunk_pct", "PG_HOST_FIRST_CHUNK_PCT", 100},  // host drop-in: size of the first-computed chunk, % of the others
    // host drop-in: the last pass as ONE launch whose items count per row
    // chunk, each chunk's D2H waiting on its counter (cuStreamWaitValue32):
    // the pass itself runs 9.8 vs 11.7 ms, but the hub front's chains hold
    // warp slots and the later chunks finish late (e2e 23.3-24.0 vs 22.8 ms,
    // profiles/e2e_seq_sweep_r02.log), so off
    {"host_seq", "PG_HOST_SEQ", 0},
    // W': 1 / 2 = 4 chain + 4 copy warps per block, one chain warp per SMSP
    // (6 / 10 ring slots). Alone it is faster (products 10.6 -> 7.7 ms), but
    // holding whole SMs it slows the forked chains it overlaps (products
    // backward_epp 17.0 -> 28.6 ms, profiles/atb_quad_sweep_r02.log); 3
    // (default) = only for W' over whole matrices (no row gather: the
    // all-active / if-else / Global EPP chains, products 47 -> 39 ms)
    {"atb_quad", "PG_ATB_QUAD", 3},
    // host drop-in below host_min_mb: D2H-overlap chunks (0/1 = off; the
    // Reddit top path split in 2 computes 0.94 vs 0.62 ms, so no gain:
    // profiles/e2e_small_chunks_sweep_r02.log)
    {"host_small_chunks", "PG_HOST_SMALL_CHUNKS", 0},
    // wide rows: 256-bit row gathers, two 128-column items per warp
    // (k_agg_vec8): 1 on, 0 off, 2 auto (rows wider than 64 columns, from
    // 2^21 edges per call)
    {"vec8", "PG_VEC8", 2},
    // aggregate_pull<double>: hub-kernel degree threshold (0 = by the call's bytes)
    {"f64_hub_min", "PG_F64_HUB_MIN", 0},
    // grouped Fast (k_agg_grp): 1 = groups handed to workers dynamically
    {"grp_dynamic", "PG_GRP_DYNAMIC", 0},
    // k_agg_vec8 wide rows: edges per batch per half-warp (0 = 4; 3, 6)
    {"vec8_u", "PG_VEC8_U", 0},
    // row-range calls (host pipeline chunks, shards): 1 = hubs on the side kernel, 0 = inline front
    {"range_side_hubs", "PG_RANGE_SIDE_HUBS", 1},
};
static_assert(sizeof(kTuneKeys) / sizeof(kTuneKeys[0]) == kTuneRangeSideHubs + 1,
              "kTuneKeys and enum TuneKeyId (pg_internal.h) must list the same keys in the same order");
std::atomic<int64_t> g_tune[sizeof(kTuneKeys) / sizeof(kTuneKeys[0])];
int64_t g_tune_def[sizeof(kTuneKeys) / sizeof(kTuneKeys[0])];  // $PG_<KEY> at load, else built-in
std::once_flag g_tune_once;
void tune_init() {
    for (size_t i = 0; i < sizeof(kTuneKeys) / sizeof(kTuneKeys[0]); ++i) {
        const char* e = std::getenv(kTuneKeys[i].env);
        g_tune_def[i] = e ? std::atoll(e) : kTuneKeys[i].def;
        g_tune[i].store(g_tune_def[i]);
    }
}
}  // namespace

bool row_kernel_on(uint64_t dim) {
    const uint64_t nq = (dim + 3) / 4;
    return nq > 32 && nq <= 192 && tuning(kTuneRowKernel) != 0;
}

int64_t tuning(int key) {
    std::call_once(g_tune_once, tune_init);
    return g_tune[key].load(std::memory_order_relaxed);
}

bool set_tuning(const char* name, int64_t value) {
    std::call_once(g_tune_once, tune_init);
    for (size_t i = 0; i < sizeof(kTuneKeys) / sizeof(kTuneKeys[0]); ++i)
        if (std::strcmp(kTuneKeys[i].name, name) == 0) {
            g_tune[i].store(value < 0 ? g_tune_def[i] : value);
            return true;
        }
    return false;
}

namespace {

__device__ __forceinline__ float4 ldg4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// float4 accumulator held as two packed fp32 pairs for Blackwell's FFMA2 /
// FADD2, with the reference's separately rounded multiply and add:
//   p = fma.rn.f32x2(w, x, nz) with nz = -0.0 passed at RUN time, which is
//       exactly round(w*x) (w*x + -0 == w*x for every w*x, signed zeros
//       included);
//   acc = add.rn.f32x2(acc, p).
// A compile-time -0 (or plain mul.rn.f32x2 + add.rn.f32x2) lets ptxas fold
// the pair into one FFMA2 that rounds once — not the reference's result.
// Half the FP instructions of scalar FMUL+FADD; bit-identical.
struct Acc {
    unsigned long long lo, hi;
};
struct Zs {
    unsigned long long nz, pz;  // (-0,-0) and (+0,+0), from a kernel argument
};
const float2 kZeros = make_float2(-0.0f, 0.0f);  // host side: the kernel argument

__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 unpk2(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ Zs zs_of(float2 z) { return {pk2(z.x, z.x), pk2(z.y, z.y)}; }

__device__ __forceinline__ void acc_step(Acc& a, float w, const float4& x, const Zs& z) {
    const unsigned long long ww = pk2(w, w);
    unsigned long long p0, p1;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p0) : "l"(ww), "l"(pk2(x.x, x.y)), "l"(z.nz));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p1) : "l"(ww), "l"(pk2(x.z, x.w)), "l"(z.nz));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a.lo) : "l"(a.lo), "l"(p0));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a.hi) : "l"(a.hi), "l"(p1));
}

// zero, or the current output (accumulate semantics, aggregate.hpp:50-55)
__device__ __forceinline__ Acc acc_load(const float* orow, uint32_t col, uint32_t dim, bool doit) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (doit && col < dim) {
        if (col + 3 < dim) v = *reinterpret_cast<const float4*>(orow);
        else {
            v.x = orow[0];
            if (col + 1 < dim) v.y = orow[1];
            if (col + 2 < dim) v.z = orow[2];
        }
    }
    return {pk2(v.x, v.y), pk2(v.z, v.w)};
}

// acc + 0 (-0 -> +0, aggregate.hpp:82), then a streaming store of the
// columns inside dim
__device__ __forceinline__ void acc_store(float* orow, uint32_t col, uint32_t dim, Acc a, const Zs& z) {
    if (col >= dim) return;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a.lo) : "l"(a.lo), "l"(z.pz));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a.hi) : "l"(a.hi), "l"(z.pz));
    const float2 l = unpk2(a.lo), h = unpk2(a.hi);
    if (col + 3 < dim) {
        __stcs(reinterpret_cast<float4*>(orow), make_float4(l.x, l.y, h.x, h.y));
    } else {
        orow[0] = l.x;
        if (col + 1 < dim) orow[1] = l.y;
        if (col + 2 < dim) orow[2] = h.x;
    }
}

// 128-bit read-only row gather at base + src * ld_bytes: one IMAD.WIDE.U32
// per edge (the 32x32->64 multiply-add cannot overflow for ld_bytes < 2^32).
// LDM (tuning "ld_cg") selects the load flavour of the row gathers:
//   0/1 ld.global.nc (read-only path, L1 allocating; default)
//   2   ld.global.cg (L2 only)
//   3   ld.global.nc.L1::no_allocate
//   4   ld.global (plain)
//   5   ld.global.nc.L1::evict_last
// (the records, streamed once, use L1::no_allocate when LDM == 6 and an
// L2 evict_first policy when LDM == 7; rows nc)
template <int LDM = 0>
__device__ __forceinline__ float4 ld_row(const char* base, uint32_t src, uint32_t ld_bytes) {
    float4 r;
    const char* p = base + static_cast<uint64_t>(src) * ld_bytes;
    if constexpr (LDM == 2)
        asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    else if constexpr (LDM == 3)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p));
    else if constexpr (LDM == 4)
        asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    else if constexpr (LDM == 5)
        asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p));
    else if constexpr (LDM == 9) {  // rows kept in L2 ahead of the streamed records / outputs
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p), "l"(pol));
    }
    else
        asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
template <int LDM = 0>
__device__ __forceinline__ Edge ld_rec_m(const Edge* p) {
    Edge r;
    if constexpr (LDM == 6)
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    else if constexpr (LDM == 7) {
        // streamed once per pass: first out of L2, so the gathered rows stay
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
    } else
        asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ Edge ld_rec(const Edge* p) {
    Edge r;
    asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

// A runtime-zero value that depends on all U gathered rows. Folded into the
// -0 addend of every multiply (bit-neutral: zmask is 0 at run time), it makes
// every FP op of the batch wait for the whole batch, so ptxas has to issue
// all U row gathers back to back (without it, it interleaves load/use pairs
// and a warp keeps one or two gathers in flight).
template <int U>
__device__ __forceinline__ Zs batch_dep(const float4 (&x)[U], const Zs& z, uint32_t zmask) {
    uint32_t all = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) all ^= __float_as_uint(x[u].x);
    all &= zmask;
    Zs r = z;
    r.nz ^= (static_cast<unsigned long long>(all) << 32) | all;
    return r;
}

// ---- AggExt helpers (engine chains) ----
__device__ __forceinline__ uint32_t ext_out_row(const AggExt& x, uint32_t d) {
    return x.out_rows ? __ldg(x.out_rows + d) : d;
}
// relu_backward on a finished row slice (dense_matrix.hpp:107-113):
// pre > 0 ? v : +0, element by element for the columns inside dim
__device__ __forceinline__ float4 ext_relu(const AggExt& x, uint32_t d, uint32_t row, uint32_t col, uint32_t dim,
                                           float4 v) {
    if (!x.relu_pre) return v;
    const uint32_t prow = x.pre_rows ? __ldg(x.pre_rows + d) : row;
    const float* pr = x.relu_pre + static_cast<uint64_t>(prow) * x.ld_pre + col;
    v.x = pr[0] > 0.f ? v.x : 0.f;
    if (col + 1 < dim) v.y = pr[1] > 0.f ? v.y : 0.f;
    if (col + 2 < dim) v.z = pr[2] > 0.f ? v.z : 0.f;
    if (col + 3 < dim) v.w = pr[3] > 0.f ? v.w : 0.f;
    return v;
}
__device__ __forceinline__ bool ext_dst_on(const AggExt& x, uint32_t d) {
    return !x.dst_bits || ((__ldg(x.dst_bits + (d >> 5)) >> (d & 31)) & 1u);
}
__device__ __forceinline__ bool ext_src_on(const AggExt& x, uint32_t u) {
    return (__ldg(x.src_bits + (u >> 5)) >> (u & 31)) & 1u;
}
// acc + 0, relu epilogue, store of the columns inside dim
__device__ __forceinline__ void acc_store_ext(float* orow, uint32_t col, uint32_t dim, Acc a, const Zs& z,
                                              const AggExt& x, uint32_t d, uint32_t row) {
    if (col >= dim) return;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a.lo) : "l"(a.lo), "l"(z.pz));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a.hi) : "l"(a.hi), "l"(z.pz));
    const float2 l = unpk2(a.lo), h = unpk2(a.hi);
    float4 v = ext_relu(x, d, row, col, dim, make_float4(l.x, l.y, h.x, h.y));
    if (col + 3 < dim) {
        __stcs(reinterpret_cast<float4*>(orow), v);
    } else {
        orow[0] = v.x;
        if (col + 1 < dim) orow[1] = v.y;
        if (col + 2 < dim) orow[2] = v.z;
    }
}

// LPD lanes per (destination, chunk); each lane one float4 column. Per batch
// of U edges: U edge-record loads, U row gathers (all in flight), then the
// U ordered accumulate steps. Lanes past dim gather their chunk's first
// float4 (in bounds, the sector lane 0 reads anyway; discarded) so no load
// is predicated and no extra sector is fetched.
template <int LPD, int U, bool FILT, int CG = 0, bool RW = false, int BS = 256>
__global__ void __launch_bounds__(BS, (BS == 256 ? (U <= 8 ? 4 : 2) : 1024 / BS)) k_agg_vec4(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                 const Edge* __restrict__ edges,
                                                 const uint32_t* __restrict__ order, uint32_t d_begin,
                                                 uint64_t n_items, uint32_t chunks,
                                                 const float* __restrict__ in, uint32_t ld_in_bytes,
                                                 float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                 int accumulate, float2 zeros, uint32_t zmask,
                                                 int chunk_major, AggExt ext) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    if (item >= n_items) return;
    const Zs z = zs_of(zeros);
    // destination-major (the chunks of one destination on neighbouring warps)
    // or chunk-major (one column chunk of every destination, then the next:
    // the per-pass source working set is S x chunk bytes)
    // chunk_major >= 2: the first chunk_major - 2 destinations (the hubs at
    // the head of the degree order) go destination-major ahead of the
    // chunk-major rest, so every hub chunk starts at the beginning of the pass
    const uint64_t nd = n_items / chunks;
    const uint64_t nf = chunk_major > 1 ? static_cast<uint64_t>(chunk_major - 2) : 0;
    uint32_t di, ci;
    if (!chunk_major || item < nf * chunks) {
        di = static_cast<uint32_t>(item / chunks);
        ci = static_cast<uint32_t>(item % chunks);
    } else {
        const uint64_t r = item - nf * chunks, nr = nd - nf;
        di = static_cast<uint32_t>(nf + r % nr);
        ci = static_cast<uint32_t>(r / nr);
    }
    const uint32_t d = __ldg(order + d_begin + di);
    if (FILT && !ext_dst_on(ext, d)) return;
    const uint32_t q = ci * LPD + static_cast<uint32_t>(t % LPD);
    const uint32_t col = q * 4;
    const bool active = col < dim;
    uint64_t e = __ldg(ebeg + d);
    const uint64_t end = __ldg(eend + d);
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * LPD * 4u) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));  // per-lane 64-bit base: IMAD.WIDE adds it
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
    Acc acc = acc_load(orow, col, dim, accumulate);
    // Narrow rows (LPD <= 8 lanes per destination): the U records of a batch
    // are loaded spread over the sub-warp's lanes (one 32-byte segment per
    // sub-warp and instruction instead of U single-record loads, each a
    // separate L1 wavefront per sub-warp) and handed out by sub-warp shuffles.
    constexpr int NPL = (U + LPD - 1) / LPD;
    const unsigned sl = static_cast<unsigned>(t % LPD);
    const unsigned submask = LPD >= 32 ? 0xffffffffu : (((1u << LPD) - 1u) << (lane_id() & ~(LPD - 1u)));
    // Wide rows (RW, LPD >= 16): a record WINDOW — LPD consecutive records,
    // one per lane, loaded coalesced one window ahead (a 256-byte request per
    // 32 edges instead of one broadcast record load per edge) and handed out
    // by shuffles: the L1 sees one request per gathered row.
    constexpr bool kWin = RW && LPD >= 16 && (LPD % U == 0);
    uint64_t wbase = e;
    Edge win = make_uint2(0u, 0u), nwin = make_uint2(0u, 0u);
    if constexpr (kWin) {
        if (e + sl < end) win = ld_rec(edges + e + sl);
        if (e + LPD + sl < end) nwin = ld_rec(edges + e + LPD + sl);
    }
    auto batch_recs = [&](Edge (&ed)[U], uint32_t n) {
        if constexpr (kWin) {
            (void)n;  // records past the destination's end are zero records (row 0, discarded)
            if (e - wbase == static_cast<uint64_t>(LPD)) {  // window consumed: slide
                wbase += LPD;
                win = nwin;
                nwin = wbase + LPD + sl < end ? ld_rec(edges + wbase + LPD + sl) : make_uint2(0u, 0u);
            }
            const unsigned off = static_cast<unsigned>(e - wbase);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if constexpr (CG == 8 && LPD == 32) {
                    // REDUX lands the record in a uniform register: no
                    // per-lane register write on the L1 -> RF path
                    const bool me = sl == off + u;
                    ed[u].x = __reduce_or_sync(0xffffffffu, me ? win.x : 0u);
                    ed[u].y = __reduce_or_sync(0xffffffffu, me ? win.y : 0u);
                } else {
                    ed[u].x = __shfl_sync(submask, win.x, off + u, LPD);
                    ed[u].y = __shfl_sync(submask, win.y, off + u, LPD);
                }
            }
        } else if constexpr (LPD <= 8) {
            Edge mine[NPL];
#pragma unroll
            for (int i = 0; i < NPL; ++i) {
                const unsigned k = sl + i * LPD;
                mine[i] = ld_rec_m<CG>(edges + e + (k < n ? k : n - 1));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ed[u].x = __shfl_sync(submask, mine[u / LPD].x, u % LPD, LPD);
                ed[u].y = __shfl_sync(submask, mine[u / LPD].y, u % LPD, LPD);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec_m<CG>(edges + e + (u < static_cast<int>(n) ? u : n - 1));
        }
    };
    for (; e + U <= end; e += U) {
        Edge ed[U];
        batch_recs(ed, U);
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (FILT && !ext_src_on(ext, ed[u].x)) x[u] = make_float4(0.f, 0.f, 0.f, 0.f);  // skipped: +-0 term
            else x[u] = ld_row<(CG >= 6 && CG <= 8 ? 0 : CG)>(base, ed[u].x, ld_in_bytes);
        }
        const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
    }
    if (e < end) {  // remainder (< U edges) as one batch: all gathers in flight
        const uint32_t n = static_cast<uint32_t>(end - e);
        Edge ed[U];
        batch_recs(ed, n);
        float4 x[U];
        // slots past the list are not gathered (predicated off): for short
        // lists the remainder is the whole item, and duplicate gathers of the
        // last row cost L1 requests and register writeback
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if ((FILT && !ext_src_on(ext, ed[u].x)) || u >= static_cast<int>(n)) x[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            else x[u] = ld_row<(CG >= 6 && CG <= 8 ? 0 : CG)>(base, ed[u].x, ld_in_bytes);
        }
        const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(n)) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
    }
    acc_store_ext(orow, col, dim, acc, z, ext, d, row);
}

// 256-bit row gathers (tuning "vec8"): sm_100 has LDG.E.ENL2.256, one
// 32-byte load per lane. LPD lanes of 8 floats own a (destination, chunk):
// LPD = 16 covers a 128-column chunk, so a warp carries TWO items of
// k_agg_vec4<32>'s — the same items, chunk order and per-column fp32
// chains, with half the load instructions per gathered byte and one record
// load (two addresses) per edge pair instead of one broadcast per edge;
// LPD = 2 / 4 / 8 are k_agg_vec4<4 / 8 / 16>'s narrow rows (widths <= 16 /
// 32 / 64) with the batch's records spread over the sub-warp and shuffled.
// Needs a 32-byte aligned input and an 8-float row pitch.
__device__ __forceinline__ void ld_row8(const char* base, uint32_t src, uint32_t ld_bytes, float4& a, float4& b) {
    const char* p = base + static_cast<uint64_t>(src) * ld_bytes;
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}
template <int LPD, int U, bool FILT>
__global__ void __launch_bounds__(256, (U <= 3 ? 5 : U == 4 ? 4 : 3)) k_agg_vec8(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                     const Edge* __restrict__ edges,
                                                     const uint32_t* __restrict__ order, uint32_t d_begin,
                                                     uint64_t n_items, uint32_t chunks,
                                                     const float* __restrict__ in, uint32_t ld_in_bytes,
                                                     float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                     int accumulate, float2 zeros, uint32_t zmask, int chunk_major,
                                                     AggExt ext) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    if (item >= n_items) return;
    const Zs z = zs_of(zeros);
    const uint64_t nd = n_items / chunks;
    const uint64_t nf = chunk_major > 1 ? static_cast<uint64_t>(chunk_major - 2) : 0;
    uint32_t di, ci;
    if (!chunk_major || item < nf * chunks) {
        di = static_cast<uint32_t>(item / chunks);
        ci = static_cast<uint32_t>(item % chunks);
    } else {
        const uint64_t r = item - nf * chunks, nr = nd - nf;
        di = static_cast<uint32_t>(nf + r % nr);
        ci = static_cast<uint32_t>(r / nr);
    }
    const uint32_t d = __ldg(order + d_begin + di);
    if (FILT && !ext_dst_on(ext, d)) return;
    constexpr uint32_t kChunk = 8u * LPD;
    const unsigned sl = static_cast<unsigned>(t % LPD);
    const uint32_t col = ci * kChunk + sl * 8u;
    const bool active = col < dim;
    uint64_t e = __ldg(ebeg + d);
    const uint64_t end = __ldg(eend + d);
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * kChunk) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
    Acc a0 = acc_load(orow, col, dim, accumulate), a1 = acc_load(orow + 4, col + 4, dim, accumulate);
    constexpr int NPL = (U + LPD - 1) / LPD;
    const unsigned submask = LPD >= 32 ? 0xffffffffu : (((1u << LPD) - 1u) << (lane_id() & ~(LPD - 1u)));
    auto batch_recs = [&](Edge (&ed)[U], uint32_t n) {
        if constexpr (LPD <= 8) {
            Edge mine[NPL];
#pragma unroll
            for (int i = 0; i < NPL; ++i) {
                const unsigned k = sl + i * LPD;
                mine[i] = ld_rec(edges + e + (k < n ? k : n - 1));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ed[u].x = __shfl_sync(submask, mine[u / LPD].x, u % LPD, LPD);
                ed[u].y = __shfl_sync(submask, mine[u / LPD].y, u % LPD, LPD);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + (u < static_cast<int>(n) ? u : n - 1));
        }
    };
    auto gather = [&](const Edge& ed, float4& xa, float4& xb) {
        if (FILT && !ext_src_on(ext, ed.x)) xa = xb = make_float4(0.f, 0.f, 0.f, 0.f);  // skipped: +-0 term
        else ld_row8(base, ed.x, ld_in_bytes, xa, xb);
    };
    for (; e + U <= end; e += U) {
        Edge ed[U];
        batch_recs(ed, U);
        float4 x[2 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) gather(ed[u], x[2 * u], x[2 * u + 1]);
        const Zs zz = batch_dep<2 * U>(x, z, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float w = __uint_as_float(ed[u].y);
            acc_step(a0, w, x[2 * u], zz);
            acc_step(a1, w, x[2 * u + 1], zz);
        }
    }
    if (e < end) {
        const uint32_t n = static_cast<uint32_t>(end - e);
        Edge ed[U];
        batch_recs(ed, n);
        float4 x[2 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < static_cast<int>(n)) gather(ed[u], x[2 * u], x[2 * u + 1]);
            else x[2 * u] = x[2 * u + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const Zs zz = batch_dep<2 * U>(x, z, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(n)) {
                const float w = __uint_as_float(ed[u].y);
                acc_step(a0, w, x[2 * u], zz);
                acc_step(a1, w, x[2 * u + 1], zz);
            }
    }
    acc_store_ext(orow, col, dim, a0, z, ext, d, row);
    acc_store_ext(orow + 4, col + 4, dim, a1, z, ext, d, row);
}

// Whole-row warps for wide rows (tuning "row_kernel"): one warp per
// destination over the whole row, NS float4 slots per lane (slot j = float4
// columns 32 j + lane). What bounds k_agg_vec4 on the Reddit layer-0 path is
// the L1 -> register writeback (ncu l1tex__lsu_writeback_active 85 %,
// data_pipe_lsu_wavefronts 87 %; the L2 -> L1 fill is at 49 %): it costs one
// cycle per register written per lane, so a 128-column item pays 4 cycles of
// row data plus 2 of broadcast edge record per edge — a third of the
// writeback is records. Here one record serves the whole row: for 602
// columns 5 x 4 + 2 = 22 cycles per edge instead of 5 x (4 + 2) = 30. The
// per-pass source working set is the whole row, so the path runs as more
// (L2-sized) source segments. Same fp32 order as k_agg_vec4 (per column,
// ascending edge, separately rounded multiply and add): bit-identical.
// Lanes past dim in the last slot re-read the slot's first float4 (same
// sector, in bounds) and discard it.
template <int NS, int U>
__global__ void __launch_bounds__(256, 2) k_agg_row(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                    const Edge* __restrict__ edges,
                                                    const uint32_t* __restrict__ order, uint32_t d_begin,
                                                    uint32_t nd, const float* __restrict__ in, uint32_t ld_in_bytes,
                                                    float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                    int accumulate, float2 zeros, uint32_t zmask, AggExt ext) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= nd) return;
    const uint32_t lane = lane_id();
    const Zs z = zs_of(zeros);
    const uint32_t d = __ldg(order + d_begin + w);
    uint64_t e = __ldg(ebeg + d);
    const uint64_t end = __ldg(eend + d);
    const uint32_t nq = (dim + 3) / 4;
    // slot j < NS - 1 sits at byte 512 j from the lane's slot-0 column; the
    // last slot's lanes past dim fall back to the slot's first float4
    const uint32_t qlast = (NS - 1) * 32 + lane;
    const uint32_t off_last = (qlast < nq ? qlast : (NS - 1) * 32u) * 16u - lane * 16u;
    const char* base = reinterpret_cast<const char*>(in) + lane * 16u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out;
    Acc acc[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) acc[j] = acc_load(orow + (j * 32 + lane) * 4, (j * 32 + lane) * 4, dim, accumulate);
    auto gather = [&](const Edge (&ed)[U], float4 (&x)[U][NS]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const char* p = base + static_cast<uint64_t>(ed[u].x) * ld_in_bytes;
#pragma unroll
            for (int j = 0; j < NS; ++j)
                x[u][j] = ld_row<0>(p + (j + 1 < NS ? j * 512u : off_last), 0u, 0u);
        }
    };
    auto fold = [&](const float4 (&x)[U][NS]) {
        uint32_t all = 0;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < NS; ++j) all ^= __float_as_uint(x[u][j].x);
        all &= zmask;
        Zs r = z;
        r.nz ^= (static_cast<unsigned long long>(all) << 32) | all;
        return r;
    };
    for (; e + U <= end; e += U) {
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + u);
        float4 x[U][NS];
        gather(ed, x);
        const Zs zz = fold(x);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < NS; ++j) acc_step(acc[j], __uint_as_float(ed[u].y), x[u][j], zz);
    }
    if (e < end) {
        const uint32_t n = static_cast<uint32_t>(end - e);
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + (u < static_cast<int>(n) ? u : 0));
        float4 x[U][NS];
        gather(ed, x);
        const Zs zz = fold(x);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(n))
#pragma unroll
                for (int j = 0; j < NS; ++j) acc_step(acc[j], __uint_as_float(ed[u].y), x[u][j], zz);
    }
#pragma unroll
    for (int j = 0; j < NS; ++j)
        acc_store_ext(orow + (j * 32 + lane) * 4, (j * 32 + lane) * 4, dim, acc[j], z, ext, d, row);
}

// Source-window lockstep (tuning "vec_window"): the 16 warps of a 512-thread
// CTA are 16 consecutive (degree-sorted, similar) destinations of one column
// chunk. They walk the CTA's source range in nwin windows, each warp taking
// only its edges below the window end, with a CTA barrier between windows,
// so the rows the destinations share are gathered within one window and hit
// in L1 (32 such destinations share 31 % of their sources on Reddit layer
// 0). Same per-column ascending-edge order: bit-identical.
template <int U>
__global__ void __launch_bounds__(512, 2) k_agg_vec4w(const uint64_t* __restrict__ ebeg,
                                                     const uint64_t* __restrict__ eend,
                                                     const Edge* __restrict__ edges,
                                                     const uint32_t* __restrict__ order, uint32_t d_begin,
                                                     uint64_t n_items, uint32_t chunks,
                                                     const float* __restrict__ in, uint32_t ld_in_bytes,
                                                     float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                     int accumulate, float2 zeros, uint32_t zmask, int chunk_major,
                                                     uint32_t win_edges, AggExt ext) {
    __shared__ uint32_t s_lo, s_hi, s_cnt;
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t >> 5;
    const bool valid = item < n_items;
    if (threadIdx.x == 0) {
        s_lo = 0xffffffffu;
        s_hi = 0u;
        s_cnt = 0u;
    }
    __syncthreads();
    const Zs z = zs_of(zeros);
    const uint64_t nd = n_items / chunks;
    const uint64_t nf = chunk_major > 1 ? static_cast<uint64_t>(chunk_major - 2) : 0;
    uint32_t di = 0, ci = 0;
    if (!chunk_major || item < nf * chunks) {
        di = static_cast<uint32_t>(item / chunks);
        ci = static_cast<uint32_t>(item % chunks);
    } else {
        const uint64_t r = item - nf * chunks, nr = nd - nf;
        di = static_cast<uint32_t>(nf + r % nr);
        ci = static_cast<uint32_t>(r / nr);
    }
    const uint32_t lane = lane_id();
    const uint32_t d = valid ? __ldg(order + d_begin + di) : 0u;
    const uint32_t col = (ci * 32 + lane) * 4;
    const bool active = valid && col < dim;
    uint64_t e = valid ? __ldg(ebeg + d) : 0, end = valid ? __ldg(eend + d) : 0;
    if (lane == 0 && e < end) {
        atomicMin(&s_lo, __ldg(&edges[e].x));
        atomicMax(&s_hi, __ldg(&edges[end - 1].x));
        atomicMax(&s_cnt, end - e < 0xffffffffull ? static_cast<uint32_t>(end - e) : 0xffffffffu);
    }
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * 128u) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    const uint32_t row = valid ? ext_out_row(ext, d) : 0u;
    float* orow = out + row * ld_out + col;
    Acc acc = acc_load(orow, col, active ? dim : 0u, accumulate);
    __syncthreads();
    const uint32_t lo = s_lo, hi = s_hi;
    const uint32_t nwin = s_cnt ? min(64u, max(1u, s_cnt / max(1u, win_edges))) : 0u;
    const uint64_t span = static_cast<uint64_t>(hi) - lo + 1;
    for (uint32_t w = 0; w < nwin; ++w) {
        const uint64_t wend = lo + span * (w + 1) / nwin;  // exclusive
        while (e < end) {
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + (e + u < end ? u : 0));
            // the window's edges are a prefix of the batch (sources ascend)
            uint32_t n_ok = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) n_ok += (e + u < end && ed[u].x < wend) ? 1u : 0u;
            if (!n_ok) break;
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                x[u] = u < static_cast<int>(n_ok) ? ld_row<0>(base, ed[u].x, ld_in_bytes)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < static_cast<int>(n_ok)) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
            e += n_ok;
            if (n_ok < U) break;
        }
        __syncthreads();
    }
    if (valid) acc_store_ext(orow, col, dim, acc, z, ext, d, row);
}

// One launch over a SEQUENCE of destination runs (the host drop-in's last
// pass, tuning "host_seq"): run s covers items [item0, item0 + nd*chunks)
// of destinations dlist[dofs .. dofs+nd), destination-major (the hub front)
// or column-chunk-major, and each finished item bumps counters[counter] after
// a system-scope fence, so a copy stream can wait (cuStreamWaitValue32) for a
// row chunk's last item and start its D2H while the launch goes on: no
// per-chunk launch tails. The body is k_agg_vec4's (LPD 32, U 8): the same
// per-column ascending-edge order, bit-identical.
template <int U>
__global__ void __launch_bounds__(256, 4) k_agg_vec4_seq(const uint64_t* __restrict__ ebeg,
                                                        const uint64_t* __restrict__ eend,
                                                        const Edge* __restrict__ edges,
                                                        const uint32_t* __restrict__ dlist, SeqTable tab,
                                                        uint64_t n_items, uint32_t chunks,
                                                        const float* __restrict__ in, uint32_t ld_in_bytes,
                                                        float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                        int accumulate, float2 zeros, uint32_t zmask,
                                                        unsigned* __restrict__ counters) {
    __shared__ uint32_t s_cnt[8];  // the completion counter of each warp's item (~0u: none)
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t >> 5;
    const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
    uint32_t si = 0;
    while (si + 1 < tab.nseg && item >= tab.seg[si + 1].item0) ++si;
    const SeqSeg sg = tab.seg[si];
    const uint64_t local = item - sg.item0;
    // (items past a run's nd * chunks are the CTA-alignment padding)
    if (item < n_items && local < static_cast<uint64_t>(sg.nd) * chunks) {  // no early return: the CTA meets below
        const uint32_t di = static_cast<uint32_t>(sg.dest_major ? local / chunks : local % sg.nd);
        const uint32_t ci = static_cast<uint32_t>(sg.dest_major ? local % chunks : local / sg.nd);
        const Zs z = zs_of(zeros);
        const uint32_t d = __ldg(dlist + sg.dofs + di);
        const uint32_t col = (ci * 32 + lane) * 4;
        const bool active = col < dim;
        uint64_t e = __ldg(ebeg + d);
        const uint64_t end = __ldg(eend + d);
        const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * 128u) * 4u;
        asm("mov.b64 %0, %0;" : "+l"(base));
        float* orow = out + d * ld_out + col;
        Acc acc = acc_load(orow, col, dim, accumulate);
        for (; e + U <= end; e += U) {
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + u);
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = ld_row<0>(base, ed[u].x, ld_in_bytes);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
        }
        if (e < end) {
            const uint32_t n = static_cast<uint32_t>(end - e);
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + (u < static_cast<int>(n) ? u : n - 1));
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                x[u] = u < static_cast<int>(n) ? ld_row<0>(base, ed[u].x, ld_in_bytes) : make_float4(0.f, 0.f, 0.f, 0.f);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < static_cast<int>(n)) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
        }
        if (active) {
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc.lo) : "l"(acc.lo), "l"(z.pz));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc.hi) : "l"(acc.hi), "l"(z.pz));
            const float2 l = unpk2(acc.lo), h = unpk2(acc.hi);
            if (col + 3 < dim) {
                *reinterpret_cast<float4*>(orow) = make_float4(l.x, l.y, h.x, h.y);
            } else {
                orow[0] = l.x;
                if (col + 1 < dim) orow[1] = l.y;
                if (col + 2 < dim) orow[2] = h.x;
            }
        }
        if (lane == 0) s_cnt[wib] = sg.counter;
    } else if (lane == 0) {
        s_cnt[wib] = ~0u;
    }
    // every thread's stores ordered before the CTA's completion marks (one
    // atomic per distinct counter per CTA, not per warp: the counters of a
    // chunk are hit by every CTA of its items)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nw = blockDim.x >> 5;
        for (uint32_t w = 0; w < nw; ++w) {
            const uint32_t c = s_cnt[w];
            if (c == ~0u) continue;
            bool seen = false;
            for (uint32_t v = 0; v < w; ++v) seen |= s_cnt[v] == c;
            if (seen) continue;
            uint32_t k = 0;
            for (uint32_t v = w; v < nw; ++v) k += s_cnt[v] == c;
            atomicAdd(counters + c, k);
        }
    }
}

template <int NS>
void launch_row_ns(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order,
                   uint32_t d_begin, uint32_t nd, const float* in, uint64_t ld_in, float* out, uint64_t ld_out,
                   uint32_t dim, bool accumulate, cudaStream_t s, const AggExt& ext, int u) {
    const unsigned grid = grid_for(static_cast<uint64_t>(nd) * 32, 256);
    const uint32_t ldb = static_cast<uint32_t>(ld_in * 4);
    if (u >= 4)
        k_agg_row<NS, 4><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, nd, in, ldb, out, ld_out, dim,
                                              accumulate, kZeros, 0u, ext);
    else if (u == 3)
        k_agg_row<NS, 3><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, nd, in, ldb, out, ld_out, dim,
                                              accumulate, kZeros, 0u, ext);
    else
        k_agg_row<NS, 2><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, nd, in, ldb, out, ld_out, dim,
                                              accumulate, kZeros, 0u, ext);
    PG_LAUNCH("k_agg_row");
}

// ---- CommitMode::Fast, group partitioned (PG_AGG_GROUPED) ----------------
// aggregate.hpp:84-115: one (sub-)warp per (neighbour group, column chunk):
// the group's <= gs edges accumulate in edge order into a zero scratch,
// then commit — a plain out += scratch when the destination owns a single
// group, atomic adds (red.global.add.v4.f32) otherwise. Load balance comes
// from the group size, so the structure-aware gs selector (gs_model.cpp,
// group_cost.cpp) shapes the GPU schedule here. Across groups of one
// destination the fp32 order follows the atomics: within tolerance of the
// reference's Fast (and Deterministic) result, not bit-exact.
template <int LPD, int U>
__global__ void __launch_bounds__(256, (U <= 8 ? 4 : 2)) k_agg_groups(
    const uint64_t* __restrict__ gbeg, const uint64_t* __restrict__ gend, const uint32_t* __restrict__ gdest,
    const uint64_t* __restrict__ dest_groups, const Edge* __restrict__ edges, uint64_t n_items, uint32_t chunks,
    const float* __restrict__ in, uint32_t ld_in_bytes, float* __restrict__ out, uint64_t ld_out, uint32_t dim,
    int accumulate, float2 zeros, uint32_t zmask, int chunk_major) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    if (item >= n_items) return;
    const Zs z = zs_of(zeros);
    const uint64_t ng = n_items / chunks;
    const uint64_t gi = chunk_major ? item % ng : item / chunks;
    const uint32_t ci = static_cast<uint32_t>(chunk_major ? item / ng : item % chunks);
    const uint32_t d = __ldg(gdest + gi);
    const uint32_t col = (ci * LPD + static_cast<uint32_t>(t % LPD)) * 4;
    const bool active = col < dim;
    uint64_t e = __ldg(gbeg + gi);
    const uint64_t end = __ldg(gend + gi);
    const bool multi = __ldg(dest_groups + d + 1) - __ldg(dest_groups + d) > 1;
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * LPD * 4u) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    Acc acc{0ull, 0ull};  // scratch, zero filled (aggregate.hpp:93)
    for (; e + U <= end; e += U) {
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + u);
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld_row(base, ed[u].x, ld_in_bytes);
        const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
    }
    if (e < end) {
        const uint32_t n = static_cast<uint32_t>(end - e);
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + (u < static_cast<int>(n) ? u : n - 1));
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld_row(base, ed[u].x, ld_in_bytes);
        const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(n)) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
    }
    if (!active) return;
    float* orow = out + d * ld_out + col;
    const float2 l = unpk2(acc.lo), h = unpk2(acc.hi);
    const float4 v = make_float4(l.x, l.y, h.x, h.y);
    const bool full = col + 3 < dim;
    if (multi) {  // #pragma omp atomic (aggregate.hpp:105-109); output zeroed by the caller
        if (full) {
            atomicAdd(reinterpret_cast<float4*>(orow), v);
        } else {
            atomicAdd(orow, v.x);
            if (col + 1 < dim) atomicAdd(orow + 1, v.y);
            if (col + 2 < dim) atomicAdd(orow + 2, v.z);
        }
        return;
    }
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);  // out += scratch (aggregate.hpp:102-103)
    if (accumulate) {
        if (full) o = *reinterpret_cast<const float4*>(orow);
        else {
            o.x = orow[0];
            if (col + 1 < dim) o.y = orow[1];
            if (col + 2 < dim) o.z = orow[2];
        }
    }
    o.x = __fadd_rn(o.x, v.x);
    o.y = __fadd_rn(o.y, v.y);
    o.z = __fadd_rn(o.z, v.z);
    o.w = __fadd_rn(o.w, v.w);
    if (full) {
        *reinterpret_cast<float4*>(orow) = o;
    } else {
        orow[0] = o.x;
        if (col + 1 < dim) orow[1] = o.y;
        if (col + 2 < dim) orow[2] = o.z;
    }
}

// Fast with a CTA-segmented reduction (tuning "grouped_seg", off by default:
// measured 1.6x faster at gs = 1 but 5-40 % slower over gs 8-512, where the
// barrier and the serial run sums cost more than the atomics they save):
// the items of a CTA are consecutive groups of one column chunk, so the
// groups of a destination that land in the same CTA are combined in shared
// memory, in group order, by the run's first item, which commits once — a
// plain store when the run holds all of the destination's groups, one
// atomic add per column otherwise. Global atomics drop from one per extra
// group to one per CTA boundary a destination straddles.
template <int LPD, int U>
__global__ void __launch_bounds__(256, 4) k_agg_groups_seg(
    const uint64_t* __restrict__ gbeg, const uint64_t* __restrict__ gend, const uint32_t* __restrict__ gdest,
    const uint64_t* __restrict__ dest_groups, const Edge* __restrict__ edges, uint64_t n_items, uint32_t chunks,
    const float* __restrict__ in, uint32_t ld_in_bytes, float* __restrict__ out, uint64_t ld_out, uint32_t dim,
    int accumulate, float2 zeros, uint32_t zmask) {
    constexpr int IPC = 256 / LPD;  // items per CTA
    __shared__ float4 part[256];
    __shared__ uint32_t s_dest[IPC], s_chunk[IPC];
    __shared__ uint64_t s_group[IPC];
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    const unsigned it = threadIdx.x / LPD, sub = threadIdx.x % LPD;
    const bool valid = item < n_items;
    const Zs z = zs_of(zeros);
    const uint64_t ng = n_items / chunks;
    const uint64_t gi = valid ? item % ng : 0;  // chunk-major: consecutive items are consecutive groups
    const uint32_t ci = valid ? static_cast<uint32_t>(item / ng) : 0;
    const uint32_t d = valid ? __ldg(gdest + gi) : 0xffffffffu;
    const uint32_t col = (ci * LPD + sub) * 4;
    const bool active = valid && col < dim;
    Acc acc{0ull, 0ull};
    if (valid) {
        uint64_t e = __ldg(gbeg + gi);
        const uint64_t end = __ldg(gend + gi);
        const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * LPD * 4u) * 4u;
        asm("mov.b64 %0, %0;" : "+l"(base));
        for (; e + U <= end; e += U) {
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + u);
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = ld_row(base, ed[u].x, ld_in_bytes);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
        }
        if (e < end) {
            const uint32_t n = static_cast<uint32_t>(end - e);
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = ld_rec(edges + e + (u < static_cast<int>(n) ? u : n - 1));
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = ld_row(base, ed[u].x, ld_in_bytes);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < static_cast<int>(n)) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
        }
    }
    const float2 l = unpk2(acc.lo), h = unpk2(acc.hi);
    part[threadIdx.x] = make_float4(l.x, l.y, h.x, h.y);
    if (sub == 0) {
        s_dest[it] = d;
        s_chunk[it] = ci;
        s_group[it] = gi;
    }
    __syncthreads();
    if (!active) return;
    if (it > 0 && s_dest[it - 1] == d && s_chunk[it - 1] == ci) return;  // not the head of its run
    int last = it;
    while (last + 1 < IPC && s_dest[last + 1] == d && s_chunk[last + 1] == ci) ++last;
    float4 v = part[it * LPD + sub];
    for (int k = it + 1; k <= last; ++k) {  // the run's partials in group order
        const float4 p = part[k * LPD + sub];
        v.x = __fadd_rn(v.x, p.x);
        v.y = __fadd_rn(v.y, p.y);
        v.z = __fadd_rn(v.z, p.z);
        v.w = __fadd_rn(v.w, p.w);
    }
    float* orow = out + d * ld_out + col;
    const bool full = col + 3 < dim;
    const bool whole = s_group[it] == __ldg(dest_groups + d) && s_group[last] + 1 == __ldg(dest_groups + d + 1);
    if (!whole) {  // the destination's other groups commit from other CTAs: output zeroed by the caller
        if (full) {
            atomicAdd(reinterpret_cast<float4*>(orow), v);
        } else {
            atomicAdd(orow, v.x);
            if (col + 1 < dim) atomicAdd(orow + 1, v.y);
            if (col + 2 < dim) atomicAdd(orow + 2, v.z);
        }
        return;
    }
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (accumulate) {
        if (full) o = *reinterpret_cast<const float4*>(orow);
        else {
            o.x = orow[0];
            if (col + 1 < dim) o.y = orow[1];
            if (col + 2 < dim) o.z = orow[2];
        }
    }
    o.x = __fadd_rn(o.x, v.x);
    o.y = __fadd_rn(o.y, v.y);
    o.z = __fadd_rn(o.z, v.z);
    o.w = __fadd_rn(o.w, v.w);
    if (full) {
        *reinterpret_cast<float4*>(orow) = o;
    } else {
        orow[0] = o.x;
        if (col + 1 < dim) orow[1] = o.y;
        if (col + 2 < dim) orow[2] = o.z;
    }
}

template <int LPD>
void launch_groups(const uint64_t* gbeg, const uint64_t* gend, const uint32_t* gdest, const uint64_t* dest_groups,
                   const Edge* edges, uint64_t G, uint32_t chunks, const float* in, uint64_t ld_in, float* out,
                   uint64_t ld_out, uint32_t dim, bool accumulate, cudaStream_t s) {
    const uint64_t items = G * chunks;
    if (tuning(kTuneGroupedSeg) == 1) {
        k_agg_groups_seg<LPD, 8><<<grid_for(items * LPD, 256), 256, 0, s>>>(
            gbeg, gend, gdest, dest_groups, edges, items, chunks, in, static_cast<uint32_t>(ld_in * 4), out, ld_out,
            dim, accumulate, kZeros, 0u);
        PG_LAUNCH("k_agg_groups_seg");
        return;
    }
    k_agg_groups<LPD, 8><<<grid_for(items * LPD, 256), 256, 0, s>>>(
        gbeg, gend, gdest, dest_groups, edges, items, chunks, in, static_cast<uint32_t>(ld_in * 4), out, ld_out, dim,
        accumulate, kZeros, 0u, chunks > 1 && tuning(kTuneChunkMajor) ? 1 : 0);
    PG_LAUNCH("k_agg_groups");
}

// Heavy wide destinations (non-pipelined, heavy_wide_pipe = 0): 32-edge record
// batches broadcast by shuffle, a plain float4 accumulator and scalar FMUL/FADD — in this form ptxas keeps
// all U = 32 gathers of a batch in flight (154 registers, measured 8-way
// shard hub rank 11.3 -> 4.1 ms on B200).
__device__ __forceinline__ void acc4_scalar(float4& a, float w, const float4& x) {
    a.x = __fadd_rn(a.x, __fmul_rn(w, x.x));
    a.y = __fadd_rn(a.y, __fmul_rn(w, x.y));
    a.z = __fadd_rn(a.z, __fmul_rn(w, x.z));
    a.w = __fadd_rn(a.w, __fmul_rn(w, x.w));
}

template <int U>
__global__ void __launch_bounds__(256) k_agg_wide_lat(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                     const Edge* __restrict__ edges,
                                                     const uint32_t* __restrict__ order, uint32_t d_begin,
                                                     uint64_t n_items, uint32_t chunks,
                                                     const float* __restrict__ in, uint64_t ld_in,
                                                     float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                     int accumulate, uint32_t zmask, AggExt ext) {
    const uint64_t item = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (item >= n_items) return;
    const unsigned lane = lane_id();
    const uint32_t d = order[d_begin + item / chunks];
    const uint32_t col = (static_cast<uint32_t>(item % chunks) * 32 + lane) * 4;
    const bool active = col < dim;
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
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
    Edge nxt = eb + lane < ee ? __ldg(edges + eb + lane) : make_uint2(0u, 0u);
    for (uint64_t e0 = eb; e0 < ee; e0 += 32) {
        const Edge cur = nxt;
        if (e0 + 32 + lane < ee) nxt = __ldg(edges + e0 + 32 + lane);
        const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(32), ee - e0));
        if (n == 32) {
#pragma unroll
            for (int s = 0; s < 32; s += U) {
                uint32_t src[U];
                float w[U];
                float4 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    src[u] = __shfl_sync(0xffffffffu, cur.x, s + u);
                    w[u] = __uint_as_float(__shfl_sync(0xffffffffu, cur.y, s + u));
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    x[u] = active ? ldg4(icol + src[u] * ld_in) : make_float4(0.f, 0.f, 0.f, 0.f);
                // every multiply of the batch depends on all U loads through a
                // mask that is zero at run time (bit-neutral): the scheduler
                // has to issue the whole batch of gathers first
                uint32_t all = 0;
#pragma unroll
                for (int u = 0; u < U; ++u) all ^= __float_as_uint(x[u].x);
                all &= zmask;
#pragma unroll
                for (int u = 0; u < U; ++u) acc4_scalar(acc, __uint_as_float(__float_as_uint(w[u]) ^ all), x[u]);
            }
        } else {
            for (uint32_t j = 0; j < n; ++j) {
                const uint32_t src = __shfl_sync(0xffffffffu, cur.x, j);
                const float w = __uint_as_float(__shfl_sync(0xffffffffu, cur.y, j));
                const float4 x = active ? ldg4(icol + src * ld_in) : make_float4(0.f, 0.f, 0.f, 0.f);
                acc4_scalar(acc, w, x);
            }
        }
    }
    if (!active) return;
    acc.x = __fadd_rn(acc.x, 0.f);
    acc.y = __fadd_rn(acc.y, 0.f);
    acc.z = __fadd_rn(acc.z, 0.f);
    acc.w = __fadd_rn(acc.w, 0.f);
    acc = ext_relu(ext, d, row, col, dim, acc);
    if (col + 3 < dim) {
        __stcs(reinterpret_cast<float4*>(orow), acc);
    } else {
        orow[0] = acc.x;
        if (col + 1 < dim) orow[1] = acc.y;
        if (col + 2 < dim) orow[2] = acc.z;
    }
}

// Heavy narrow destinations (rows of <= 64 floats): a warp per (hub, 32-float
// column chunk), one SCALAR column per lane. A float4-per-lane layout leaves
// a 16-float row on 4 lanes and its serial chain at ~6 instructions per
// edge; here every lane carries one column's chain (FMUL + FADD per edge)
// while all 32 lanes keep a 32-edge batch of row gathers in flight (records
// loaded coalesced one per lane, sources broadcast by shuffle, the batch
// forced in flight by the runtime-zero dependency). The hub's chain is the
// only serial part: ~deg x 4 cycles.
template <bool FILT>
__global__ void __launch_bounds__(256) k_agg_narrow_lat(const uint64_t* __restrict__ ebeg,
                                                       const uint64_t* __restrict__ eend,
                                                       const Edge* __restrict__ edges,
                                                       const uint32_t* __restrict__ order, uint32_t d_begin,
                                                       uint64_t n_items, uint32_t chunks,
                                                       const float* __restrict__ in, uint64_t ld_in,
                                                       float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                       int accumulate, uint32_t zmask, AggExt ext) {
    const uint64_t item = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (item >= n_items) return;
    const unsigned lane = lane_id();
    const uint32_t d = order[d_begin + item / chunks];
    if (FILT && !ext_dst_on(ext, d)) return;
    const uint32_t col = static_cast<uint32_t>(item % chunks) * 32 + lane;
    const bool active = col < dim;
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
    float acc = (accumulate && active) ? *orow : 0.f;
    const float* icol = in + (active ? col : 0u);
    Edge nxt = eb + lane < ee ? __ldg(edges + eb + lane) : make_uint2(0u, 0u);
    for (uint64_t e0 = eb; e0 < ee; e0 += 32) {
        Edge cur = nxt;
        if (e0 + 32 + lane < ee) nxt = __ldg(edges + e0 + 32 + lane);
        const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(32), ee - e0));
        if (FILT && lane < n && !ext_src_on(ext, cur.x)) cur.y = 0u;  // skipped: a +-0 term
        if (n == 32) {
            float x[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint32_t src = __shfl_sync(0xffffffffu, cur.x, u);
                x[u] = __ldg(icol + static_cast<uint64_t>(src) * ld_in);
            }
            uint32_t all = 0;
#pragma unroll
            for (int u = 0; u < 32; ++u) all ^= __float_as_uint(x[u]);
            all &= zmask;
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const float w = __uint_as_float(__shfl_sync(0xffffffffu, cur.y, u) ^ all);
                acc = __fadd_rn(acc, __fmul_rn(w, x[u]));
            }
        } else {
            for (uint32_t j = 0; j < n; ++j) {
                const uint32_t src = __shfl_sync(0xffffffffu, cur.x, j);
                const float w = __uint_as_float(__shfl_sync(0xffffffffu, cur.y, j));
                acc = __fadd_rn(acc, __fmul_rn(w, __ldg(icol + static_cast<uint64_t>(src) * ld_in)));
            }
        }
    }
    if (!active) return;
    acc = __fadd_rn(acc, 0.f);
    if (ext.relu_pre) {
        const uint32_t prow = ext.pre_rows ? __ldg(ext.pre_rows + d) : row;
        acc = ext.relu_pre[static_cast<uint64_t>(prow) * ext.ld_pre + col] > 0.f ? acc : 0.f;
    }
    *orow = acc;
}

// Heavy wide destinations, software-pipelined (tuning "heavy_wide_pipe"):
// a hub is one serial chain per column, so its time is (edges / batch) x
// (gather latency + fold). Here the gathers of batch t+1 are issued before
// batch t is folded (two register batches of U rows, ~160 registers: hubs
// are few, occupancy is irrelevant), so the fold hides under the next
// batch's latency. Records are loaded coalesced one per lane 32 at a time
// and broadcast by shuffle; the runtime-zero dependency keeps each batch's
// gathers issued together.
template <int U>
__global__ void __launch_bounds__(64) k_agg_wide_pipe(const uint64_t* __restrict__ ebeg,
                                                     const uint64_t* __restrict__ eend,
                                                     const Edge* __restrict__ edges,
                                                     const uint32_t* __restrict__ order, uint32_t d_begin,
                                                     uint64_t n_items, uint32_t chunks,
                                                     const float* __restrict__ in, uint32_t ld_in_bytes,
                                                     float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                     int accumulate, uint32_t zmask, AggExt ext, int chunk_major) {
    static_assert(32 % U == 0, "U divides the 32-record window");
    const uint64_t item = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (item >= n_items) return;
    const unsigned lane = lane_id();
    // chunk-major: every hub's chunk 0 first, like the concurrent main
    // kernel, so both gather from the same column chunk of the segment
    const uint64_t nhub = n_items / chunks;
    const uint32_t d = order[d_begin + (chunk_major ? item % nhub : item / chunks)];
    const uint32_t ci = static_cast<uint32_t>(chunk_major ? item / nhub : item % chunks);
    const uint32_t col = (ci * 32 + lane) * 4;
    const bool active = col < dim;
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (accumulate && active) {
        if (col + 3 < dim) acc = *reinterpret_cast<const float4*>(orow);
        else {
            acc.x = orow[0];
            if (col + 1 < dim) acc.y = orow[1];
            if (col + 2 < dim) acc.z = orow[2];
        }
    }
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * 128u) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    const uint64_t nb = (ee - eb + U - 1) / U;
    // record window: 32 records, one per lane; batch b uses records
    // [eb + b*U, eb + b*U + U) = lanes ((b*U) % 32) ... of window (b*U)/32
    Edge win = eb + lane < ee ? __ldg(edges + eb + lane) : make_uint2(0u, 0u);
    Edge nwin = eb + 32 + lane < ee ? __ldg(edges + eb + 32 + lane) : make_uint2(0u, 0u);
    float4 xa[U], xb[U];
    float wa[U], wb[U];
    auto gather = [&](uint64_t b, float4 (&x)[U], float (&w)[U]) {
        const int s0 = static_cast<int>((b * U) & 31);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t src = __shfl_sync(0xffffffffu, win.x, s0 + u);
            w[u] = __uint_as_float(__shfl_sync(0xffffffffu, win.y, s0 + u));  // 0 past the end
            x[u] = ld_row(base, src, ld_in_bytes);
        }
        if (s0 + U == 32) {  // window consumed: slide
            win = nwin;
            const uint64_t e = eb + (b + 1) * U + 32 + lane;
            nwin = e < ee ? __ldg(edges + e) : make_uint2(0u, 0u);
        }
    };
    auto fold = [&](const float4 (&x)[U], const float (&w)[U]) {
        uint32_t all = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) all ^= __float_as_uint(x[u].x);
        all &= zmask;
#pragma unroll
        for (int u = 0; u < U; ++u) acc4_scalar(acc, __uint_as_float(__float_as_uint(w[u]) ^ all), x[u]);
    };
    if (nb) gather(0, xa, wa);
    for (uint64_t b = 0; b < nb; b += 2) {
        if (b + 1 < nb) gather(b + 1, xb, wb);  // in flight while batch b folds
        fold(xa, wa);
        if (b + 1 < nb) {
            if (b + 2 < nb) gather(b + 2, xa, wa);
            fold(xb, wb);
        }
    }
    if (!active) return;
    acc.x = __fadd_rn(acc.x, 0.f);
    acc.y = __fadd_rn(acc.y, 0.f);
    acc.z = __fadd_rn(acc.z, 0.f);
    acc.w = __fadd_rn(acc.w, 0.f);
    acc = ext_relu(ext, d, row, col, dim, acc);
    if (col + 3 < dim) {
        __stcs(reinterpret_cast<float4*>(orow), acc);
    } else {
        orow[0] = acc.x;
        if (col + 1 < dim) orow[1] = acc.y;
        if (col + 2 < dim) orow[2] = acc.z;
    }
}


// Scalar fallback for unaligned rows (ld or base not 16-byte aligned).
// k_agg_wide_pipe with a float2 per lane (tuning heavy_wide_pipe 5): a hub
// item covers 64 columns, so the same registers hold twice the rows — U = 32
// per batch, two batches (64 rows) in flight per chain — and a hub has twice
// the items. A hub's time is its serial chain: edges x gather latency /
// rows in flight.
__device__ __forceinline__ float2 ld_row2(const char* base, uint32_t src, uint32_t ld_bytes) {
    float2 r;
    const char* p = base + static_cast<uint64_t>(src) * ld_bytes;
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}
template <int U>
__global__ void __launch_bounds__(64) k_agg_wide_pipe2(const uint64_t* __restrict__ ebeg,
                                                      const uint64_t* __restrict__ eend,
                                                      const Edge* __restrict__ edges,
                                                      const uint32_t* __restrict__ order, uint32_t d_begin,
                                                      uint64_t n_items, uint32_t chunks,
                                                      const float* __restrict__ in, uint32_t ld_in_bytes,
                                                      float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                      int accumulate, uint32_t zmask, AggExt ext) {
    static_assert(32 % U == 0, "U divides the 32-record window");
    const uint64_t item = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (item >= n_items) return;
    const unsigned lane = lane_id();
    const uint32_t d = order[d_begin + item / chunks];
    const uint32_t ci = static_cast<uint32_t>(item % chunks);
    const uint32_t col = (ci * 32 + lane) * 2;
    const bool active = col < dim;
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
    float2 acc = make_float2(0.f, 0.f);
    if (accumulate && active) {
        acc.x = orow[0];
        if (col + 1 < dim) acc.y = orow[1];
    }
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * 64u) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    const uint64_t nb = (ee - eb + U - 1) / U;
    Edge win = eb + lane < ee ? __ldg(edges + eb + lane) : make_uint2(0u, 0u);
    Edge nwin = eb + 32 + lane < ee ? __ldg(edges + eb + 32 + lane) : make_uint2(0u, 0u);
    float2 xa[U], xb[U];
    float wa[U], wb[U];
    auto gather = [&](uint64_t b, float2 (&x)[U], float (&w)[U]) {
        const int s0 = static_cast<int>((b * U) & 31);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t src = __shfl_sync(0xffffffffu, win.x, s0 + u);
            w[u] = __uint_as_float(__shfl_sync(0xffffffffu, win.y, s0 + u));  // 0 past the end
            x[u] = ld_row2(base, src, ld_in_bytes);
        }
        if (s0 + U == 32) {  // window consumed: slide
            win = nwin;
            const uint64_t e = eb + (b + 1) * U + 32 + lane;
            nwin = e < ee ? __ldg(edges + e) : make_uint2(0u, 0u);
        }
    };
    auto fold = [&](const float2 (&x)[U], const float (&w)[U]) {
        uint32_t all = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) all ^= __float_as_uint(x[u].x);
        all &= zmask;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float wu = __uint_as_float(__float_as_uint(w[u]) ^ all);
            acc.x = __fadd_rn(acc.x, __fmul_rn(wu, x[u].x));
            acc.y = __fadd_rn(acc.y, __fmul_rn(wu, x[u].y));
        }
    };
    if (nb) gather(0, xa, wa);
    for (uint64_t b = 0; b < nb; b += 2) {
        if (b + 1 < nb) gather(b + 1, xb, wb);  // in flight while batch b folds
        fold(xa, wa);
        if (b + 1 < nb) {
            if (b + 2 < nb) gather(b + 2, xa, wa);
            fold(xb, wb);
        }
    }
    if (!active) return;
    acc.x = __fadd_rn(acc.x, 0.f);
    acc.y = __fadd_rn(acc.y, 0.f);
    if (ext.relu_pre) {
        const uint32_t prow = ext.pre_rows ? __ldg(ext.pre_rows + d) : row;
        const float* pr = ext.relu_pre + static_cast<uint64_t>(prow) * ext.ld_pre + col;
        acc.x = pr[0] > 0.f ? acc.x : 0.f;
        if (col + 1 < dim) acc.y = pr[1] > 0.f ? acc.y : 0.f;
    }
    orow[0] = acc.x;
    if (col + 1 < dim) orow[1] = acc.y;
}

template <int U>
__global__ void __launch_bounds__(256) k_agg_scalar(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                   const Edge* __restrict__ edges,
                                                   const uint32_t* __restrict__ order, uint32_t d_begin,
                                                   uint64_t n_items, uint32_t chunks,
                                                   const float* __restrict__ in, uint64_t ld_in,
                                                   float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                   int accumulate, AggExt ext) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / 32;
    if (item >= n_items) return;
    const uint32_t d = order[d_begin + item / chunks];
    if (!ext_dst_on(ext, d)) return;
    const uint32_t col = static_cast<uint32_t>(item % chunks) * 32 + lane_id();
    const bool active = col < dim;
    uint64_t e = ebeg[d];
    const uint64_t end = eend[d];
    const uint32_t row = ext_out_row(ext, d);
    float acc = (accumulate && active) ? out[row * ld_out + col] : 0.f;
    auto take = [&](const Edge& ed) {
        return active && (!ext.src_bits || ext_src_on(ext, ed.x)) ? __ldg(in + ed.x * ld_in + col) : 0.f;
    };
    for (; e + U <= end; e += U) {
        Edge ed[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ed[u] = __ldg(edges + e + u);
        float x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = take(ed[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __fadd_rn(acc, __fmul_rn(__uint_as_float(ed[u].y), x[u]));
    }
    for (; e < end; ++e) {
        const Edge ed = __ldg(edges + e);
        acc = __fadd_rn(acc, __fmul_rn(__uint_as_float(ed.y), take(ed)));
    }
    if (!active) return;
    acc = __fadd_rn(acc, 0.f);
    if (ext.relu_pre) {
        const uint32_t prow = ext.pre_rows ? __ldg(ext.pre_rows + d) : row;
        acc = ext.relu_pre[static_cast<uint64_t>(prow) * ext.ld_pre + col] > 0.f ? acc : 0.f;
    }
    out[row * ld_out + col] = acc;
}

// ---- heavy destinations: TMA bulk-copy ring ---------------------------------
// One CTA = one producer warp + one consumer warp per (heavy destination,
// 32-float4 column chunk). The producer streams the destination's gradient
// row chunks into a kHeavyStages-deep shared-memory ring with
// cp.async.bulk (one 16..512-byte copy per edge, UBLKCP in SASS) completing
// on mbarriers; the consumer warp applies them in ascending edge order
// (lane = float4 column), so the summation order — and hence every bit —
// is the reference's while a 50K-edge hub still has ~64 KB in flight.
constexpr int kHeavyStages = 4;
constexpr int kHeavyStageBytes = 16384;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra.uni DONE;\n\t"
        "bra.uni LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int CHQ>
__host__ __device__ constexpr int heavy_T() {
    return kHeavyStageBytes / (CHQ * 16);
}
template <int CHQ>
constexpr size_t heavy_smem() {
    return kHeavyStages * (kHeavyStageBytes + heavy_T<CHQ>() * 4) + 2 * kHeavyStages * 8;
}

template <int CHQ>
__global__ void __launch_bounds__(64) k_agg_heavy(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                 const Edge* __restrict__ edges,
                                                 const uint32_t* __restrict__ order, uint32_t d_begin,
                                                 uint32_t chunks, uint32_t nq_total,
                                                 const float* __restrict__ in, uint64_t ld_in,
                                                 float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                 int accumulate, float2 zeros) {
    constexpr int T = heavy_T<CHQ>();
    constexpr int NS = kHeavyStages;
    extern __shared__ __align__(128) unsigned char smem[];
    float4* buf = reinterpret_cast<float4*>(smem);
    float* wbuf = reinterpret_cast<float*>(smem + NS * kHeavyStageBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * (kHeavyStageBytes + T * 4));
    uint64_t* empty = full + NS;

    const uint32_t item = blockIdx.x;
    const uint32_t d = order[d_begin + item / chunks];
    const uint32_t c = item % chunks;
    const uint32_t q0 = c * CHQ;
    const uint32_t nqc = min(static_cast<uint32_t>(CHQ), nq_total - q0);
    const uint32_t row_bytes = nqc * 16;
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint64_t ntiles = (ee - eb + T - 1) / T;
    const unsigned lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 32);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // producer warp
        for (uint64_t t = 0; t < ntiles; ++t) {
            const int s = static_cast<int>(t % NS);
            const uint32_t ph = static_cast<uint32_t>((t / NS) & 1);
            mbar_wait(&empty[s], ph ^ 1u);
            const uint64_t e0 = eb + t * T;
            const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - e0));
            if (lane == 0) mbar_expect_tx(&full[s], n * row_bytes);
            __syncwarp();
            for (uint32_t j = lane; j < n; j += 32) {
                const Edge ed = __ldg(edges + e0 + j);
                wbuf[s * T + j] = __uint_as_float(ed.y);
                bulk_g2s(buf + (static_cast<size_t>(s) * T + j) * CHQ, in + ed.x * ld_in + q0 * 4, row_bytes,
                         &full[s]);
            }
            mbar_arrive(&full[s]);
        }
        return;
    }
    // consumer warp: lane = float4 column of the chunk
    const Zs z = zs_of(zeros);
    const bool active = lane < nqc;
    const uint32_t col = (q0 + lane) * 4;
    float* orow = out + d * ld_out + col;
    Acc acc = acc_load(orow, col, dim, accumulate && active);
    for (uint64_t t = 0; t < ntiles; ++t) {
        const int s = static_cast<int>(t % NS);
        const uint32_t ph = static_cast<uint32_t>((t / NS) & 1);
        mbar_wait(&full[s], ph);
        const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - (eb + t * T)));
        if (active) {
            const float4* sb = buf + static_cast<size_t>(s) * T * CHQ + lane;
            const float* sw = wbuf + s * T;
            for (uint32_t j = 0; j < n; ++j) acc_step(acc, sw[j], sb[j * CHQ], z);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (active) acc_store(orow, col, dim, acc, z);
}

// Wide-row hubs on a whole-row TMA ring (tuning heavy_wide_pipe = 3): one
// CTA per hub destination, a producer warp that bulk-copies WHOLE rows (one
// cp.async.bulk of ld bytes per edge, every column chunk at once) into a
// kRingStages-deep shared-memory ring, and one consumer warp per 128-column
// chunk folding the staged rows in edge order (per column, ascending edge,
// fl(w*x) then fl(acc + .): bit-identical). A hub is a serial chain per
// column: its time is rows x the slower of the copy issue (~28 SM cycles per
// bulk op) and the fold; k_agg_wide_pipe gathers the same row five times
// (once per chunk warp) with 32 loads in flight per warp instead.
constexpr int kRingStages = 4;
constexpr int kRingRows = 8;  // rows per stage

__global__ void __launch_bounds__(288) k_agg_hub_ring(const uint64_t* __restrict__ ebeg,
                                                     const uint64_t* __restrict__ eend,
                                                     const Edge* __restrict__ edges,
                                                     const uint32_t* __restrict__ order, uint32_t d_begin,
                                                     const float* __restrict__ in, uint32_t ld_in_bytes,
                                                     float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                     int accumulate, float2 zeros, AggExt ext) {
    constexpr int NS = kRingStages, T = kRingRows;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t nwc = (blockDim.x >> 5) - 1;  // consumer warps = 128-column chunks
    unsigned char* buf = smem;                   // NS x T rows of ld_in_bytes
    float* wbuf = reinterpret_cast<float*>(smem + static_cast<size_t>(NS) * T * ld_in_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(wbuf + NS * T);
    uint64_t* empty = full + NS;
    const uint32_t d = order[d_begin + blockIdx.x];
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint64_t ntiles = (ee - eb + T - 1) / T;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int st = 0; st < NS; ++st) {
            mbar_init(&full[st], 32);
            mbar_init(&empty[st], nwc);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == nwc) {  // producer
        for (uint64_t t = 0; t < ntiles; ++t) {
            const int st = static_cast<int>(t % NS);
            const uint32_t ph = static_cast<uint32_t>((t / NS) & 1);
            mbar_wait(&empty[st], ph ^ 1u);
            const uint64_t e0 = eb + t * T;
            const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - e0));
            if (lane == 0) mbar_expect_tx(&full[st], n * ld_in_bytes);
            __syncwarp();
            if (lane < n) {
                const Edge ed = __ldg(edges + e0 + lane);
                wbuf[st * T + lane] = __uint_as_float(ed.y);
                bulk_g2s(buf + (static_cast<size_t>(st) * T + lane) * ld_in_bytes,
                         reinterpret_cast<const char*>(in) + static_cast<uint64_t>(ed.x) * ld_in_bytes, ld_in_bytes,
                         &full[st]);
            }
            mbar_arrive(&full[st]);
        }
        return;
    }
    const Zs z = zs_of(zeros);
    const uint32_t col = (warp * 32 + lane) * 4;
    const bool active = col < dim;
    const uint32_t row = ext_out_row(ext, d);
    float* orow = out + row * ld_out + col;
    Acc acc = acc_load(orow, col, dim, accumulate && active);
    for (uint64_t t = 0; t < ntiles; ++t) {
        const int st = static_cast<int>(t % NS);
        const uint32_t ph = static_cast<uint32_t>((t / NS) & 1);
        mbar_wait(&full[st], ph);
        const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - (eb + t * T)));
        if (active) {
            const unsigned char* sb = buf + static_cast<size_t>(st) * T * ld_in_bytes + col * 4;
            const float* sw = wbuf + st * T;
#pragma unroll
            for (int j = 0; j < T; ++j)
                if (j < static_cast<int>(n))
                    acc_step(acc, sw[j], *reinterpret_cast<const float4*>(sb + static_cast<size_t>(j) * ld_in_bytes),
                             z);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (active) acc_store_ext(orow, col, dim, acc, z, ext, d, row);
}

void launch_hub_ring(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order,
                     uint32_t d_begin, uint32_t nh, const float* in, uint64_t ld_in, float* out, uint64_t ld_out,
                     uint32_t dim, bool accumulate, cudaStream_t s, const AggExt& ext) {
    const uint32_t nq = (dim + 3) / 4, chunks = (nq + 31) / 32;
    const size_t smem = static_cast<size_t>(kRingStages) * kRingRows * ld_in * 4 + kRingStages * kRingRows * 4 +
                        2 * kRingStages * 8;
    PG_CUDA(cudaFuncSetAttribute(k_agg_hub_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_agg_hub_ring<<<nh, 32 * (chunks + 1), smem, s>>>(ebeg, eend, edges, order, d_begin, in,
                                                       static_cast<uint32_t>(ld_in * 4), out, ld_out, dim, accumulate,
                                                       kZeros, ext);
    PG_LAUNCH("k_agg_hub_ring");
}

template <int CHQ>
void launch_heavy(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order, uint32_t d_begin, uint32_t nh,
                  uint32_t nq, const float* in, uint64_t ld_in, float* out, uint64_t ld_out, uint32_t dim,
                  bool accumulate, cudaStream_t s) {
    static thread_local std::vector<char> attr_set;  // per device
    constexpr size_t smem = heavy_smem<CHQ>();
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    if (static_cast<int>(attr_set.size()) <= dev) attr_set.resize(dev + 1, 0);
    if (!attr_set[dev]) {
        PG_CUDA(cudaFuncSetAttribute(k_agg_heavy<CHQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        attr_set[dev] = 1;
    }
    const uint32_t chunks = (nq + CHQ - 1) / CHQ;
    k_agg_heavy<CHQ><<<nh * chunks, 64, smem, s>>>(ebeg, eend, edges, order, d_begin, chunks, nq, in, ld_in, out,
                                                   ld_out, dim, accumulate, kZeros);
    PG_LAUNCH("k_agg_heavy");
}

// ---- heavy destinations: cooperative LDG-staged double buffer -----------------
// One 256-thread CTA per (heavy destination, column chunk). All 8 warps
// gather the next tile of T edges' row chunks (128-bit LDG into registers,
// then shared memory) while warp 0's column lanes fold the current tile in
// ascending edge order. 32 KB per tile, ~64 KB in flight per CTA.
constexpr int kCoopTileBytes = 32768;

template <int CHQ>
__host__ __device__ constexpr int coop_T() {
    return kCoopTileBytes / (CHQ * 16);
}

constexpr int kCoopFoldBatch = 32;  // rows loaded ahead of their chain steps in the scalar fold

template <int CHQ, bool FILT>
__global__ void __launch_bounds__(256) k_agg_heavy_coop(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                       const Edge* __restrict__ edges,
                                                       const uint32_t* __restrict__ order, uint32_t d_begin,
                                                       uint32_t chunks, uint32_t nq_total,
                                                       const float* __restrict__ in, uint64_t ld_in,
                                                       float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                       int accumulate, float2 zeros, AggExt ext) {
    constexpr int T = coop_T<CHQ>();
    constexpr int PER = T * CHQ / 256;  // float4 gathers per thread per tile
    extern __shared__ __align__(128) unsigned char smem[];
    float4* tile = reinterpret_cast<float4*>(smem);                          // [2][T*CHQ]
    float* wt = reinterpret_cast<float*>(smem + 2 * kCoopTileBytes);         // [2][T]

    const uint32_t item = blockIdx.x;
    const uint32_t d = order[d_begin + item / chunks];
    if (FILT && !ext_dst_on(ext, d)) return;  // uniform per CTA
    const uint32_t c = item % chunks;
    const uint32_t q0 = c * CHQ;
    const uint32_t nqc = min(static_cast<uint32_t>(CHQ), nq_total - q0);
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint64_t ntiles = (ee - eb + T - 1) / T;
    const unsigned tid = threadIdx.x, lane = tid & 31;

    float4 r[PER];
    float rw[PER];
    // records of tile t+1 are loaded while tile t-1 folds and its rows are
    // issued while tile t folds: no record -> row round trip on the
    // critical path (ptxas otherwise serialises each record/row pair)
    Edge ed[PER];
    auto recs = [&](uint64_t t) {
        const uint64_t e0 = eb + t * T;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const unsigned idx = tid + 256u * k;
            const unsigned j = idx / CHQ, q = idx % CHQ;
            const bool ok = e0 + j < ee && q < nqc;
            ed[k] = ok ? __ldg(edges + e0 + j) : make_uint2(0xffffffffu, 0u);
        }
    };
    auto rows = [&]() {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const unsigned idx = tid + 256u * k;
            const unsigned q = idx % CHQ;
            const bool ok = ed[k].x != 0xffffffffu;
            const bool take = ok && (!FILT || ext_src_on(ext, ed[k].x));  // skipped: +-0 term
            r[k] = take ? ldg4(in + static_cast<uint64_t>(ed[k].x) * ld_in + (q0 + q) * 4)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
            rw[k] = __uint_as_float(ed[k].y);
        }
    };
    auto stash = [&](int b) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const unsigned idx = tid + 256u * k;
            tile[b * T * CHQ + idx] = r[k];
            if (idx % CHQ == 0) wt[b * T + idx / CHQ] = rw[k];
        }
    };

    const Zs z = zs_of(zeros);
    const uint32_t row = ext_out_row(ext, d);
    if constexpr (CHQ <= 8) {
        // rows of <= 32 floats: fold one SCALAR column per lane (FMUL + FADD
        // per edge) instead of a float4 on CHQ lanes (6 instructions per
        // edge on a quarter of the warp) — the hub's serial chain is the
        // critical path of the narrow top-layer SpMM
        const uint32_t scol = q0 * 4 + lane;
        const bool sowner = tid < 32 && scol < dim && lane < 4 * nqc;
        float* srow = out + row * ld_out + scol;
        float sacc = (sowner && accumulate) ? *srow : 0.f;
        if (ntiles) {
            recs(0);
            rows();
            stash(0);
            if (ntiles > 1) recs(1);
        }
        __syncthreads();
        for (uint64_t t = 0; t < ntiles; ++t) {
            const int b = static_cast<int>(t & 1);
            if (t + 1 < ntiles) {  // tile t+1's rows and tile t+2's records in flight during the fold
                rows();
                if (t + 2 < ntiles) recs(t + 2);
            }
            if (sowner) {
                const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - (eb + t * T)));
                const float* sb = reinterpret_cast<const float*>(tile + b * T * CHQ) + lane;
                const float* sw = wt + b * T;
                // kCoopFoldBatch rows' loads ahead of their chain steps: the
                // fold is the hub's serial chain (one FADD per edge), not the
                // LDS latency (Reddit top path 0.727 -> 0.635 ms at 16)
                constexpr int B = kCoopFoldBatch;
                uint32_t j = 0;
                for (; j + B <= n; j += B) {
                    float pw[B], px[B];
#pragma unroll
                    for (int u = 0; u < B; ++u) {
                        pw[u] = sw[j + u];
                        px[u] = sb[(j + u) * CHQ * 4];
                    }
#pragma unroll
                    for (int u = 0; u < B; ++u) sacc = __fadd_rn(sacc, __fmul_rn(pw[u], px[u]));
                }
                for (; j < n; ++j) sacc = __fadd_rn(sacc, __fmul_rn(sw[j], sb[j * CHQ * 4]));
            }
            if (t + 1 < ntiles) stash(b ^ 1);
            __syncthreads();
        }
        if (sowner) {
            float v = __fadd_rn(sacc, 0.f);
            if (ext.relu_pre) {
                const uint32_t prow = ext.pre_rows ? __ldg(ext.pre_rows + d) : row;
                v = ext.relu_pre[static_cast<uint64_t>(prow) * ext.ld_pre + scol] > 0.f ? v : 0.f;
            }
            *srow = v;
        }
    } else {
        const bool owner = tid < 32 && lane < nqc;
        const uint32_t col = (q0 + lane) * 4;
        float* orow = out + row * ld_out + col;
        Acc acc = acc_load(orow, col, dim, owner && accumulate);
        if (ntiles) {
            recs(0);
            rows();
            stash(0);
            if (ntiles > 1) recs(1);
        }
        __syncthreads();
        for (uint64_t t = 0; t < ntiles; ++t) {
            const int b = static_cast<int>(t & 1);
            if (t + 1 < ntiles) {  // tile t+1's rows and tile t+2's records in flight during the fold
                rows();
                if (t + 2 < ntiles) recs(t + 2);
            }
            if (owner) {
                const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - (eb + t * T)));
                const float4* sb = tile + b * T * CHQ + lane;
                const float* sw = wt + b * T;
                // 8 rows' loads ahead of their chain steps (the serial chain
                // is the hub's critical path, not the LDS latency)
                uint32_t j = 0;
                for (; j + 8 <= n; j += 8) {
                    float pw[8];
                    float4 px[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        pw[u] = sw[j + u];
                        px[u] = sb[(j + u) * CHQ];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc_step(acc, pw[u], px[u], z);
                }
                for (; j < n; ++j) acc_step(acc, sw[j], sb[j * CHQ], z);
            }
            if (t + 1 < ntiles) stash(b ^ 1);
            __syncthreads();
        }
        if (owner) acc_store_ext(orow, col, dim, acc, z, ext, d, row);
    }
}

template <int CHQ, bool FILT>
void launch_heavy_coop(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order, uint32_t d_begin,
                       uint32_t nh, uint32_t nq, const float* in, uint64_t ld_in, float* out, uint64_t ld_out,
                       uint32_t dim, bool accumulate, cudaStream_t s, const AggExt& ext) {
    static thread_local std::vector<char> attr_set;
    constexpr size_t smem = 2 * kCoopTileBytes + 2 * coop_T<CHQ>() * 4;
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    if (static_cast<int>(attr_set.size()) <= dev) attr_set.resize(dev + 1, 0);
    if (!attr_set[dev]) {
        PG_CUDA(cudaFuncSetAttribute(k_agg_heavy_coop<CHQ, FILT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        attr_set[dev] = 1;
    }
    const uint32_t chunks = (nq + CHQ - 1) / CHQ;
    k_agg_heavy_coop<CHQ, FILT><<<nh * chunks, 256, smem, s>>>(ebeg, eend, edges, order, d_begin, chunks, nq, in,
                                                               ld_in, out, ld_out, dim, accumulate, kZeros, ext);
    PG_LAUNCH("k_agg_heavy_coop");
}

// TMA bulk-copy ring for heavy narrow destinations (tuning "heavy_tma")
bool heavy_use_tma() { return tuning(kTuneHeavyTma) == 1; }

template <int CHQ>
void launch_heavy_any(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order, uint32_t d_begin,
                      uint32_t nh, uint32_t nq, const float* in, uint64_t ld_in, float* out, uint64_t ld_out,
                      uint32_t dim, bool accumulate, cudaStream_t s, const AggExt& ext) {
    if (ext.src_bits || ext.dst_bits)
        launch_heavy_coop<CHQ, true>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim, accumulate,
                                     s, ext);
    else if (heavy_use_tma() && !ext.any())
        launch_heavy<CHQ>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim, accumulate, s);
    else
        launch_heavy_coop<CHQ, false>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim,
                                      accumulate, s, ext);
}

// ---- CommitMode::Fast, group partitioned, atomic-free (PG_AGG_GROUPED) ----
// aggregate.hpp:84-115 with the groups as the unit of work and no global
// atomics. A CTA owns one schedule range: consecutive groups that hold whole
// destinations (or one slice of a hub destination's groups). Per (range,
// column chunk):
//  1. the range's edge records — contiguous, since its groups are — are
//     staged into shared memory with one cp.async.bulk (TMA bulk copy,
//     mbarrier completion; windows above kGrpEdgeCap stream from global);
//  2. a worker = LPD lanes (one float4 column each) takes one group at a
//     time (groups w, w + W, ...): per batch of U edges, records from shared
//     memory (broadcast LDS), U 128-bit row gathers in flight, ordered
//     separately-rounded accumulate into a zero scratch (aggregate.hpp:93),
//     the group's partial row into shared memory;
//  3. segmented reduction in group order: the head worker of each
//     destination's run adds its groups' partials in order and stores the
//     row once (out = init + sum, + 0) — or, for a hub slice, stores the
//     slice partial to its scratch slot; k_grp_fixup then adds a hub's
//     slices in slice order.
// Deterministic run to run; a destination with one group is bit-equal to
// the Deterministic kernel (same serial chain); across groups the sum is
// re-associated (Fast semantics, within the fp32 tolerance). gs sets the
// work unit and the partial-sum count, so the structure-aware gs selector
// shapes this schedule.
constexpr int kGrpEdgeCap = 4096;  // staged records per CTA (32 KB)

template <int LPD>
__host__ __device__ constexpr int grp_workers() { return 256 / LPD; }
template <int LPD>
__host__ __device__ constexpr int grp_gcap() { return 4 * grp_workers<LPD>(); }
template <int LPD>
constexpr size_t grp_smem() {
    return (kGrpEdgeCap + 2) * sizeof(Edge) + static_cast<size_t>(grp_gcap<LPD>()) * LPD * 16 +
           3ull * grp_gcap<LPD>() * 4 + 16;
}

template <int LPD, int U>
__global__ void __launch_bounds__(256, 4) k_agg_grp(const uint4* __restrict__ ranges, uint32_t nranges,
                                                   const uint64_t* __restrict__ gbeg, const uint64_t* __restrict__ gend,
                                                   const uint32_t* __restrict__ gdest, const Edge* __restrict__ edges,
                                                   const float* __restrict__ in, uint32_t ld_in_bytes,
                                                   float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                   int accumulate, float* __restrict__ scratch, uint64_t ld_scr,
                                                   float2 zeros, uint32_t zmask,
                                                   const uint64_t* __restrict__ seg_lo,
                                                   const uint64_t* __restrict__ seg_hi, int dyn) {
    constexpr int W = grp_workers<LPD>();
    __shared__ uint32_t next_group;  // dyn: groups handed out in order, one at a time
    constexpr int GCAP = grp_gcap<LPD>();
    extern __shared__ __align__(128) unsigned char smem[];
    Edge* recs = reinterpret_cast<Edge*>(smem);
    float4* part = reinterpret_cast<float4*>(smem + (kGrpEdgeCap + 2) * sizeof(Edge));
    uint32_t* sgb = reinterpret_cast<uint32_t*>(part + GCAP * LPD);
    uint32_t* sge = sgb + GCAP;
    uint32_t* sdst = sge + GCAP;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sdst + GCAP + (GCAP & 1));

    const uint32_t ri = blockIdx.x % nranges, ci = blockIdx.x / nranges;
    const uint4 r = ranges[ri];
    const uint64_t g0 = static_cast<uint64_t>(r.x) | (static_cast<uint64_t>(r.y) << 32);
    const uint32_t ng = r.z, slot = r.w;
    const uint64_t e0 = __ldg(gbeg + g0), e1 = __ldg(gend + g0 + ng - 1);
    const bool staged = e1 - e0 <= kGrpEdgeCap;
    const uint64_t ebase = staged ? (e0 & ~1ull) : e0;  // 16-byte aligned window start
    const unsigned tid = threadIdx.x;
    if (staged && tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == 0) next_group = W;
    for (uint32_t lg = tid; lg < ng; lg += 256) {
        uint64_t gb = __ldg(gbeg + g0 + lg), ge = __ldg(gend + g0 + lg);
        const uint32_t dd = __ldg(gdest + g0 + lg);
        if (seg_lo) {  // an L2-sized source segment: the group's part of it (maybe empty)
            gb = max(gb, __ldg(seg_lo + dd));
            ge = max(gb, min(ge, __ldg(seg_hi + dd)));
        }
        sgb[lg] = static_cast<uint32_t>(gb - ebase);
        sge[lg] = static_cast<uint32_t>(ge - ebase);
        sdst[lg] = dd;
    }
    __syncthreads();
    if (staged) {
        if (tid == 0) {
            // the edge stream is padded (kEdgePad): rounding the end up stays in bounds
            const uint32_t bytes = static_cast<uint32_t>(((e1 - ebase) * sizeof(Edge) + 15) & ~15ull);
            mbar_expect_tx(bar, bytes);
            bulk_g2s(recs, edges + ebase, bytes, bar);
            mbar_arrive(bar);
        }
        mbar_wait(bar, 0);
    }
    const Zs z = zs_of(zeros);
    const unsigned w = tid / LPD, sl = tid % LPD;
    const uint32_t col = (ci * LPD + sl) * 4;
    const bool active = col < dim;
    const char* base = reinterpret_cast<const char*>(in) + (active ? col : ci * LPD * 4u) * 4u;
    asm("mov.b64 %0, %0;" : "+l"(base));
    const uint32_t srecs = static_cast<uint32_t>(__cvta_generic_to_shared(recs));
    // a record: from the staged window (LDS, one broadcast per sub-warp) or,
    // for windows past kGrpEdgeCap, straight from global
    auto rec = [&](uint32_t i) -> Edge {
        if (staged) {
            Edge r;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(srecs + i * 8u));
            return r;
        }
        return ld_rec(edges + ebase + i);
    };
    const unsigned submask = LPD >= 32 ? 0xffffffffu : (((1u << LPD) - 1u) << (lane_id() & ~(LPD - 1u)));
    // the next group of this worker: static round robin, or (dyn) the CTA's
    // next unclaimed group — a worker that drew short groups takes more, so
    // the reduction barrier waits less (the partials, their order and the
    // result do not depend on which worker computed a group)
    auto next = [&](uint32_t lg) -> uint32_t {
        if (!dyn) return lg + W;
        uint32_t nl = 0;
        if (sl == 0) nl = atomicAdd(&next_group, 1u);
        return __shfl_sync(submask, nl, 0, LPD);
    };
    for (uint32_t lg = w; lg < ng; lg = next(lg)) {
        uint32_t e = sgb[lg];
        const uint32_t end = sge[lg];
        Acc acc{0ull, 0ull};  // the group's zero scratch (aggregate.hpp:93)
        for (; e + U <= end; e += U) {
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = rec(e + u);
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = ld_row(base, ed[u].x, ld_in_bytes);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
        }
        if (e < end) {
            const uint32_t n = end - e;
            Edge ed[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = rec(e + (u < static_cast<int>(n) ? u : n - 1));
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = ld_row(base, ed[u].x, ld_in_bytes);
            const Zs zz = batch_dep<U>(x, z, zmask);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < static_cast<int>(n)) acc_step(acc, __uint_as_float(ed[u].y), x[u], zz);
        }
        const float2 l = unpk2(acc.lo), h = unpk2(acc.hi);
        part[lg * LPD + sl] = make_float4(l.x, l.y, h.x, h.y);
    }
    __syncthreads();
    // segmented reduction over the range's groups, in group order
    for (uint32_t lg = w; lg < ng; lg += W) {
        const uint32_t d = sdst[lg];
        if (lg > 0 && sdst[lg - 1] == d) continue;  // not the head of its destination's run
        uint32_t last = lg;
        while (last + 1 < ng && sdst[last + 1] == d) ++last;
        float4 v = part[lg * LPD + sl];
        for (uint32_t k = lg + 1; k <= last; ++k) {
            const float4 p = part[k * LPD + sl];
            v.x = __fadd_rn(v.x, p.x);
            v.y = __fadd_rn(v.y, p.y);
            v.z = __fadd_rn(v.z, p.z);
            v.w = __fadd_rn(v.w, p.w);
        }
        if (!active) continue;
        const bool full = col + 3 < dim;
        if (slot != 0xffffffffu) {  // hub slice: its partial, combined by k_grp_fixup
            float* srow = scratch + slot * ld_scr + col;
            if (full) {
                *reinterpret_cast<float4*>(srow) = v;
            } else {
                srow[0] = v.x;
                if (col + 1 < dim) srow[1] = v.y;
                if (col + 2 < dim) srow[2] = v.z;
            }
            continue;
        }
        float* orow = out + d * ld_out + col;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (accumulate) {
            if (full) o = *reinterpret_cast<const float4*>(orow);
            else {
                o.x = orow[0];
                if (col + 1 < dim) o.y = orow[1];
                if (col + 2 < dim) o.z = orow[2];
            }
        }
        // out (+)= scratch (aggregate.hpp:102-103), then + 0 (aggregate.hpp:82)
        o.x = __fadd_rn(__fadd_rn(o.x, v.x), 0.f);
        o.y = __fadd_rn(__fadd_rn(o.y, v.y), 0.f);
        o.z = __fadd_rn(__fadd_rn(o.z, v.z), 0.f);
        o.w = __fadd_rn(__fadd_rn(o.w, v.w), 0.f);
        if (full) {
            __stcs(reinterpret_cast<float4*>(orow), o);
        } else {
            orow[0] = o.x;
            if (col + 1 < dim) orow[1] = o.y;
            if (col + 2 < dim) orow[2] = o.z;
        }
    }
}

// Hub destinations: out[d] = init + slice_0 + slice_1 + ... (slice order),
// + 0; and the rows of destinations without groups on overwrite.
template <int LPD>
__global__ void __launch_bounds__(256) k_grp_fixup(const uint4* __restrict__ hubs, uint32_t nhubs,
                                                  const uint32_t* __restrict__ empty, uint32_t nempty,
                                                  uint32_t chunks, const float* __restrict__ scratch, uint64_t ld_scr,
                                                  float* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                  int accumulate) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    const uint64_t nitems = static_cast<uint64_t>(nhubs + nempty) * chunks;
    if (item >= nitems) return;
    const uint32_t hi = static_cast<uint32_t>(item % (nhubs + nempty));
    const uint32_t ci = static_cast<uint32_t>(item / (nhubs + nempty));
    const uint32_t col = (ci * LPD + static_cast<uint32_t>(t % LPD)) * 4;
    if (col >= dim) return;
    const bool full = col + 3 < dim;
    if (hi >= nhubs) {  // a destination without groups: overwrite -> +0 row
        if (accumulate) return;
        float* orow = out + __ldg(empty + (hi - nhubs)) * ld_out + col;
        if (full) {
            *reinterpret_cast<float4*>(orow) = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            orow[0] = 0.f;
            if (col + 1 < dim) orow[1] = 0.f;
            if (col + 2 < dim) orow[2] = 0.f;
        }
        return;
    }
    const uint4 h = hubs[hi];
    float* orow = out + static_cast<uint64_t>(h.x) * ld_out + col;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (accumulate) {
        if (full) o = *reinterpret_cast<const float4*>(orow);
        else {
            o.x = orow[0];
            if (col + 1 < dim) o.y = orow[1];
            if (col + 2 < dim) o.z = orow[2];
        }
    }
    for (uint32_t k = 0; k < h.z; ++k) {
        const float* sr = scratch + static_cast<uint64_t>(h.y + k) * ld_scr + col;
        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
        if (full) p = *reinterpret_cast<const float4*>(sr);
        else {
            p.x = sr[0];
            if (col + 1 < dim) p.y = sr[1];
            if (col + 2 < dim) p.z = sr[2];
        }
        o.x = __fadd_rn(o.x, p.x);
        o.y = __fadd_rn(o.y, p.y);
        o.z = __fadd_rn(o.z, p.z);
        o.w = __fadd_rn(o.w, p.w);
    }
    o.x = __fadd_rn(o.x, 0.f);
    o.y = __fadd_rn(o.y, 0.f);
    o.z = __fadd_rn(o.z, 0.f);
    o.w = __fadd_rn(o.w, 0.f);
    if (full) {
        *reinterpret_cast<float4*>(orow) = o;
    } else {
        orow[0] = o.x;
        if (col + 1 < dim) orow[1] = o.y;
        if (col + 2 < dim) orow[2] = o.z;
    }
}

// Host: the schedule over the base CSR's offsets (groups of destination d
// are [off[d] + j gs, min(off[d] + (j+1) gs, off[d+1])), grouping.cpp:7-27).
// Ranges close before a destination that would push them past gcap groups
// or kGrpEdgeCap edges; a destination alone past either limit is a hub,
// cut into slices within both (one group per slice at least).
void build_grp_sched(const uint64_t* offsets_dev, uint32_t D, uint32_t gs, uint32_t workers, Groups::GrpSched& sc,
                     cudaStream_t s) {
    std::vector<uint64_t> off(static_cast<uint64_t>(D) + 1);
    PG_CUDA(cudaMemcpyAsync(off.data(), offsets_dev, off.size() * 8, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    const uint64_t gcap = 4ull * workers;
    std::vector<uint4> ranges, hubs;
    std::vector<uint32_t> empty;
    uint32_t nslots = 0;
    uint64_t g = 0, cur_g0 = 0, cur_ng = 0, cur_e = 0;
    auto close = [&] {
        if (cur_ng) ranges.push_back(make_uint4(static_cast<uint32_t>(cur_g0), static_cast<uint32_t>(cur_g0 >> 32),
                                                static_cast<uint32_t>(cur_ng), 0xffffffffu));
        cur_ng = cur_e = 0;
    };
    for (uint32_t d = 0; d < D; ++d) {
        const uint64_t deg = off[d + 1] - off[d];
        if (deg == 0) {
            empty.push_back(d);
            continue;
        }
        const uint64_t k = (deg + gs - 1) / gs;
        if (k > gcap || deg > static_cast<uint64_t>(kGrpEdgeCap)) {
            close();
            const uint32_t first = nslots;
            uint64_t j = 0;
            while (j < k) {
                uint64_t cnt = 0, e = 0;
                while (j + cnt < k && cnt < gcap) {
                    const uint64_t ge = std::min<uint64_t>(gs, deg - (j + cnt) * gs);
                    if (cnt && e + ge > static_cast<uint64_t>(kGrpEdgeCap)) break;
                    e += ge;
                    ++cnt;
                }
                ranges.push_back(make_uint4(static_cast<uint32_t>(g + j), static_cast<uint32_t>((g + j) >> 32),
                                            static_cast<uint32_t>(cnt), nslots++));
                j += cnt;
            }
            hubs.push_back(make_uint4(d, first, nslots - first, 0u));
            g += k;
            continue;
        }
        if (cur_ng + k > gcap || cur_e + deg > static_cast<uint64_t>(kGrpEdgeCap)) close();
        if (!cur_ng) cur_g0 = g;
        cur_ng += k;
        cur_e += deg;
        g += k;
    }
    close();
    sc.workers = workers;
    sc.nranges = static_cast<uint32_t>(ranges.size());
    sc.nhubs = static_cast<uint32_t>(hubs.size());
    sc.nslots = nslots;
    sc.nempty = static_cast<uint32_t>(empty.size());
    sc.ranges = DevBuf<uint4>(ranges.size(), s);
    sc.hubs = DevBuf<uint4>(hubs.size(), s);
    sc.empty = DevBuf<uint32_t>(empty.size(), s);
    if (!ranges.empty())
        PG_CUDA(cudaMemcpyAsync(sc.ranges.get(), ranges.data(), ranges.size() * 16, cudaMemcpyHostToDevice, s));
    if (!hubs.empty()) PG_CUDA(cudaMemcpyAsync(sc.hubs.get(), hubs.data(), hubs.size() * 16, cudaMemcpyHostToDevice, s));
    if (!empty.empty())
        PG_CUDA(cudaMemcpyAsync(sc.empty.get(), empty.data(), empty.size() * 4, cudaMemcpyHostToDevice, s));
    PG_CUDA(cudaStreamSynchronize(s));
}

template <int LPD>
void launch_grp(Groups& G, const Groups::GrpSched& sc, const Edge* edges, uint32_t chunks, const float* in,
                uint64_t ld_in, float* out, uint64_t ld_out, uint32_t dim, bool accumulate, cudaStream_t s,
                const uint64_t* seg_lo, const uint64_t* seg_hi) {
    static std::mutex mu;
    static std::vector<char> attr;
    constexpr size_t smem = grp_smem<LPD>();
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        if (static_cast<int>(attr.size()) <= dev) attr.resize(dev + 1, 0);
        if (!attr[dev]) {
            PG_CUDA(cudaFuncSetAttribute(k_agg_grp<LPD, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            attr[dev] = 1;
        }
    }
    const uint64_t ld_scr = (static_cast<uint64_t>(dim) + 3) & ~3ull;
    DevBuf<float> scratch(static_cast<uint64_t>(sc.nslots) * ld_scr, s);
    if (sc.nranges) {
        k_agg_grp<LPD, 8><<<sc.nranges * chunks, 256, smem, s>>>(
            sc.ranges.get(), sc.nranges, G.gbegin.get(), G.gend.get(), G.gdest.get(), edges, in,
            static_cast<uint32_t>(ld_in * 4), out, ld_out, dim, accumulate, scratch.get(), ld_scr, kZeros, 0u, seg_lo,
            seg_hi, static_cast<int>(tuning(kTuneGrpDynamic)));
        PG_LAUNCH("k_agg_grp");
    }
    const uint64_t fix = static_cast<uint64_t>(sc.nhubs + (accumulate ? 0 : sc.nempty)) * chunks;
    if (fix) {
        k_grp_fixup<LPD><<<grid_for(fix * LPD, 256), 256, 0, s>>>(sc.hubs.get(), sc.nhubs, sc.empty.get(),
                                                                accumulate ? 0u : sc.nempty, chunks, scratch.get(),
                                                                ld_scr, out, ld_out, dim, accumulate);
        PG_LAUNCH("k_grp_fixup");
    }
}

// ---- aggregate_pull<double> (aggregate.hpp:56-122 with T = double) --------
// The reference's default precision (run_config.hpp:53 Precision::F64): per
// destination and column, ascending edge order, acc = fl(acc + fl(w * x))
// in f64 with w the path's f64 weight unconverted (static_cast<double>),
// separately rounded (__dmul_rn / __dadd_rn: no contraction, like the
// default-flag x86-64 build), then acc + 0. A (sub-)warp owns (destination,
// column chunk), a lane a double2 (one 128-bit gather per edge per lane);
// U edges in flight. Source id of edge e: src[e * src_stride] (the
// gather-folded parent position, the local id, or the vertex id).
// The f64 twin of batch_dep: the first weight of a batch XOR a runtime-zero
// function of all its gathered rows (zmask = 0), so the chain's first DMUL
// waits for every gather and ptxas issues them all back to back.
template <int N>
__device__ __forceinline__ double f64_batch_dep(double w0, const double2 (&x)[N], unsigned long long zmask) {
    unsigned long long all = 0;
#pragma unroll
    for (int u = 0; u < N; ++u) all ^= static_cast<unsigned long long>(__double_as_longlong(x[u].x));
    return __longlong_as_double(static_cast<long long>(static_cast<unsigned long long>(__double_as_longlong(w0)) ^
                                                       (all & zmask)));
}

template <int LPD, int U>
__global__ void __launch_bounds__(256) k_agg_f64(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                const uint32_t* __restrict__ src,
                                                uint32_t src_stride, const double* __restrict__ w,
                                                const uint32_t* __restrict__ order, uint64_t n_items, uint32_t chunks,
                                                uint32_t n_front, const double* __restrict__ in, uint64_t ld_in,
                                                double* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                int accumulate, unsigned long long zmask) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    if (item >= n_items) return;
    // chunk-major, except the first n_front destinations (the longest lists,
    // at the head of the degree order): destination-major ahead of the rest,
    // so every chunk of them starts at the beginning of the pass
    const uint64_t nd = n_items / chunks;
    uint32_t d, ci;
    if (item < static_cast<uint64_t>(n_front) * chunks) {
        d = __ldg(order + item / chunks);
        ci = static_cast<uint32_t>(item % chunks);
    } else {
        const uint64_t r = item - static_cast<uint64_t>(n_front) * chunks, nr = nd - n_front;
        d = __ldg(order + n_front + r % nr);
        ci = static_cast<uint32_t>(r / nr);
    }
    const uint32_t col = (ci * LPD + static_cast<uint32_t>(t % LPD)) * 2;
    const bool active = col < dim;
    const bool pair = col + 1 < dim;
    uint64_t e = __ldg(ebeg + d);
    const uint64_t end = __ldg(eend + d);
    const double* icol = in + (active ? col : 0u);
    double* orow = out + d * ld_out + col;
    double a0 = 0.0, a1 = 0.0;
    if (accumulate && active) {
        a0 = orow[0];
        if (pair) a1 = orow[1];
    }
    for (; e + U <= end; e += U) {
        uint32_t sr[U];
        double ww[U];
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            sr[u] = __ldg(src + (e + u) * src_stride);
            ww[u] = __ldg(w + e + u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldg(reinterpret_cast<const double2*>(icol + sr[u] * ld_in));
        ww[0] = f64_batch_dep<U>(ww[0], x, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a0 = __dadd_rn(a0, __dmul_rn(ww[u], x[u].x));
            a1 = __dadd_rn(a1, __dmul_rn(ww[u], x[u].y));
        }
    }
    if (e < end) {  // remainder (< U edges) as one batch: all gathers in flight
        const uint32_t n = static_cast<uint32_t>(end - e);
        uint32_t sr[U];
        double ww[U];
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t eu = e + (u < static_cast<int>(n) ? u : 0);
            sr[u] = __ldg(src + eu * src_stride);
            ww[u] = __ldg(w + eu);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            x[u] = u < static_cast<int>(n) ? __ldg(reinterpret_cast<const double2*>(icol + sr[u] * ld_in))
                                           : make_double2(0.0, 0.0);
        ww[0] = f64_batch_dep<U>(ww[0], x, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(n)) {
                a0 = __dadd_rn(a0, __dmul_rn(ww[u], x[u].x));
                a1 = __dadd_rn(a1, __dmul_rn(ww[u], x[u].y));
            }
    }
    if (!active) return;
    orow[0] = __dadd_rn(a0, 0.0);
    if (pair) orow[1] = __dadd_rn(a1, 0.0);
}

// Wide f64 rows with 256-bit gathers (ld.global.nc.v4.f64, one 32-byte load
// per lane and edge): 16 lanes of 4 doubles own a 64-double chunk, two items
// per warp, so a record load (source id + f64 weight) serves two items.
// Same items (chunk-major), per-column chains and bits as k_agg_f64<32>.
// Needs a 32-byte aligned input and a 4-double row pitch.
__device__ __forceinline__ void ld_row4d(const double* p, double2& a, double2& b) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
                 : "l"(p));
}
template <int U>
__global__ void __launch_bounds__(256) k_agg_f64v(const uint64_t* __restrict__ ebeg, const uint64_t* __restrict__ eend,
                                                 const uint32_t* __restrict__ src, uint32_t src_stride,
                                                 const double* __restrict__ w, const uint32_t* __restrict__ order,
                                                 uint64_t n_items, uint32_t chunks, const double* __restrict__ in,
                                                 uint64_t ld_in, double* __restrict__ out, uint64_t ld_out,
                                                 uint32_t dim, int accumulate, unsigned long long zmask) {
    constexpr int LPD = 16;
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t item = t / LPD;
    if (item >= n_items) return;
    const uint64_t nd = n_items / chunks;
    const uint32_t d = __ldg(order + item % nd);
    const uint32_t ci = static_cast<uint32_t>(item / nd);  // chunk-major
    const uint32_t col = ci * 64u + static_cast<uint32_t>(t % LPD) * 4u;
    const bool active = col < dim;
    uint64_t e = __ldg(ebeg + d);
    const uint64_t end = __ldg(eend + d);
    const double* icol = in + (active ? col : ci * 64u);
    double* orow = out + d * ld_out + col;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (accumulate && active)
        for (int k = 0; k < 4; ++k)
            if (col + k < dim) a[k] = orow[k];
    auto step = [&](double wv, const double2& x0, const double2& x1) {
        a[0] = __dadd_rn(a[0], __dmul_rn(wv, x0.x));
        a[1] = __dadd_rn(a[1], __dmul_rn(wv, x0.y));
        a[2] = __dadd_rn(a[2], __dmul_rn(wv, x1.x));
        a[3] = __dadd_rn(a[3], __dmul_rn(wv, x1.y));
    };
    for (; e + U <= end; e += U) {
        uint32_t sr[U];
        double ww[U];
        double2 x[2 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            sr[u] = __ldg(src + (e + u) * src_stride);
            ww[u] = __ldg(w + e + u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) ld_row4d(icol + sr[u] * ld_in, x[2 * u], x[2 * u + 1]);
        ww[0] = f64_batch_dep<2 * U>(ww[0], x, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u) step(ww[u], x[2 * u], x[2 * u + 1]);
    }
    if (e < end) {
        const uint32_t n = static_cast<uint32_t>(end - e);
        uint32_t sr[U];
        double ww[U];
        double2 x[2 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t eu = e + (u < static_cast<int>(n) ? u : 0);
            sr[u] = __ldg(src + eu * src_stride);
            ww[u] = __ldg(w + eu);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < static_cast<int>(n)) ld_row4d(icol + sr[u] * ld_in, x[2 * u], x[2 * u + 1]);
            else x[2 * u] = x[2 * u + 1] = make_double2(0.0, 0.0);
        }
        ww[0] = f64_batch_dep<2 * U>(ww[0], x, zmask);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(n)) step(ww[u], x[2 * u], x[2 * u + 1]);
    }
    if (!active) return;
    for (int k = 0; k < 4; ++k)
        if (col + k < dim) orow[k] = __dadd_rn(a[k], 0.0);
}

// aggregate_pull<double> hub destinations (the longest lists): a CTA per
// (hub, CW-column chunk). All 256 threads gather a tile of T edges' row
// slices into shared memory (double-buffered: tile t+1's rows in flight
// while tile t folds); CW owner threads then run each column's serial
// chain over the tile in edge order — the reference's order, so the same
// bits as k_agg_f64, with the gathers no longer one latency per batch of 8.
template <int CW>
__global__ void __launch_bounds__(256) k_agg_f64_hub(const uint64_t* __restrict__ ebeg,
                                                    const uint64_t* __restrict__ eend,
                                                    const uint32_t* __restrict__ src, uint32_t src_stride,
                                                    const double* __restrict__ w, const uint32_t* __restrict__ order,
                                                    uint32_t chunks, const double* __restrict__ in, uint64_t ld_in,
                                                    double* __restrict__ out, uint64_t ld_out, uint32_t dim,
                                                    int accumulate) {
    constexpr int H = CW / 2;             // double2 per row slice
    constexpr int T = 16384 / (CW * 8);   // edges per tile (16 KB of rows)
    constexpr int PER = T * H / 256;      // double2 gathers per thread per tile
    __shared__ __align__(16) double2 tile[2][T * H];
    __shared__ double wt[2][T];
    const uint32_t d = order[blockIdx.x / chunks];
    const uint32_t c0 = (blockIdx.x % chunks) * CW;
    const uint64_t eb = ebeg[d], ee = eend[d];
    const uint64_t ntiles = (ee - eb + T - 1) / T;
    const unsigned tid = threadIdx.x;
    double2 r[PER];
    double rw[PER];
    auto rows = [&](uint64_t t) {
        const uint64_t e0 = eb + t * T;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const unsigned idx = tid + 256u * k;
            const unsigned j = idx / H, q = idx % H;
            const uint32_t col = c0 + 2 * q;
            if (e0 + j < ee) {
                const uint32_t sr = __ldg(src + (e0 + j) * src_stride);
                r[k] = col < dim ? __ldg(reinterpret_cast<const double2*>(in + static_cast<uint64_t>(sr) * ld_in + col))
                                 : make_double2(0.0, 0.0);
                rw[k] = __ldg(w + e0 + j);
            } else {
                r[k] = make_double2(0.0, 0.0);
                rw[k] = 0.0;
            }
        }
    };
    auto stash = [&](int b) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const unsigned idx = tid + 256u * k;
            tile[b][idx] = r[k];
            if (idx % H == 0) wt[b][idx / H] = rw[k];
        }
    };
    const uint32_t col = c0 + tid;
    const bool owner = tid < CW && col < dim;
    double* orow = out + static_cast<uint64_t>(d) * ld_out + col;
    double acc = owner && accumulate ? *orow : 0.0;
    if (ntiles) {
        rows(0);
        stash(0);
    }
    __syncthreads();
    for (uint64_t t = 0; t < ntiles; ++t) {
        const int b = static_cast<int>(t & 1);
        if (t + 1 < ntiles) rows(t + 1);
        if (owner) {
            const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(T), ee - (eb + t * T)));
            const double* sb = reinterpret_cast<const double*>(tile[b]) + tid;
            const double* sw = wt[b];
            uint32_t j = 0;
            for (; j + 8 <= n; j += 8) {
                double pw[8], px[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    pw[u] = sw[j + u];
                    px[u] = sb[(j + u) * CW];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(pw[u], px[u]));
            }
            for (; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(sw[j], sb[j * CW]));
        }
        if (t + 1 < ntiles) stash(b ^ 1);
        __syncthreads();
    }
    if (owner) *orow = __dadd_rn(acc, 0.0);
}

struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

// one side stream per (device, calling stream): two calls running
// concurrently on different streams (the host pipeline's hub chunk beside
// the other chunks) must not queue their hub kernels behind each other
SideStream& side_stream(cudaStream_t caller) {
    struct Entry {
        int dev;
        cudaStream_t caller;
        SideStream ss;
    };
    static thread_local std::deque<Entry> per;  // stable references
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    for (auto& e : per)
        if (e.dev == dev && e.caller == caller) return e.ss;
    // bounded: past 16 (device, stream) pairs every new caller shares the
    // device's first side stream (still correct, only serialised)
    int same_dev = 0;
    for (auto& e : per) same_dev += e.dev == dev;
    if (same_dev >= 16)
        for (auto& e : per)
            if (e.dev == dev) return e.ss;
    per.push_back(Entry{dev, caller, SideStream{}});
    SideStream& ss = per.back().ss;
    int prio = 0;  // the caller's priority (a high-priority caller's hubs stay high)
    if (caller) PG_CUDA(cudaStreamGetPriority(caller, &prio));
    PG_CUDA(cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, prio));
    PG_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    PG_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
    return ss;
}

// 256-bit gathers: 1 on, 0 off, 2 (default) from 2^21 edges per call. On
// small calls (arxiv, 0.6-1.1M edges: 0.24 -> 0.36 ms) the longest lists —
// twice the columns per lane — set the length; on the large ones the halved
// load count wins (Reddit layer 0 15.65 -> 15.15 ms, products 4.77 -> 4.13)
// Narrow rows (2 / 4 / 8 lanes of 8 floats) only when forced: the Reddit top
// path (width 16, 75.6M edges) runs 0.61 -> 0.94 ms with them.
bool vec8_on(const AggExt& ext, int lpd) {
    const int64_t v = tuning(kTuneVec8);
    return v == 1 || (v == 2 && lpd == 32 && ext.n_edges >= (1ull << 21));
}

template <int LPD, int U>
void launch_vec4(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order, uint32_t d_begin,
                 uint32_t nd, uint32_t chunks, const float* in, uint64_t ld_in, float* out, uint64_t ld_out,
                 uint32_t dim, bool accumulate, cudaStream_t s, const AggExt& ext, uint32_t n_front = 0) {
    const uint64_t items = static_cast<uint64_t>(nd) * chunks;
    int cm = chunks > 1 && tuning(kTuneChunkMajor) ? 1 : 0;
    if (cm && n_front) cm = 2 + static_cast<int>(std::min(n_front, nd));
    // gather load flavour (tuning "ld_cg", see ld_row): measured on the
    // Reddit layer-0 path, the default read-only L1-allocating load is best
    const int ldm = static_cast<int>(tuning(kTuneLdCg));
    const unsigned grid = grid_for(items * LPD, 256);
    const uint32_t ldb = static_cast<uint32_t>(ld_in * 4);
    if constexpr (U <= 8 && LPD >= 4) {
        if (vec8_on(ext, LPD) && ldb % 32 == 0 && reinterpret_cast<uintptr_t>(in) % 32 == 0) {
            constexpr int U8 = U / 2;
            const unsigned g8 = grid_for(items * (LPD / 2), 256);
            const int64_t vu8 = tuning(kTuneVec8U);
            if constexpr (LPD == 32 && U == 8) {
                // edges per batch per half-warp (tuning vec8_u; 0 = 4)
                if (vu8 == 3 && !(ext.src_bits || ext.dst_bits)) {
                    k_agg_vec8<16, 3, false><<<g8, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in,
                                                                ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm, ext);
                    PG_LAUNCH("k_agg_vec8");
                    return;
                }
                if (vu8 == 6 && !(ext.src_bits || ext.dst_bits)) {
                    k_agg_vec8<16, 6, false><<<g8, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in,
                                                                ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm, ext);
                    PG_LAUNCH("k_agg_vec8");
                    return;
                }
            }
            if (ext.src_bits || ext.dst_bits)
                k_agg_vec8<LPD / 2, U8, true><<<g8, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in,
                                                                 ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm, ext);
            else
                k_agg_vec8<LPD / 2, U8, false><<<g8, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks,
                                                                  in, ldb, out, ld_out, dim, accumulate, kZeros, 0u,
                                                                  cm, ext);
            PG_LAUNCH("k_agg_vec8");
            return;
        }
    }
    if (ext.src_bits || ext.dst_bits)
        k_agg_vec4<LPD, U, true><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                      ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (LPD == 32 && tuning(kTuneRecWindow) == 2)
        k_agg_vec4<LPD, U, false, 8, true><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in,
                                                                ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (LPD >= 16 && tuning(kTuneRecWindow) == 1)
        k_agg_vec4<LPD, U, false, 0, true><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in,
                                                                ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 2)
        k_agg_vec4<LPD, U, false, 2><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 3)
        k_agg_vec4<LPD, U, false, 3><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 4)
        k_agg_vec4<LPD, U, false, 4><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 5)
        k_agg_vec4<LPD, U, false, 5><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 6)
        k_agg_vec4<LPD, U, false, 6><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 7)
        k_agg_vec4<LPD, U, false, 7><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (ldm == 9)
        k_agg_vec4<LPD, U, false, 9><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                          ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    else if (LPD == 32 && U == 8 && tuning(kTuneVecWindow) > 0)
        k_agg_vec4w<8><<<grid_for(items * LPD, 512), 512, 0, s>>>(
            ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm,
            static_cast<uint32_t>(tuning(kTuneVecWindow)), ext);
    else if (LPD == 32 && U == 8 && tuning(kTuneVecBlock) == 1024)
        // 32 destinations of one column chunk per CTA, started together: the
        // CTA's warps walk their (degree-sorted, similar) lists in step, so
        // shared sources hit in L1
        k_agg_vec4<LPD, U, false, 0, false, 1024><<<grid_for(items * LPD, 1024), 1024, 0, s>>>(
            ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm,
            ext);
    else if (LPD == 32 && U == 8 && tuning(kTuneVecBlock) == 512)
        k_agg_vec4<LPD, U, false, 0, false, 512><<<grid_for(items * LPD, 512), 512, 0, s>>>(
            ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out, ld_out, dim, accumulate, kZeros, 0u, cm,
            ext);
    else
        k_agg_vec4<LPD, U, false><<<grid, 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks, in, ldb, out,
                                                       ld_out, dim, accumulate, kZeros, 0u, cm, ext);
    PG_LAUNCH("k_agg_vec4");
}

__global__ void k_relu_backward(const float* __restrict__ g, uint64_t ldg, const float* __restrict__ pre,
                                uint64_t ldp, float* __restrict__ out, uint64_t ldo, uint64_t rows,
                                uint64_t cols) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= rows * cols) return;
    const uint64_t r = i / cols, c = i % cols;
    out[r * ldo + c] = pre[r * ldp + c] > 0.f ? g[r * ldg + c] : 0.f;
}

// blockIdx.y strides rows, x covers columns: no 64-bit div/mod per element
__global__ void k_copy_rows(const float* __restrict__ src, uint64_t lds, float* __restrict__ dst, uint64_t ldd,
                            uint64_t rows, uint32_t cols) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    // evict-first loads and stores: the host pipeline repacks segments while
    // the SpMM keeps its gather working set in L2
    for (uint64_t r = blockIdx.y; r < rows; r += gridDim.y) __stcs(dst + r * ldd + c, __ldcs(src + r * lds + c));
}

__global__ void k_gather_rows(const float* __restrict__ src, uint64_t lds, const uint32_t* __restrict__ ids,
                              uint64_t k, float* __restrict__ out, uint64_t ldo, uint64_t cols) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= k * cols) return;
    const uint64_t r = i / cols, c = i % cols;
    out[r * ldo + c] = src[static_cast<uint64_t>(ids[r]) * lds + c];
}

}  // namespace

void aggregate_seq(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* dlist,
                   const SeqTable& tab, uint64_t n_items, uint32_t chunks, const float* in, uint64_t ld_in, float* out,
                   uint64_t ld_out, uint32_t dim, bool accumulate, unsigned* counters, cudaStream_t s) {
    if (!n_items) return;
    k_agg_vec4_seq<8><<<grid_for(n_items * 32, 256), 256, 0, s>>>(ebeg, eend, edges, dlist, tab, n_items, chunks, in,
                                                                 static_cast<uint32_t>(ld_in * 4), out, ld_out, dim,
                                                                 accumulate, kZeros, 0u, counters);
    PG_LAUNCH("k_agg_vec4_seq");
}

void aggregate_det(const uint64_t* ebeg, const uint64_t* eend, const Edge* edges, const uint32_t* order, uint32_t D,
                   uint32_t d_begin, uint32_t d_end, uint32_t n_heavy, const float* in, uint64_t ld_in,
                   float* out, uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s, const AggExt& ext) {
    (void)D;
    if (d_end <= d_begin || dim == 0) return;
    uint32_t nd = d_end - d_begin;
    const uint32_t dim32 = static_cast<uint32_t>(dim);
    const bool vec = (ld_in % 4 == 0) && (ld_out % 4 == 0) &&
                     (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0) && ld_in >= ((dim + 3) & ~3ull) &&
                     ld_in < (1ull << 30) && (!ext.relu_pre || ext.ld_pre >= dim);
    const bool filt = ext.src_bits || ext.dst_bits;
    const uint32_t nq = (dim32 + 3) / 4;
    // heavy wide destinations (k_agg_wide_lat) take no activity filter: the
    // filtered (if-else) traversal keeps them on the main kernel
    const uint32_t nh = vec && !(filt && nq > 16) ? std::min(n_heavy, nd) : 0;
    // tuning "hub_inline": wide-row hubs stay in the main kernel as its
    // destination-major front instead of a concurrent side kernel
    const bool inline_hubs =
        nh && nq > 16 && !filt && !ext.side_hubs && tuning(kTuneHubInline) != 0 && !row_kernel_on(dim32);
    if (nh && !inline_hubs) {
        // heavy prefix of the degree order on a forked stream, concurrent
        // with the main kernel over the rest; joined back into s
        SideStream& ss = side_stream(s);
        PG_CUDA(cudaEventRecord(ss.fork, s));
        PG_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
        if (nq > 16) {
            // wide rows: latency-optimised warp kernel, 32 row gathers in
            // flight per lane, 5 column-chunk warps per 602-wide destination
            const uint32_t chunks = (nq + 31) / 32;
            const uint64_t items = static_cast<uint64_t>(nh) * chunks;
            // whole-row TMA ring: rows up to 8 chunks (1024 floats) and a
            // ring that fits the 227-KB shared memory
            if (tuning(kTuneHeavyWidePipe) == 4) {
                // cooperative tiles: all eight warps of a (hub, 128-column
                // chunk) CTA gather 64-row tiles into shared memory while
                // warp 0 folds the previous one
                launch_heavy_coop<32, false>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim32,
                                             accumulate, ss.s, ext);
            } else if (tuning(kTuneHeavyWidePipe) == 3 && chunks <= 8 &&
                static_cast<uint64_t>(kRingStages) * kRingRows * ld_in * 4 <= (200u << 10) &&
                (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
                launch_hub_ring(ebeg, eend, edges, order, d_begin, nh, in, ld_in, out, ld_out, dim32, accumulate, ss.s,
                                ext);
            } else if (tuning(kTuneHeavyWidePipe) == 5 && ld_in % 2 == 0 && (reinterpret_cast<uintptr_t>(in) & 7) == 0) {
                const uint32_t ch2 = (dim32 + 63) / 64;
                const uint64_t it2 = static_cast<uint64_t>(nh) * ch2;
                k_agg_wide_pipe2<32><<<grid_for(it2 * 32, 64), 64, 0, ss.s>>>(
                    ebeg, eend, edges, order, d_begin, it2, ch2, in, static_cast<uint32_t>(ld_in * 4), out, ld_out,
                    dim32, accumulate, 0u, ext);
                PG_LAUNCH("k_agg_wide_pipe2");
            } else if (tuning(kTuneHeavyWidePipe) >= 1) {
                k_agg_wide_pipe<16><<<grid_for(items * 32, 64), 64, 0, ss.s>>>(
                    ebeg, eend, edges, order, d_begin, items, chunks, in, static_cast<uint32_t>(ld_in * 4), out,
                    ld_out, dim32, accumulate, 0u, ext, tuning(kTuneHeavyWidePipe) == 2 ? 1 : 0);
                PG_LAUNCH("k_agg_wide_pipe");
            } else {
                k_agg_wide_lat<32><<<grid_for(items * 32, 256), 256, 0, ss.s>>>(
                    ebeg, eend, edges, order, d_begin, items, chunks, in, ld_in, out, ld_out, dim32, accumulate, 0u,
                    ext);
                PG_LAUNCH("k_agg_wide_lat");
            }
        } else if (tuning(kTuneHeavyNarrow) == 1 && !heavy_use_tma()) {
            // narrow rows: scalar column per lane, 32-edge batches in flight
            const uint32_t chunks = (dim32 + 31) / 32;
            const uint64_t items = static_cast<uint64_t>(nh) * chunks;
            if (filt)
                k_agg_narrow_lat<true><<<grid_for(items * 32, 256), 256, 0, ss.s>>>(
                    ebeg, eend, edges, order, d_begin, items, chunks, in, ld_in, out, ld_out, dim32, accumulate, 0u,
                    ext);
            else
                k_agg_narrow_lat<false><<<grid_for(items * 32, 256), 256, 0, ss.s>>>(
                    ebeg, eend, edges, order, d_begin, items, chunks, in, ld_in, out, ld_out, dim32, accumulate, 0u,
                    ext);
            PG_LAUNCH("k_agg_narrow_lat");
        } else if (nq > 8)
            launch_heavy_any<16>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim32, accumulate,
                                 ss.s, ext);
        else if (nq > 4)
            launch_heavy_any<8>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim32, accumulate,
                                ss.s, ext);
        else
            launch_heavy_any<4>(ebeg, eend, edges, order, d_begin, nh, nq, in, ld_in, out, ld_out, dim32, accumulate,
                                ss.s, ext);
        PG_CUDA(cudaEventRecord(ss.join, ss.s));
        d_begin += nh;
        nd -= nh;
        if (nd) aggregate_det(ebeg, eend, edges, order, D, d_begin, d_begin + nd, 0, in, ld_in, out, ld_out, dim,
                              accumulate, s, ext);
        PG_CUDA(cudaStreamWaitEvent(s, ss.join, 0));
        return;
    }
    if (!vec) {
        const uint32_t chunks = (dim32 + 31) / 32;
        const uint64_t items = static_cast<uint64_t>(nd) * chunks;
        k_agg_scalar<8><<<grid_for(items * 32, 256), 256, 0, s>>>(ebeg, eend, edges, order, d_begin, items, chunks,
                                                                 in, ld_in, out, ld_out, dim32, accumulate, ext);
        PG_LAUNCH("k_agg_scalar");
        return;
    }
    if (nq > 16 && !filt && row_kernel_on(dim32)) {
        const int u = static_cast<int>(tuning(kTuneRowU));
        switch ((nq + 31) / 32) {
            case 2: launch_row_ns<2>(ebeg, eend, edges, order, d_begin, nd, in, ld_in, out, ld_out, dim32, accumulate, s, ext, u); break;
            case 3: launch_row_ns<3>(ebeg, eend, edges, order, d_begin, nd, in, ld_in, out, ld_out, dim32, accumulate, s, ext, u); break;
            case 4: launch_row_ns<4>(ebeg, eend, edges, order, d_begin, nd, in, ld_in, out, ld_out, dim32, accumulate, s, ext, u); break;
            case 5: launch_row_ns<5>(ebeg, eend, edges, order, d_begin, nd, in, ld_in, out, ld_out, dim32, accumulate, s, ext, u); break;
            default: launch_row_ns<6>(ebeg, eend, edges, order, d_begin, nd, in, ld_in, out, ld_out, dim32, accumulate, s, ext, u); break;
        }
        return;
    }
    if (nq > 16) {
        const uint32_t chunks = (nq + 31) / 32;
        int64_t vu = tuning(kTuneVecU);
        // very short lists: the remainder batch is the whole item and 4 slots
        // waste less (products top path, 4.1 edges per destination: 1.50 ->
        // 1.23 ms); from ~8 on, 8 in flight wins (arxiv layer 0 at 8.6:
        // 0.114 vs 0.155 ms; Reddit layer 0 at 492: 15.5 vs 19.0 ms)
        if (vu == 0) vu = ext.avg_degree && ext.avg_degree < 8 ? 4 : 8;  // auto (default)
        if (tuning(kTuneWideLpd) == 16)  // 64-float chunks: half the per-pass source working set
            launch_vec4<16, 8>(ebeg, eend, edges, order, d_begin, nd, (nq + 15) / 16, in, ld_in, out, ld_out, dim32,
                               accumulate, s, ext);
        else if (vu == 4)
            launch_vec4<32, 4>(ebeg, eend, edges, order, d_begin, nd, chunks, in, ld_in, out, ld_out, dim32, accumulate,
                               s, ext);
        else if (vu == 16)
            launch_vec4<32, 16>(ebeg, eend, edges, order, d_begin, nd, chunks, in, ld_in, out, ld_out, dim32,
                                accumulate, s, ext);
        else
            launch_vec4<32, 8>(ebeg, eend, edges, order, d_begin, nd, chunks, in, ld_in, out, ld_out, dim32, accumulate,
                               s, ext, inline_hubs ? nh : 0);
    } else if (nq > 8) {
        launch_vec4<16, 8>(ebeg, eend, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s, ext);
    } else if (nq > 4) {
        launch_vec4<8, 8>(ebeg, eend, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s, ext);
    } else if (tuning(kTuneNarrowU) == 16) {
        launch_vec4<4, 16>(ebeg, eend, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s, ext);
    } else {
        launch_vec4<4, 8>(ebeg, eend, edges, order, d_begin, nd, 1, in, ld_in, out, ld_out, dim32, accumulate, s, ext);
    }
}

void aggregate_groups(const uint64_t* gbeg, const uint64_t* gend, const uint32_t* gdest, const uint64_t* dest_groups,
                      uint32_t D, uint64_t G, const Edge* edges, const float* in, uint64_t ld_in, float* out,
                      uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s) {
    if (dim == 0) return;
    if (!accumulate && D) PG_CUDA(cudaMemset2DAsync(out, ld_out * 4, 0, dim * 4, D, s));
    if (G == 0) return;
    const bool vec = (ld_in % 4 == 0) && (ld_out % 4 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0) && ld_in >= ((dim + 3) & ~3ull) &&
                     ld_in < (1ull << 30);
    if (!vec) fail(kConfig, "grouped aggregation needs 16-byte rows (ld % 4 == 0, aligned base)");
    const uint32_t dim32 = static_cast<uint32_t>(dim);
    const uint32_t nq = (dim32 + 3) / 4;
    if (nq > 16)
        launch_groups<32>(gbeg, gend, gdest, dest_groups, edges, G, (nq + 31) / 32, in, ld_in, out, ld_out, dim32,
                          true, s);
    else if (nq > 8)
        launch_groups<16>(gbeg, gend, gdest, dest_groups, edges, G, 1, in, ld_in, out, ld_out, dim32, true, s);
    else if (nq > 4)
        launch_groups<8>(gbeg, gend, gdest, dest_groups, edges, G, 1, in, ld_in, out, ld_out, dim32, true, s);
    else
        launch_groups<4>(gbeg, gend, gdest, dest_groups, edges, G, 1, in, ld_in, out, ld_out, dim32, true, s);
}

void aggregate_groups_af(Groups& G, const uint64_t* offsets_dev, uint32_t D, const Edge* edges, const float* in,
                         uint64_t ld_in, float* out, uint64_t ld_out, uint64_t dim, bool accumulate, cudaStream_t s,
                         const uint64_t* seg_lo, const uint64_t* seg_hi) {
    if (dim == 0 || D == 0) return;
    const bool vec = (ld_in % 4 == 0) && (ld_out % 4 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0) && ld_in >= ((dim + 3) & ~3ull) &&
                     ld_in < (1ull << 30);
    if (!vec) fail(kConfig, "grouped aggregation needs 16-byte rows (ld % 4 == 0, aligned base)");
    const uint32_t dim32 = static_cast<uint32_t>(dim);
    const uint32_t nq = (dim32 + 3) / 4;
    const int lpd = nq > 16 ? 32 : nq > 8 ? 16 : nq > 4 ? 8 : 4;
    const uint32_t workers = 256 / lpd;
    Groups::GrpSched* sc = nullptr;
    for (auto& x : G.grp_scheds)
        if (x->workers == workers) sc = x.get();
    if (!sc) {
        G.grp_scheds.push_back(std::make_unique<Groups::GrpSched>());
        sc = G.grp_scheds.back().get();
        build_grp_sched(offsets_dev, D, G.gs, workers, *sc, lib_stream(G.device));
    }
    const uint32_t chunks = lpd == 32 ? (nq + 31) / 32 : 1;
    if (lpd == 32) launch_grp<32>(G, *sc, edges, chunks, in, ld_in, out, ld_out, dim32, accumulate, s, seg_lo, seg_hi);
    else if (lpd == 16)
        launch_grp<16>(G, *sc, edges, chunks, in, ld_in, out, ld_out, dim32, accumulate, s, seg_lo, seg_hi);
    else if (lpd == 8) launch_grp<8>(G, *sc, edges, chunks, in, ld_in, out, ld_out, dim32, accumulate, s, seg_lo, seg_hi);
    else launch_grp<4>(G, *sc, edges, chunks, in, ld_in, out, ld_out, dim32, accumulate, s, seg_lo, seg_hi);
}

void aggregate_f64(const uint64_t* ebeg, const uint64_t* eend, const uint32_t* src, uint32_t src_stride,
                   const double* w, const uint32_t* order, uint32_t D, uint32_t n_hub, uint32_t n_front,
                   const double* in, uint64_t ld_in, double* out, uint64_t ld_out, uint64_t dim, bool accumulate,
                   cudaStream_t s, uint64_t n_edges) {
    if (D == 0 || dim == 0) return;
    if (ld_in % 2 || ld_out % 2 || reinterpret_cast<uintptr_t>(in) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
        fail(kConfig, "aggregate_pull<double>: rows must be 16-byte aligned (even ld, aligned base)");
    const uint32_t d32 = static_cast<uint32_t>(dim);
    const int acc = accumulate ? 1 : 0;
    n_hub = std::min(n_hub, D);
    SideStream* ss = nullptr;
    if (n_hub) {  // the hubs on the forked side stream, concurrent with the rest
        ss = &side_stream(s);
        PG_CUDA(cudaEventRecord(ss->fork, s));
        PG_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
        if (dim <= 16) {
            k_agg_f64_hub<16><<<n_hub, 256, 0, ss->s>>>(ebeg, eend, src, src_stride, w, order, 1u, in, ld_in, out,
                                                       ld_out, d32, acc);
        } else {
            const uint32_t ch = static_cast<uint32_t>((dim + 31) / 32);
            k_agg_f64_hub<32><<<static_cast<unsigned>(n_hub) * ch, 256, 0, ss->s>>>(
                ebeg, eend, src, src_stride, w, order, ch, in, ld_in, out, ld_out, d32, acc);
        }
        PG_LAUNCH("k_agg_f64_hub");
        PG_CUDA(cudaEventRecord(ss->join, ss->s));
    }
    const uint32_t nd = D - n_hub;
    if (nd) {
        const uint32_t* ord = order + n_hub;
        const uint32_t np = static_cast<uint32_t>((dim + 1) / 2);  // double2 per row
        const int lpd = np > 16 ? 32 : np > 8 ? 16 : np > 4 ? 8 : 4;
        const uint32_t chunks = (np + lpd - 1) / lpd;
        const uint32_t nf = chunks > 1 ? std::min(n_front > n_hub ? n_front - n_hub : 0u, nd) : 0u;
        const uint64_t items = static_cast<uint64_t>(nd) * chunks;
        const unsigned grid = grid_for(items * lpd, 256);
        const int64_t v8 = tuning(kTuneVec8);
        if (lpd == 32 && (v8 == 1 || (v8 == 2 && n_edges >= (1ull << 21))) && ld_in % 4 == 0 &&
            reinterpret_cast<uintptr_t>(in) % 32 == 0) {
            // 256-bit gathers for rows wider than 32 doubles, on the f32
            // rule (tuning vec8; arxiv's 0.6M-edge top path: 0.27 vs 0.29 ms
            // without; Reddit layer 0 40.7 -> 38.6 ms, products 11.9 -> 8.3)
            const uint64_t it = static_cast<uint64_t>(nd) * ((dim + 63) / 64);
            k_agg_f64v<4><<<grid_for(it * 16, 256), 256, 0, s>>>(ebeg, eend, src, src_stride, w, ord, it,
                                                                 static_cast<uint32_t>((dim + 63) / 64), in, ld_in,
                                                                 out, ld_out, d32, acc, 0ull);
        } else if (lpd == 32)
            k_agg_f64<32, 8><<<grid, 256, 0, s>>>(ebeg, eend, src, src_stride, w, ord, items, chunks, nf, in, ld_in,
                                                  out, ld_out, d32, acc, 0ull);
        else if (lpd == 16)
            k_agg_f64<16, 8><<<grid, 256, 0, s>>>(ebeg, eend, src, src_stride, w, ord, items, chunks, nf, in, ld_in,
                                                  out, ld_out, d32, acc, 0ull);
        else if (lpd == 8)
            k_agg_f64<8, 8><<<grid, 256, 0, s>>>(ebeg, eend, src, src_stride, w, ord, items, chunks, nf, in, ld_in,
                                                 out, ld_out, d32, acc, 0ull);
        else
            k_agg_f64<4, 8><<<grid, 256, 0, s>>>(ebeg, eend, src, src_stride, w, ord, items, chunks, nf, in, ld_in,
                                                 out, ld_out, d32, acc, 0ull);
        PG_LAUNCH("k_agg_f64");
    }
    if (ss) PG_CUDA(cudaStreamWaitEvent(s, ss->join, 0));
}

void relu_backward(const float* grad, uint64_t ldg, const float* pre, uint64_t ldp, float* out, uint64_t ldo,
                   uint64_t rows, uint64_t cols, cudaStream_t s) {
    if (rows * cols == 0) return;
    k_relu_backward<<<grid_for(rows * cols, 256), 256, 0, s>>>(grad, ldg, pre, ldp, out, ldo, rows, cols);
    PG_LAUNCH("k_relu_backward");
}

void copy_rows(const float* src, uint64_t lds, float* dst, uint64_t ldd, uint64_t rows, uint64_t cols,
               cudaStream_t s) {
    if (rows * cols == 0) return;
    const unsigned tx = cols >= 256 ? 256 : 128;
    dim3 grid(static_cast<unsigned>((cols + tx - 1) / tx), static_cast<unsigned>(std::min<uint64_t>(rows, 16384)));
    k_copy_rows<<<grid, tx, 0, s>>>(src, lds, dst, ldd, rows, static_cast<uint32_t>(cols));
    PG_LAUNCH("k_copy_rows");
}

void gather_rows(const float* src, uint64_t lds, const uint32_t* ids, uint64_t k, float* out, uint64_t ldo,
                 uint64_t cols, cudaStream_t s) {
    if (k * cols == 0) return;
    k_gather_rows<<<grid_for(k * cols, 256), 256, 0, s>>>(src, lds, ids, k, out, ldo, cols);
    PG_LAUNCH("k_gather_rows");
}

}  // namespace pg
