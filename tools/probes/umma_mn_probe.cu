// Probe of tcgen05.mma kind::tf32 operand layouts (one CTA, M=128, N=32,
// K=8): K-major SW128 (the y_grad kernel's form) as the control, then
// MN-major SW128 with the two candidate LBO/SBO assignments. Prints, per
// variant, the max |D - A.B| over the tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_probe tools/probes/umma_mn_probe.cu && /tmp/umma_probe
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// mode 0: A,B K-major; 1: A,B MN-major (LBO = MN atom stride, SBO = K group stride);
// 2: MN-major with LBO/SBO swapped
__global__ void probe(const float* A, const float* B, float* D, int mode) {
    // A: M=128 x K=8, B: N=32 x K=8 (row-major [m][k], [n][k])
    __shared__ __align__(1024) unsigned char sm[16384 + 4096];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    unsigned char* As = sm;                  // K-major: 128 rows x 128 B
    unsigned char* Bs = sm + 16384;          // 32 rows x 128 B
    const int tid = threadIdx.x;
    for (int i = tid; i < 16384 + 4096; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    if (mode == 0) {
        // K-major SW128: row m (128 B = 32 floats of K; only 8 used), chunk c of row m at c ^ (m & 7)
        for (int e = tid; e < 128 * 8; e += blockDim.x) {
            int m = e / 8, k = e % 8;
            int off = m * 128 + (((k >> 2) ^ (m & 7)) << 4) + (k & 3) * 4;
            *reinterpret_cast<float*>(As + off) = A[m * 8 + k];
        }
        for (int e = tid; e < 32 * 8; e += blockDim.x) {
            int n = e / 8, k = e % 8;
            int off = n * 128 + (((k >> 2) ^ (n & 7)) << 4) + (k & 3) * 4;
            *reinterpret_cast<float*>(Bs + off) = B[n * 8 + k];
        }
    } else if (mode >= 3) {
        // MN-major SWIZZLE_128B_BASE32B (layout type 1, CUTLASS Layout_MN_SW128_32B_Atom):
        // atom = 4 K rows x 32 MN floats (512 B), 32-byte units XORed with (k & 3);
        // A: 4 MN atoms 512 B apart, K groups 2048 B apart; B: one atom, K groups 512 B apart
        for (int e = tid; e < 128 * 8; e += blockDim.x) {
            int m = e / 8, k = e % 8;
            int off = (k / 4) * 2048 + (m / 32) * 512 + (k % 4) * 128 + ((((m % 32) >> 3) ^ (k % 4)) << 5) + (m & 7) * 4;
            *reinterpret_cast<float*>(As + off) = A[m * 8 + k];
        }
        for (int e = tid; e < 32 * 8; e += blockDim.x) {
            int n = e / 8, k = e % 8;
            int off = (k / 4) * 512 + (k % 4) * 128 + (((n >> 3) ^ (k % 4)) << 5) + (n & 7) * 4;
            *reinterpret_cast<float*>(Bs + off) = B[n * 8 + k];
        }
    } else {
        // MN-major SW128: atom = 8 K rows x 32 MN floats (1024 B); atoms along MN 1024 B apart
        for (int e = tid; e < 128 * 8; e += blockDim.x) {
            int m = e / 8, k = e % 8;
            int off = (m / 32) * 1024 + k * 128 + ((((m % 32) >> 2) ^ k) << 4) + (m & 3) * 4;
            *reinterpret_cast<float*>(As + off) = A[m * 8 + k];
        }
        for (int e = tid; e < 32 * 8; e += blockDim.x) {
            int n = e / 8, k = e % 8;
            int off = k * 128 + (((n >> 2) ^ k) << 4) + (n & 3) * 4;
            *reinterpret_cast<float*>(Bs + off) = B[n * 8 + k];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (tid == 0) {
        uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
        uint64_t ad, bd;
        if (mode == 0) {
            ad = desc(sa(As), 16, 1024);
            bd = desc(sa(Bs), 16, 1024);
        } else {
            idesc |= (1u << 15) | (1u << 16);
            if (mode == 1) {
                ad = desc(sa(As), 1024, 4096);
                bd = desc(sa(Bs), 1024, 4096);
            } else if (mode == 2) {
                ad = desc(sa(As), 4096, 1024);
                bd = desc(sa(Bs), 4096, 1024);
            } else if (mode == 3) {  // layout type 1, LBO = MN atom stride, SBO = K group stride
                ad = (desc(sa(As), 512, 2048) & ~(7ull << 61)) | (1ull << 61);
                bd = (desc(sa(Bs), 512, 512) & ~(7ull << 61)) | (1ull << 61);
            } else {                 // swapped
                ad = (desc(sa(As), 2048, 512) & ~(7ull << 61)) | (1ull << 61);
                bd = (desc(sa(Bs), 512, 512) & ~(7ull << 61)) | (1ull << 61);
            }
        }
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc)
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                     : "memory");
    }
    __syncwarp();
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra.uni D;\n\tbra.uni W;\nD:\n\t}" ::"r"(
            sa(&bar))
        : "memory");
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int warp = tid / 32, lane = tid % 32;
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 32 + j] = __uint_as_float(v[j]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main() {
    std::vector<float> A(128 * 8), B(32 * 8), D(128 * 32);
    for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 7) % 13) - 6;
    for (int i = 0; i < 32 * 8; ++i) B[i] = (float)((i * 5) % 11) - 5;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 5; ++mode) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0, mag = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 32; ++n) {
                double s = 0;
                for (int k = 0; k < 8; ++k) s += (double)A[m * 8 + k] * B[n * 8 + k];
                worst = fmax(worst, fabs(s - D[m * 32 + n]));
                mag = fmax(mag, fabs(s));
            }
        printf("mode %d (%s): max |D - AB| = %g (max |AB| %g) D[0..3]=%g %g %g %g err=%s\n", mode,
               mode == 0 ? "K-major" : mode == 1 ? "MN SW128 LBO=MN atom, SBO=K group" : mode == 2 ? "MN SW128 swapped" : mode == 3 ? "MN SW128_BASE32B LBO=MN atom, SBO=K group" : "MN SW128_BASE32B swapped", worst, mag,
               D[0], D[1], D[2], D[3], cudaGetErrorString(e));
    }
    return 0;
}
