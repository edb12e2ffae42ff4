// Probe of the 2-SM tcgen05 MMA (cta_group::2) in the TS form the conv kernels use:
//   C[256][128] = A[256][8] * B[128][8]^T, kind::tf32, A in TMEM (CTA r of the pair holds rows
//   128 r .. 128 r + 127), B K-major SWIZZLE_NONE in shared memory (CTA r holds rows 64 r .. 64 r + 63
//   at the same offset), D in each CTA's TMEM (its 128 rows x 128 columns).  The leader CTA issues
//   the MMA; the commit multicasts to both CTAs' barriers.  Prints the max error (0 = correct).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o pair_mma_test pair_mma_test.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr int M = 256, N = 128, K = 8;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_probe(const float* A, const float* B, float* C, int mode) {
    __shared__ __align__(1024) float bs[N / 2 * K];  // this CTA's B half: 64 rows x 8 k, canonical
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B half: rows 64 rank .. + 63 (mode 1: rows 0..63 in both CTAs, to see which half is read)
    for (int e = threadIdx.x; e < N / 2 * K; e += 128) {
        const int i = e / K, k = e % K;
        const int src_row = (mode == 1 ? 0 : 64 * (int)rank) + i;
        bs[((k / 4) * 1024 + (i / 8) * 128 + (i % 8) * 16 + (k % 4) * 4) / 4] = B[src_row * K + k];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    // A rows 128 rank + thread -> TMEM columns [128, 136)
    {
        float a[8];
        for (int k = 0; k < 8; ++k) a[k] = A[(128 * rank + threadIdx.x) * K + k];
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 128;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "f"(a[0]),
                     "f"(a[1]), "f"(a[2]), "f"(a[3]), "f"(a[4]), "f"(a[5]), "f"(a[6]), "f"(a[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (rank == 0 && warp == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t bd = smem_desc(smem_u32(bs), 1024, 128);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 0, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
            "r"(tmem + 128), "l"(bd), "r"(idesc));
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3));
    }
    // every thread waits for the MMA (phase 0 of its own CTA's barrier)
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}\n" ::"r"(
            smem_u32(&bar)),
        "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; ++j) C[(128 * rank + threadIdx.x) * N + c0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
    std::vector<float> A(M * K), B(N * K), C(M * N);
    for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7 + 3) % 17 - 8) / 8.0f;
    for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 5 + 1) % 13 - 6) / 4.0f;
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dC, 0, C.size() * 4);
        pair_probe<<<2, 128>>>(dA, dB, dC, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d: %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, err_lo = 0, err_hi = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                const int bn = (mode == 1) ? (n % 64) : n;  // mode 1: both halves hold rows 0..63
                for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[bn * K + k];
                const double d = std::fabs(ref - C[m * N + n]);
                err = std::max(err, d);
                (n < 64 ? err_lo : err_hi) = std::max(n < 64 ? err_lo : err_hi, d);
            }
        printf("mode %d: max err %.3g (cols 0-63 %.3g, 64-127 %.3g), C[0][0] %g C[255][127] %g\n", mode, err, err_lo,
               err_hi, C[0], C[M * N - 1]);
    }
    return 0;
}
