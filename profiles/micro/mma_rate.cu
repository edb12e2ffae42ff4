// Microbenchmark: back-to-back tcgen05.mma.cta_group::1.kind::tf32 issue rate, TS (A in TMEM) vs
// SS (A in shared memory), N = 64 / 128 / 256.  One CTA per SM, one issuing thread, operands are
// uninitialised (timing only).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared
// -Xcompiler -fPIC -o mma_rate.so mma_rate.cu ; run: python mma_rate.py
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc(int n, int m = 128) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <bool TS, int N, int M = 128>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long* cycles) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t lbo = N * 16, sb = su32(smem), sa = sb + 32768;
        const uint64_t db = sdesc(sb, lbo, 128), da = sdesc(sa, 128 * 16, 128);
        const uint32_t id = idesc(N, M);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                const uint64_t dbk = db + (uint64_t)((k & 3) * 2 * lbo >> 4);
                if (TS)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                                 "r"(tmem + 256 + (k & 3) * 8), "l"(dbk), "r"(id), "r"(1));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                                 "l"(da + (uint64_t)((k & 3) * 2 * 128 * 16 >> 4)), "l"(dbk), "r"(id), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
        const long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

extern "C" int run(int ts, int n, int iters, long long* host_cycles, float* ms) {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int smem = 32768 + 65536;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<148, 128, smem>>>(iters, d);
        cudaEventRecord(a);
        kern<<<148, 128, smem>>>(iters, d);
        cudaEventRecord(b);
    };
    if (ts && n == 64) go(mma_rate<true, 64>);
    if (ts && n == 128) go(mma_rate<true, 128>);
    if (ts && n == 256) go(mma_rate<true, 256>);
    if (!ts && n == 64) go(mma_rate<false, 64>);
    if (!ts && n == 128) go(mma_rate<false, 128>);
    if (!ts && n == 256) go(mma_rate<false, 256>);
    // M = 64 (ts 2: TS, ts 3: SS)
    if (ts == 2 && n == 128) go(mma_rate<true, 128, 64>);
    if (ts == 2 && n == 256) go(mma_rate<true, 256, 64>);
    if (ts == 3 && n == 128) go(mma_rate<false, 128, 64>);
    if (ts == 3 && n == 256) go(mma_rate<false, 256, 64>);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    cudaMemcpy(host_cycles, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (int)cudaGetLastError();
}

// Protocol cost: the conv kernel's per-chunk handshake without data.  Warp 1 lane 0 = producer
// (waits empty[s], arrives full[s]); thread 0 = MMA issuer (waits full[s], 12 MMAs, commit ->
// empty[s]).  mode 0: no waits (commit only); mode 1: full handshake.
template <int N>
__global__ void __launch_bounds__(128, 1) mma_proto(int chunks, int mode, long long* cycles) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t full[4], empty[4], fin;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&fin)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    auto wait = [](uint64_t* b, uint32_t par) {
        asm volatile("{\n\t.reg .pred P1;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W%=;\n\t}" ::"r"(su32(b)), "r"(par));
    };
    if (threadIdx.x == 32 && mode == 1) {
        for (int g = 0; g < chunks; ++g) {
            const int s = g & 3, u = g >> 2;
            if (u > 0) wait(&empty[s], (u - 1) & 1);
            asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(su32(&full[s])));
        }
    }
    if (mode == 7 && threadIdx.x < 32) {
        // whole warp runs the loop (warp-uniform descriptors), elect.sync picks the issuing lane
        const uint32_t lbo = N * 16, sb = su32(smem);
        const uint64_t db = sdesc(sb, lbo, 128);
        const uint32_t id = idesc(N);
        const long long t0 = clock64();
        for (int g = 0; g < chunks; ++g) {
            const int s = g & 3;
#pragma unroll
            for (int k = 0; k < 12; ++k)
                asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                             "r"(tmem + 256 + (k & 3) * 8), "l"(db + (uint64_t)((k & 3) * 2 * lbo >> 4)), "r"(id), "r"(1));
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&empty[s])));
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&fin)));
        wait(&fin, 0);
        if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
    }
    if (threadIdx.x == 0 && mode != 7) {
        const uint32_t lbo = N * 16, sb = su32(smem);
        const uint64_t db = sdesc(sb, lbo, 128);
        const uint32_t id = idesc(N);
        const long long t0 = clock64();
        for (int g = 0; g < chunks; ++g) {
            const int s = g & 3, u = g >> 2;
            if (mode == 1) {
                wait(&full[s], u & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
            }
#pragma unroll
            for (int k = 0; k < 12; ++k)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                             "r"(tmem + 256 + (k & 3) * 8), "l"(db + (uint64_t)((k & 3) * 2 * lbo >> 4)), "r"(id), "r"(1));
            if (mode == 1 || mode == 0 || (mode == 2 && (g & 1)) || (mode == 4 && (g & 3) == 3) || (mode == 6 && (g & 63) == 63))
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s])));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&fin)));
        wait(&fin, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

extern "C" int run_proto(int n, int mode, int chunks, long long* host_cycles) {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int smem = 65536;
    if (n == 64) {
        cudaFuncSetAttribute(mma_proto<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        mma_proto<64><<<148, 128, smem>>>(chunks, mode, d);
    } else {
        cudaFuncSetAttribute(mma_proto<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        mma_proto<128><<<148, 128, smem>>>(chunks, mode, d);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(host_cycles, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (int)cudaGetLastError();
}
