// Probe: tcgen05.cp.cta_group::1.128x256b from a K-major SWIZZLE_128B fp32 tile (what a TMA box
// with CU_TENSOR_MAP_SWIZZLE_128B writes: row r at r x 128 B, 16-byte unit u at u ^ (r & 7)) into
// TMEM lanes 0..127, 4 copies of 8 columns (k 8j .. 8j + 7: descriptor start + 32 j bytes).
// Checks that TMEM column c of lane r holds element (r, c).
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(float* out, int variant) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5;
    float* tile = reinterpret_cast<float*>(smem);
    for (int e = t; e < 128 * 32; e += blockDim.x) {
        const int r = e / 32, c = e % 32, u = c / 4;
        tile[r * 32 + ((u ^ (r & 7)) * 4) + c % 4] = r * 100.0f + c;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    if (t == 0) {
        const uint32_t a = smem_u32(tile);
        for (int j = 0; j < 4; ++j) {
            // K-major, SWIZZLE_128B (layout 2), SBO = 1024 B (8-row groups), LBO unused (1), version 1
            const uint64_t d = (uint64_t)(((a + 32 * j) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
                               ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | ((uint64_t)(variant == 0 ? 2 : 1) << 61);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 8 * j), "l"(d));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        uint32_t r[32];
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
              "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const int row = warp * 32 + (t & 31);
        for (int c = 0; c < 32; ++c) out[row * 32 + c] = __uint_as_float(r[c]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 32 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(d, 0, 128 * 32 * 4);
        k<<<1, 128, 32768>>>(d, variant);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> h(128 * 32);
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 128; ++r)
            for (int c = 0; c < 32; ++c)
                if (h[r * 32 + c] != r * 100.0f + c) {
                    if (bad < 6) printf("  (%d,%d) = %g\n", r, c, h[r * 32 + c]);
                    ++bad;
                }
        printf("variant %d (%s): %s, mismatches %d\n", variant, variant == 0 ? "SWIZZLE_128B" : "layout 1",
               cudaGetErrorString(e), bad);
    }
    return 0;
}
