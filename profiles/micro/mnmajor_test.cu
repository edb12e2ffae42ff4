// Probe of the tcgen05 TS-form MMA with an MN-major B operand in the 128-byte-swizzled layout
// produced by a 2-D TMA box (the weight gradients' B path, conv_ws.cuh Op::B_TMA):
//   C[128][N] = A[128][32] * B[32][N],  A in TMEM (lane = row, column = k), B in global as
//   [k][n] (n contiguous) loaded as N/32 boxes of {32 n, 32 k} with CU_TENSOR_MAP_SWIZZLE_128B.
// Tries descriptor variants and prints the max error of each (0 = correct).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../include -o mnmajor_test mnmajor_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "../../paper_2006_11972_b200/csrc/kernels/conv_ws.cuh"

using namespace smx::tc3;
using smx::cnn::ws::mma_commit_e;
using smx::cnn::ws::mma_ts_e;
using smx::cnn::ws::tmem_ld16;
using smx::cnn::ws::tmem_st16;

template <int N>
__global__ void probe(const CUtensorMap* tm, const float* A, float* C, uint32_t lbo, uint32_t sbo, int layout, int kstep,
                      int bmajor) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t b = smem_u32(&bar[0]), dst = smem_u32(smem);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(N * 32 * 4));
        for (int j = 0; j < N / 32; ++j)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    dst + j * 4096),
                "l"(tm), "r"(32 * j), "r"(0), "r"(b)
                : "memory");
    }
    // A row = thread -> TMEM columns [128, 160)
    float a[32];
    for (int k = 0; k < 32; ++k) a[k] = A[threadIdx.x * 32 + k];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 128;
    tmem_st16(ta, a);
    tmem_st16(ta + 16, a + 16);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    mbar_wait(&bar[0], 0);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        const uint32_t idesc = idesc_tf32(N) | (bmajor ? (1u << 16) : 0u);
        const uint32_t base = smem_u32(smem);
        for (int st = 0; st < 4; ++st) {
            uint64_t d = (uint64_t)(((base + st * kstep) >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
            mma_ts_e(tmem, tmem + 128 + st * 8, d, idesc, st ? 1u : 0u);
        }
        mma_commit_e(&bar[1]);
    }
    mbar_wait(&bar[1], 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < N; c += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[threadIdx.x * N + c + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N>
void run(CUtensorMapSwizzle swz, const char* swzname) {
    std::vector<float> A(128 * 32), B(32 * N), C(128 * N), R(128 * N, 0.f);
    for (int i = 0; i < 128 * 32; ++i) A[i] = (float)((i * 7) % 13 - 6);
    for (int i = 0; i < 32 * N; ++i) B[i] = (float)((i * 5) % 11 - 5);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n)
            for (int k = 0; k < 32; ++k) R[m * N + n] += A[m * 32 + k] * B[k * N + n];
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)N, 32}, strides[1] = {(cuuint64_t)N * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return;
    }
    CUtensorMap* dtm;
    cudaMalloc(&dtm, sizeof tm);
    cudaMemcpy(dtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    struct V {
        uint32_t lbo, sbo;
        int layout, kstep, bmajor;
        const char* name;
    } vs[] = {
        {4096, 512, 1, 1024, 1, "MN B32 lbo=4096 sbo=512 kstep=1024"},
        {512, 4096, 1, 1024, 1, "MN B32 lbo=512 sbo=4096 kstep=1024"},
        {4096, 1024, 1, 1024, 1, "MN B32 lbo=4096 sbo=1024 kstep=1024"},
        {1024, 4096, 1, 1024, 1, "MN B32 lbo=1024 sbo=4096 kstep=1024"},
        {4096, 512, 1, 512, 1, "MN B32 lbo=4096 sbo=512 kstep=512"},
        {4096, 1024, 2, 1024, 1, "MN SW128 lbo=4096 sbo=1024 kstep=1024"},
    };
    for (const V& v : vs) {
        cudaMemset(dC, 0, C.size() * 4);
        probe<N><<<1, 128, 64 * 1024>>>(dtm, dA, dC, v.lbo, v.sbo, v.layout, v.kstep, v.bmajor);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("N=%d %s: %s\n", N, v.name, cudaGetErrorString(e));
            return;
        }
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double mx = 0, nrm = 0;
        for (int i = 0; i < 128 * N; ++i) {
            mx = std::fmax(mx, std::fabs(C[i] - R[i]));
            nrm = std::fmax(nrm, std::fabs(C[i]));
        }
        printf("N=%d tma=%s %-40s max err %g (max |C| %g)\n", N, swzname, v.name, mx, nrm);
    }
}

int main() {
    run<64>(CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "128B_ATOM_32B");
    run<128>(CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "128B_ATOM_32B");
    run<64>(CU_TENSOR_MAP_SWIZZLE_128B, "128B");
    return 0;
}
// Result on B200 (profiles/r02/mnmajor_test.txt): only TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B +
// descriptor layout type 1 (SWIZZLE_128B_BASE32B), LBO 4096, SBO 512, k-step 1024 B is exact; the
// plain 128B swizzle with layout type 2 makes the MN-major tf32 MMA write zeros.
