// Probe: SS-form tcgen05.mma kind::tf32 with BOTH operands MN-major in shared memory
// (SWIZZLE_128B_BASE32B, written by TMA boxes with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B), where the
// A operand's four 32-element M atoms start at an arbitrary 128-byte row offset `s` of a TMA tile
// and are `L` rows apart (LBO = 128 L bytes) -- the addressing an implicit-GEMM weight gradient
// needs to read shifted im2col windows straight out of one staged input tile:
//   C[m = 32 j + c][n] = sum_{k < 8} G[s + j L + k][c] * B[k][n]
// Variants: descriptor base-offset field (bits 49-51) = 0 or (addr >> 7) & 7; L in {4, 5, 17}.
// Then a throughput loop: cycles per SS MMA (M 128, N 64 / 128, K 8) issued from a whole warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o ss_shift_test ss_shift_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "../../paper_2006_11972_b200/csrc/kernels/conv_ws.cuh"

using namespace smx::tc3;
using smx::cnn::ws::mma_commit_e;
using smx::cnn::ws::tmem_ld16;

constexpr int kR = 64;  // rows of the A tile (128 B each)

__device__ __forceinline__ void mma_ss_e(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t base_off) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)(base_off & 7) << 49) | (1ull << 61);
}

template <int N>
__global__ void probe(const CUtensorMap* tmA, const CUtensorMap* tmB, float* C, int s, int L, int bo_mode) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128));
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
    char* sa = smem;                  // A tile: kR rows x 128 B
    char* sb = smem + kR * 128;       // B tile: N/32 atoms of 32 rows x 128 B (4 KB)
    if (threadIdx.x == 0) {
        const uint32_t b = smem_u32(&bar[0]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kR * 128 + N * 32 * 4));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(sa)),
            "l"(tmA), "r"(0), "r"(0), "r"(b)
            : "memory");
        for (int j = 0; j < N / 32; ++j)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    smem_u32(sb + j * 4096)),
                "l"(tmB), "r"(32 * j), "r"(0), "r"(b)
                : "memory");
    }
    mbar_wait(&bar[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        // A MN-major (bit 15), B MN-major (bit 16)
        const uint32_t idesc = idesc_tf32(N) | (1u << 15) | (1u << 16);
        const uint32_t aaddr = smem_u32(sa) + s * 128;
        const uint32_t bo = bo_mode == 1 ? ((aaddr >> 7) & 7) : bo_mode == 2 ? ((aaddr >> 7) & 3) : 0;
        const uint64_t da = desc_mn(aaddr, L * 128, 512, bo);
        const uint64_t db = desc_mn(smem_u32(sb), 4096, 512, 0);
        mma_ss_e(tmem, da, db, idesc, 0u);
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
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

// throughput: `iters` x 12 SS MMAs (M 128, N, K 8) from one warp, commit + wait per 12
template <int N>
__global__ void rate(int iters, long long* cyc, int shifted) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t idesc = idesc_tf32(N) | (1u << 15) | (1u << 16);
        const uint32_t base = smem_u32(smem);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 12; ++j) {
                const uint32_t aaddr = base + (shifted ? (j % 3) * 128 + (j / 3) * 1024 : (j % 4) * 1024);
                mma_ss_e(tmem, desc_mn(aaddr, shifted ? 2176 : 4096, 512, shifted ? ((aaddr >> 7) & 7) : 0),
                         desc_mn(base + 24 * 1024 + (j % 4) * 1024, 4096, 512, 0), idesc, (it | j) ? 1u : 0u);
            }
            mma_commit_e(&bar);
            mbar_wait(&bar, it & 1);
        }
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

static CUtensorMap make_map(float* p, int cols, int rows, int box_rows) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows}, es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        printf("encode failed\n");
    return tm;
}

template <int N>
void run() {
    std::vector<float> G(kR * 32), B(32 * N), C(128 * N);
    for (int i = 0; i < kR * 32; ++i) G[i] = (float)((i * 7 + i / 32 * 3) % 13 - 6);
    for (int i = 0; i < 32 * N; ++i) B[i] = (float)((i * 5) % 11 - 5);
    float *dG, *dB, *dC;
    cudaMalloc(&dG, G.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tm[2] = {make_map(dG, 32, kR, kR), make_map(dB, N, 32, 32)};
    CUtensorMap* dtm;
    cudaMalloc(&dtm, sizeof tm);
    cudaMemcpy(dtm, tm, sizeof tm, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int Ls[] = {4, 5, 17};
    for (int L : Ls)
        for (int bo = 0; bo < 3; ++bo) {
            printf("N=%d L=%2d base_off=%s:", N, L, bo == 0 ? "0       " : bo == 1 ? "addr&7  " : "addr&3  ");
            for (int s = 0; s < 8; ++s) {
                if (s + 3 * L + 8 > kR) break;
                cudaMemset(dC, 0, C.size() * 4);
                probe<N><<<1, 128, 64 * 1024>>>(dtm, dtm + 1, dC, s, L, bo);
                if (cudaDeviceSynchronize() != cudaSuccess) {
                    printf(" launch error\n");
                    return;
                }
                cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
                double mx = 0;
                for (int m = 0; m < 128; ++m)
                    for (int n = 0; n < N; ++n) {
                        double r = 0;
                        for (int k = 0; k < 8; ++k) r += (double)G[(s + (m / 32) * L + k) * 32 + m % 32] * B[k * N + n];
                        mx = std::fmax(mx, std::fabs(C[m * N + n] - r));
                    }
                printf(" s%d:%g", s, mx);
            }
            printf("\n");
        }
}

template <int N>
void run_rate() {
    long long* dc;
    cudaMalloc(&dc, 148 * 8);
    cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int sh = 0; sh < 2; ++sh) {
        rate<N><<<148, 128, 64 * 1024>>>(10, dc, sh);
        rate<N><<<148, 128, 64 * 1024>>>(2000, dc, sh);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, dc, sizeof h, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        printf("SS MN/MN N=%3d %s: %.1f cycles/MMA (%s)\n", N, sh ? "shifted A starts" : "aligned A starts",
               avg / (2000 * 12), cudaGetErrorString(e));
    }
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    run<64>();
    run<128>();
    run_rate<64>();
    run_rate<128>();
    return 0;
}
