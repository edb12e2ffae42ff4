// Standalone check of the TMA tiled-load semantics the conv producers rely on: a 4-D NHWC fp32
// tensor, box (C 32, W 16 x stride 2, H 8 x stride 2, N 1) at negative / strided start
// coordinates, 128-byte swizzle, zero fill out of bounds.  Prints mismatches (0 = as expected).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_test tma_test.cu && ./tma_test
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void load_box(const CUtensorMap* tm, int c0, int w0, int h0, int n0, float* out) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) unsigned long long bar;
    float* tile = reinterpret_cast<float*>(smem);
    const unsigned tb = (unsigned)__cvta_generic_to_shared(tile), bb = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(16384));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(tb), "l"(tm), "r"(c0), "r"(w0), "r"(h0), "r"(n0), "r"(bb) : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(bb));
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = tile[i];
}

int main() {
    const int N = 3, H = 32, W = 32, C = 32;
    std::vector<float> h((size_t)N * H * W * C);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i + 1);
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 4096 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
    cuuint32_t box[4] = {32, 32, 16, 1}, es[4] = {1, 2, 2, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    CUtensorMap* dtm;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(load_box, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    int bad_total = 0;
    const int cases[][4] = {{0, -1, -1, 1}, {0, 0, 13, 2}, {0, 1, 15, 0}, {0, -1, 17, 1}};
    for (auto& cs : cases) {
        load_box<<<1, 128, 32768>>>(dtm, cs[0], cs[1], cs[2], cs[3], o);
        std::vector<float> got(4096);
        if (cudaMemcpy(got.data(), o, 4096 * 4, cudaMemcpyDeviceToHost) != cudaSuccess) { printf("kernel failed\n"); return 1; }
        int bad = 0;
        for (int row = 0; row < 128; ++row) {  // row = (hh, ww): element (c0 + k, w0 + 2 ww, h0 + 2 hh, n0)
            const int hh = row / 16, ww = row % 16;
            for (int k = 0; k < 32; ++k) {
                const int c = cs[0] + k, w = cs[1] + 2 * ww, hy = cs[2] + 2 * hh, n = cs[3];
                const float want = (w < 0 || w >= W || hy < 0 || hy >= H) ? 0.0f : h[(((size_t)n * H + hy) * W + w) * C + c];
                const int kq = k / 4, pos = row * 32 + ((kq ^ (row & 7)) * 4) + k % 4;
                if (got[pos] != want) ++bad;
            }
        }
        printf("case (%d,%d,%d,%d): %d mismatches\n", cs[0], cs[1], cs[2], cs[3], bad);
        bad_total += bad;
    }
    printf("%s\n", bad_total ? "FAIL" : "OK");
    return bad_total != 0;
}
