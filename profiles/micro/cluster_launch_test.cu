// Runtime cluster launches (cudaLaunchKernelEx + cudaLaunchAttributeClusterDimension) of a kernel
// without __cluster_dims__: which cluster shapes / block sizes / smem sizes launch.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k(int* out) {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    if (threadIdx.x == 0) out[blockIdx.y * gridDim.x + blockIdx.x] = (int)r;
}
int main() {
    int* d;
    cudaMalloc(&d, 1024 * 4);
    struct V { dim3 grid, cl; int threads; size_t smem; } vs[] = {
        {dim3(2, 1, 1), dim3(2, 1, 1), 128, 0}, {dim3(1, 2, 1), dim3(1, 2, 1), 128, 0},
        {dim3(4, 4, 4), dim3(1, 2, 1), 480, 0}, {dim3(4, 4, 4), dim3(1, 2, 1), 480, 229888},
        {dim3(4, 4, 4), dim3(2, 1, 1), 480, 229888}, {dim3(4, 4, 4), dim3(1, 2, 1), 480, 200000},
    };
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 229888);
    for (auto& v : vs) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = v.grid;
        cfg.blockDim = dim3(v.threads);
        cfg.dynamicSmemBytes = v.smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = v.cl.x;
        at[0].val.clusterDim.y = v.cl.y;
        at[0].val.clusterDim.z = v.cl.z;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("grid %u %u %u cluster %u %u %u threads %d smem %zu: %s / %s\n", v.grid.x, v.grid.y, v.grid.z, v.cl.x, v.cl.y,
               v.cl.z, v.threads, v.smem, cudaGetErrorString(e), cudaGetErrorString(e2));
        cudaGetLastError();
    }
    return 0;
}
