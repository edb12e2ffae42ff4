// Tensor-core building blocks shared by the warp-specialised kernels (conv_ws.cuh, wgrad2_at.cuh,
// conv1_tc.cuh): tile constants, the UMMA shared-memory descriptors (K-major SWIZZLE_NONE and the
// tf32 MN-major SWIZZLE_128B_BASE32B layout) and instruction descriptor for kind::tf32, mbarrier
// init / wait, 16-byte cp.async with zero fill and 8-column TMEM stores.  3xTF32: a = hi + lo; each
// k-step issues A_lo*B_hi + A_hi*B_lo + A_hi*B_hi into one fp32 TMEM accumulator (DESIGN.md §3.6 /
// §3b.4 state the tolerances).  tc::TcEpi are the epilogue selectors of the executor's GEMM calls.
#pragma once

#include "common.cuh"
#include "gemm_simt.cuh"

namespace smx {
namespace tc {

// epilogue selectors of the executor's GEMM calls (mapped onto the dense Op policies)
enum TcEpi { kTcStore = 0, kTcBiasRelu = 1, kTcBias = 2, kTcMask = 3, kTcStoreT = 4 };

}  // namespace tc
}  // namespace smx

// TS-form constants and helpers (A operand in TMEM, B in shared memory).
namespace smx {
namespace tc3 {

constexpr int kBM = 128;                         // M tile (TMEM lanes)
constexpr int kKC = 32;                          // K elements per pipeline chunk
constexpr int kKQ = kKC / 4;                     // 16-byte k-quads per chunk

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical ((8,m),2):((1,SBO),LBO) in
// 16-byte units), Blackwell version field = 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// UMMA shared-memory descriptor of an MN-major tf32 operand.  tf32 MN-major operands have one
// shared-memory layout, SWIZZLE_128B_BASE32B (layout type 1): 128-byte rows (32 elements along
// MN, one k each), 32-byte granules XOR-swizzled by (row % 4) -- what a TMA box with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes.  LBO = distance between 32-element atom columns
// along MN, SBO = distance between 4-row groups along K.  Verified by profiles/micro/mnmajor_test.cu.
__device__ __forceinline__ uint64_t smem_desc_mn32(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (1ull << 61);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity));
}

// 16-byte async copy; bytes past `valid_bytes` (0..16) are zero-filled.
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int valid_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid_bytes));
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
}

}  // namespace tc3
}  // namespace smx
