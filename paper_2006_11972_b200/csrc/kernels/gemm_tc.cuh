// Tensor-core building blocks shared by the warp-specialised kernels (conv_ws.cuh): tile
// constants, the UMMA shared-memory / instruction descriptors for kind::tf32, tcgen05.mma
// (SS and TS forms), tcgen05.commit, mbarrier init/wait, 16-byte cp.async with zero fill and
// TMEM stores.  3xTF32: a = hi + lo with hi, lo tf32; each k-step issues A_lo*B_hi + A_hi*B_lo +
// A_hi*B_hi into one fp32 TMEM accumulator (DESIGN.md §3.6 / §3b.4 state the tolerances).
// The tc::TcEpi names are the epilogue selectors the executor's GEMM calls use.
#pragma once

#include "common.cuh"
#include "gemm_simt.cuh"

namespace smx {
namespace tc {

constexpr int kBM = 128;
constexpr int kBN = 128;                         // N tile (the last tile may be narrower)
constexpr int kKC = 32;                          // K elements per pipeline chunk
constexpr int kKQ = kKC / 4;                     // 16-byte k-quads per chunk
constexpr int kThreads = 256;
// raw (as copied) tiles: K-contiguous rows of kKC k padded by 4 floats, or kKC k-rows of 128
constexpr int kRawLdK = kKC + 4;                 // floats per row, K-contiguous raw tile
constexpr int kRawLdMN = kBM + 4;                // floats per k-row, row-contiguous raw tile
constexpr int kRawTile = kBM * kRawLdK * 4;      // 18432 B >= kKC * kRawLdMN * 4 = 16896
constexpr int kRawStage = 2 * kRawTile;          // A, B
// K-major canonical: (row r, k) at (k/4)*kLbo + (r/8)*128 + (r%8)*16 + (k%4)*4  (SBO = 128)
constexpr int kLbo = kBM * 16 + 16;              // 2064: padding keeps the split pass conflict-free
constexpr int kTile = kKQ * kLbo;                // 16512 per operand per hi/lo
constexpr int kHiLo = 4 * kTile;                 // A_hi A_lo B_hi B_lo
constexpr int kSmem = 2 * kRawStage + 2 * kHiLo + 64;  // ~201 KB: one CTA per SM
constexpr int kTmemCols = 128;

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

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

// 16-byte async copy; bytes past `valid_bytes` (0..16) are zero-filled.
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int valid_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid_bytes));
}

enum TcEpi { kTcStore = 0, kTcBiasRelu = 1, kTcBias = 2, kTcMask = 3, kTcStoreT = 4 };

}  // namespace tc
}  // namespace smx

// TS-form constants and helpers (A operand in TMEM, B in shared memory).
namespace smx {
namespace tc3 {

constexpr int kBM = 128;
constexpr int kBN = 128;                         // N tile (the last tile may be narrower)
constexpr int kKC = 32;                          // K elements per pipeline chunk
constexpr int kKQ = kKC / 4;                     // 16-byte k-quads per chunk
constexpr int kThreads = 512;
constexpr int kParts = kThreads / 128;           // warps per TMEM lane quadrant
constexpr int kAK = kKC / kParts;                // A k-values per thread per chunk
// B raw (as copied) tile: K-contiguous rows of kKC k padded by 4 floats, or kKC k-rows of 128 (+4)
constexpr int kRawLdK = kKC + 4;
constexpr int kRawLdMN = kBN + 4;
constexpr int kRawTile = kBN * kRawLdK * 4;      // 18432 B >= kKC * kRawLdMN * 4 = 16896
// B K-major canonical: (row r, k) at (k/4)*kLbo + (r/8)*128 + (r%8)*16 + (k%4)*4   (SBO = 128)
constexpr int kLbo = kBN * 16 + 16;              // 2064: padding keeps the split pass conflict-free
constexpr int kTile = kKQ * kLbo;                // 16512 per hi or lo
constexpr int kSmem = 4 * kRawTile + 4 * kTile + 64;  // (raw A, raw B) x2, (B hi, B lo) x2, barriers: ~140 KB
// TMEM columns: [0,128) accumulator, then per buffer b: A_hi at 128 + 64b, A_lo at 160 + 64b
constexpr int kTmemCols = 256;

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

// D[tmem] (+)= A[tmem] * B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

// 16-byte async copy; bytes past `valid_bytes` (0..16) are zero-filled.
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int valid_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid_bytes));
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
}

__device__ __forceinline__ void split4(float4 v, float4& h, float4& l) {
    h.x = tf32_rna(v.x); l.x = tf32_rna(__fsub_rn(v.x, h.x));
    h.y = tf32_rna(v.y); l.y = tf32_rna(__fsub_rn(v.y, h.y));
    h.z = tf32_rna(v.z); l.z = tf32_rna(__fsub_rn(v.z, h.z));
    h.w = tf32_rna(v.w); l.w = tf32_rna(__fsub_rn(v.w, h.w));
}

using tc::TcEpi;
using tc::kTcStore;
using tc::kTcBiasRelu;
using tc::kTcBias;
using tc::kTcMask;
using tc::kTcStoreT;

}  // namespace tc3
}  // namespace smx
