// K1-K3 (tensor-core mode): grouped GEMM on the 5th-generation tensor cores, 3xTF32.
//
//   C_g[m][n] = epi( sum_k A_g(m,k) * B_g(n,k) ),  one (group, 128 x BN) output tile per CTA.
//
// * tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = BN (16..256), K = 8 per instruction,
//   fp32 accumulator in TMEM (BN columns x 128 lanes), issued by one thread.
// * 3xTF32 split: every operand element a becomes hi = rna_tf32(a), lo = rna_tf32(a - hi), and
//   each k-step issues A_lo*B_hi + A_hi*B_lo + A_hi*B_hi into the same accumulator, which gives
//   fp32-level products (DESIGN.md §3.6 states the resulting tolerance).
// * Operands are copied HBM -> shared memory by per-thread 16-byte cp.async (LDGSTS) in their
//   native layout (K-contiguous or row-contiguous), two chunks ahead.  Operand pointers differ per
//   group and per step (data offset, batch size), so these are async copies, not TMA.
// * A smem->smem pass then writes the hi/lo split of the landed chunk into the UMMA K-major
//   no-swizzle canonical layout (8-row x 16-byte core matrices), transposing 4x4 blocks in
//   registers for row-contiguous operands, with padded strides so it is bank-conflict free.
// * One thread issues the chunk's 12 MMAs and tcgen05.commit's them to the buffer's mbarrier,
//   which releases that hi/lo buffer two chunks later.
// * Epilogue: tcgen05.ld 32x32b -> registers -> bias/ReLU/mask -> global.
// Per-group results depend only on the group's own operands and shape (no split-K, no atomics),
// so grouped execution stays grouping-invariant and run-to-run deterministic.
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

// Async copy of rows [r0, r0+rows) x k [k0, k0+kKC) of one operand into a raw tile.
// MN == 0: element (r,k) at g[r*ld + k] -> raw[r*kRawLdK + k]; MN == 1: at g[k*ld + r] ->
// raw[k*kRawLdMN + r].  Out-of-range elements are zero-filled.
template <int MN>
__device__ __forceinline__ void load_raw(const float* g, int ld, int r0, int rows, int rlim, int k0, int klim,
                                         uint32_t dst) {
    if (MN == 0) {
        const int units = rows * kKQ;  // (row, k-quad): a warp reads 4 rows x 128 B
        for (int u = threadIdx.x; u < units; u += kThreads) {
            const int r = u / kKQ, kq = u % kKQ;
            const int row = r0 + r, k = k0 + kq * 4;
            const int valid = row < rlim ? max(0, min(4, klim - k)) : 0;
            cp16(dst + (r * kRawLdK + kq * 4) * 4, valid ? g + (long long)row * ld + k : g, valid * 4);
        }
    } else {
        const int quads = rows >> 2;
        const int units = quads * kKC;  // (row-quad, k): a warp reads 512 contiguous bytes of one k
        for (int u = threadIdx.x; u < units; u += kThreads) {
            const int rq = u % quads, k = u / quads;
            const int row = r0 + rq * 4, kk = k0 + k;
            const int valid = kk < klim ? max(0, min(4, rlim - row)) : 0;
            cp16(dst + (k * kRawLdMN + rq * 4) * 4, valid ? g + (long long)kk * ld + row : g, valid * 4);
        }
    }
}

__device__ __forceinline__ void split_store(float4 v, char* hi, char* lo, uint32_t off) {
    float4 h, l;
    h.x = tf32_rna(v.x); l.x = tf32_rna(__fsub_rn(v.x, h.x));
    h.y = tf32_rna(v.y); l.y = tf32_rna(__fsub_rn(v.y, h.y));
    h.z = tf32_rna(v.z); l.z = tf32_rna(__fsub_rn(v.z, h.z));
    h.w = tf32_rna(v.w); l.w = tf32_rna(__fsub_rn(v.w, h.w));
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
}

// raw tile -> hi/lo K-major canonical tiles.
template <int MN>
__device__ __forceinline__ void split_tile(const char* raw, int rows, char* hi, char* lo) {
    if (MN == 0) {
        const int units = rows * kKQ;  // consecutive threads: consecutive rows, same k-quad
        for (int u = threadIdx.x; u < units; u += kThreads) {
            const int r = u % rows, kq = u / rows;
            const float4 v = *reinterpret_cast<const float4*>(raw + (r * kRawLdK + kq * 4) * 4);
            split_store(v, hi, lo, kq * kLbo + (r >> 3) * 128 + (r & 7) * 16);
        }
    } else {
        const int quads = rows >> 2;
        const int units = quads * kKQ;  // 4 rows x 4 k per thread, transposed in registers
        for (int u = threadIdx.x; u < units; u += kThreads) {
            const int rq = u % quads, kq = u / quads;
            float4 c[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                c[i] = *reinterpret_cast<const float4*>(raw + ((kq * 4 + i) * kRawLdMN + rq * 4) * 4);
            const float blk[4][4] = {{c[0].x, c[1].x, c[2].x, c[3].x},
                                     {c[0].y, c[1].y, c[2].y, c[3].y},
                                     {c[0].z, c[1].z, c[2].z, c[3].z},
                                     {c[0].w, c[1].w, c[2].w, c[3].w}};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = (i + (rq >> 1)) & 3;  // rotated order: conflict-free 16-byte stores
                const int r = rq * 4 + j;
                split_store(make_float4(blk[j][0], blk[j][1], blk[j][2], blk[j][3]), hi, lo,
                            kq * kLbo + (r >> 3) * 128 + (r & 7) * 16);
            }
        }
    }
}

enum TcEpi { kTcStore = 0, kTcBiasRelu = 1, kTcBias = 2, kTcMask = 3, kTcStoreT = 4 };

template <int AM, int BMODE, int EPI>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(GemmArgs p, int /*unused*/) {
    extern __shared__ __align__(1024) char smem[];
    char* raw = smem;                                  // 2 x (A, B) raw stages
    char* hl = smem + 2 * kRawStage;                   // 2 x (A_hi, A_lo, B_hi, B_lo)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kRawStage + 2 * kHiLo);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 2 * kRawStage + 2 * kHiLo + 32);

    const int slot = p.slots[blockIdx.z];
    const int bs = (p.m_is_bs || p.k_is_bs) ? slot_bs(p, slot) : 0;
    const int M = p.m_is_bs ? bs : p.M;
    const int K = p.k_is_bs ? bs : p.K;
    const int N = p.N;
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
    if (m0 >= M || n0 >= N) return;
    const int nt = min(kBN, (N - n0 + 15) / 16 * 16);  // MMA N of this tile
    const int nlim = min(N, n0 + kBN);

    const float* A = opnd_ptr(p.a, slot, p.st, p.n_train_mask);
    const float* B = opnd_ptr(p.b, slot, p.st, p.n_train_mask);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_tf32(nt);
    const uint32_t raw_u32 = smem_u32(raw), hl_u32 = smem_u32(hl);

    const int nchunks = (K + kKC - 1) / kKC;
    auto issue = [&](int c) {
        const uint32_t st = raw_u32 + (c & 1) * kRawStage;
        load_raw<AM>(A, p.a.ld, m0, kBM, M, c * kKC, K, st);
        load_raw<BMODE>(B, p.b.ld, n0, nt, nlim, c * kKC, K, st + kRawTile);
    };
    issue(0);
    asm volatile("cp.async.commit_group;");
    if (nchunks > 1) issue(1);
    asm volatile("cp.async.commit_group;");

#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        const int b = c & 1;
        asm volatile("cp.async.wait_group 1;");
        if (c >= 2) mbar_wait(&bars[b], ((c - 2) >> 1) & 1);  // MMAs of chunk c-2 released hl[b]
        __syncthreads();
        char* h = hl + b * kHiLo;
        split_tile<AM>(raw + b * kRawStage, kBM, h, h + kTile);
        split_tile<BMODE>(raw + b * kRawStage + kRawTile, nt, h + 2 * kTile, h + 3 * kTile);
        asm volatile("fence.proxy.async.shared::cta;");
        __syncthreads();
        if (c + 2 < nchunks) issue(c + 2);  // raw[b] is consumed
        asm volatile("cp.async.commit_group;");
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ahi = hl_u32 + b * kHiLo, alo = ahi + kTile, bhi = ahi + 2 * kTile, blo = ahi + 3 * kTile;
            const int ksteps = (min(kKC, K - c * kKC) + 7) / 8;
#pragma unroll 1
            for (int s = 0; s < ksteps; ++s) {
                const uint32_t o = s * 2 * kLbo;
                const uint64_t dah = smem_desc(ahi + o, kLbo, 128), dal = smem_desc(alo + o, kLbo, 128);
                const uint64_t dbh = smem_desc(bhi + o, kLbo, 128), dbl = smem_desc(blo + o, kLbo, 128);
                const uint32_t acc0 = (c == 0 && s == 0) ? 0u : 1u;
                mma_tf32(tmem, dal, dbh, idesc, acc0);
                mma_tf32(tmem, dah, dbl, idesc, 1u);
                mma_tf32(tmem, dah, dbh, idesc, 1u);
            }
            mma_commit(&bars[b]);
        }
    }
    const int last = nchunks - 1;
    mbar_wait(&bars[last & 1], (last >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // ---- epilogue: warp w reads TMEM lanes 32*(w%4).., column half w/4 of the tile
    const int q = warp & 3, half = warp >> 2;
    const int m = m0 + q * 32 + lane;
    const int cols = nt / 2;
    float* C = p.c + p.c_stride * slot;
    const float* bias = (EPI == kTcBiasRelu || EPI == kTcBias) ? p.bias + p.bias_stride * slot : nullptr;
    const float* mask = (EPI == kTcMask) ? p.mask + p.mask_stride * slot : nullptr;
    for (int c0 = half * cols; c0 < (half + 1) * cols; c0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (m >= M) continue;
        const int nb = n0 + c0;
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x[j] = __uint_as_float(v[j]);
            const int n = nb + j;
            if (n >= N) continue;
            if (EPI == kTcBiasRelu) {
                x[j] = __fadd_rn(x[j], bias[n]);
                x[j] = x[j] > 0.0f ? x[j] : 0.0f;
            } else if (EPI == kTcBias) {
                x[j] = __fadd_rn(x[j], bias[n]);
            } else if (EPI == kTcMask) {
                x[j] = mask[(long long)m * p.ldmask + n] > 0.0f ? x[j] : 0.0f;
            }
        }
        if (EPI == kTcStoreT) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (nb + j < N) C[(long long)(nb + j) * p.ldc + m] = x[j];
        } else if (nb + 8 <= N && (p.ldc & 3) == 0) {
            float4* dst = reinterpret_cast<float4*>(C + (long long)m * p.ldc + nb);
            dst[0] = make_float4(x[0], x[1], x[2], x[3]);
            dst[1] = make_float4(x[4], x[5], x[6], x[7]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (nb + j < N) C[(long long)m * p.ldc + nb + j] = x[j];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace tc
}  // namespace smx

// Tensor-core GEMM, TS variant (A operand in TMEM): used for the weight-gradient GEMMs.
//
//   C_g[m][n] = epi( sum_k A_g(m,k) * B_g(n,k) ),  one (group, 128 x 128) output tile per CTA.
//
// * tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 16..128, K = 8 per instruction, fp32
//   accumulator in TMEM, issued by one thread.
// * 3xTF32: every operand element a becomes hi = rna_tf32(a), lo = rna_tf32(a - hi); each k-step
//   issues A_lo*B_hi + A_hi*B_lo + A_hi*B_hi into the same accumulator (fp32-level products,
//   DESIGN.md §3.6).  Operands flagged exact (the synthetic data, k/128, is exact in tf32) skip
//   their lo half and one of the three MMAs.
// * A operand never touches shared memory: each thread loads its row's 16 k-values of the next
//   chunk into registers one chunk ahead, splits them and writes hi/lo straight into TMEM with
//   tcgen05.st (lane = row, column = k); the MMA reads A from TMEM (the ".kind::tf32 [d], [a], b"
//   form).  Row-contiguous A (weight gradients) is read column by column, coalesced across the
//   warp, so no transpose is needed either.
// * B operand: per-thread 16-byte cp.async (LDGSTS) of the native layout two chunks ahead, then a
//   smem->smem pass writes the hi/lo split into the UMMA K-major SWIZZLE_NONE canonical layout
//   (transposing 4x4 blocks in registers for row-contiguous operands; padded strides keep it
//   bank-conflict free).  Operand pointers differ per group and per step (slot, data offset,
//   batch size), so these are async copies, not TMA.  (MN-major tf32 UMMA operands would need
//   the SW128_32B swizzle.)
// * tcgen05.commit on a per-buffer mbarrier releases that buffer's TMEM A and smem B halves two
//   chunks later.  Epilogue: tcgen05.ld 32x32b -> registers -> bias/ReLU/mask -> global.
// Per-group results depend only on the group's own operands and shape (no split-K, no atomics),
// so grouped execution stays grouping-invariant and run-to-run deterministic.
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

// This thread's A values of one chunk from the raw (as copied) A tile: tile row `r`, chunk-local
// k in [k, k + kAK).  Raw rows are padded so both read patterns are bank-conflict free.
template <int AM>
__device__ __forceinline__ void read_a(const char* raw, int r, int k, float* v) {
    if (AM == 0) {
#pragma unroll
        for (int q = 0; q < kAK / 4; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(raw + (r * kRawLdK + k + 4 * q) * 4);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < kAK; ++i) v[i] = *reinterpret_cast<const float*>(raw + ((k + i) * kRawLdMN + r) * 4);
    }
}

template <int AM>
__device__ __forceinline__ void load_a(const float* g, int ld, int row, int M, int k, int K, float* v) {
    if (row >= M) {
#pragma unroll
        for (int i = 0; i < kAK; ++i) v[i] = 0.0f;
        return;
    }
    if (AM == 0) {
        const float* p = g + (long long)row * ld + k;
        if (k + kAK <= K) {
#pragma unroll
            for (int q = 0; q < kAK / 4; ++q) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(p) + q);
                v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kAK; ++i) v[i] = (k + i < K) ? __ldg(p + i) : 0.0f;
        }
    } else {
        const float* p = g + (long long)k * ld + row;
#pragma unroll
        for (int i = 0; i < kAK; ++i) v[i] = (k + i < K) ? __ldg(p + (long long)i * ld) : 0.0f;
    }
}

// Async copy of B rows [r0, r0+rows) x k [k0, k0+kKC).
// MN == 0: element (r,k) at g[r*ld + k]; MN == 1: at g[k*ld + r].  Out-of-range -> 0.
// DIRECT: exact-tf32 K-contiguous operand, copied straight into the canonical layout (no split).
template <int MN, bool DIRECT>
__device__ __forceinline__ void load_b(const float* g, int ld, int r0, int rows, int rlim, int k0, int klim,
                                       uint32_t raw, uint32_t canon) {
    if (MN == 0) {
        const int units = rows * kKQ;  // (row, k-quad): a warp reads 4 rows x 128 B
        for (int u = threadIdx.x; u < units; u += kThreads) {
            const int r = u / kKQ, kq = u % kKQ;
            const int row = r0 + r, k = k0 + kq * 4;
            const int valid = row < rlim ? max(0, min(4, klim - k)) : 0;
            const uint32_t dst = DIRECT ? canon + kq * kLbo + (r >> 3) * 128 + (r & 7) * 16
                                        : raw + (r * kRawLdK + kq * 4) * 4;
            cp16(dst, valid ? g + (long long)row * ld + k : g, valid * 4);
        }
    } else {
        const int quads = rows >> 2;
        // (row-quad, k) with 32 row-quads per k (idle lanes when rows < 128): a warp reads 512
        // contiguous bytes of one k; power-of-two index math
        for (int u = threadIdx.x; u < 32 * kKC; u += kThreads) {
            const int rq = u & 31, k = u >> 5;
            if (rq >= quads) continue;
            const int row = r0 + rq * 4, kk = k0 + k;
            const int valid = kk < klim ? max(0, min(4, rlim - row)) : 0;
            cp16(raw + (k * kRawLdMN + rq * 4) * 4, valid ? g + (long long)kk * ld + row : g, valid * 4);
        }
    }
}

__device__ __forceinline__ void split4(float4 v, float4& h, float4& l) {
    h.x = tf32_rna(v.x); l.x = tf32_rna(__fsub_rn(v.x, h.x));
    h.y = tf32_rna(v.y); l.y = tf32_rna(__fsub_rn(v.y, h.y));
    h.z = tf32_rna(v.z); l.z = tf32_rna(__fsub_rn(v.z, h.z));
    h.w = tf32_rna(v.w); l.w = tf32_rna(__fsub_rn(v.w, h.w));
}

// B raw tile -> hi (and lo unless EXACT) K-major canonical tiles.
template <int MN, bool EXACT>
__device__ __forceinline__ void split_b(const char* raw, int rows, char* hi, char* lo) {
    if (MN == 0) {
        for (int u = threadIdx.x; u < 128 * kKQ; u += kThreads) {  // consecutive threads: consecutive rows
            const int r = u & 127, kq = u >> 7;
            if (r >= rows) continue;
            const float4 v = *reinterpret_cast<const float4*>(raw + (r * kRawLdK + kq * 4) * 4);
            const uint32_t off = kq * kLbo + (r >> 3) * 128 + (r & 7) * 16;
            float4 h, l;
            split4(v, h, l);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
        }
    } else {
        const int quads = rows >> 2;
        for (int u = threadIdx.x; u < 32 * kKQ; u += kThreads) {  // 4 rows x 4 k per thread, transposed
            const int rq = u & 31, kq = u >> 5;
            if (rq >= quads) continue;
            float4 c[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                c[i] = *reinterpret_cast<const float4*>(raw + ((kq * 4 + i) * kRawLdMN + rq * 4) * 4);
            const float blk[4][4] = {{c[0].x, c[1].x, c[2].x, c[3].x},
                                     {c[0].y, c[1].y, c[2].y, c[3].y},
                                     {c[0].z, c[1].z, c[2].z, c[3].z},
                                     {c[0].w, c[1].w, c[2].w, c[3].w}};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = (i + (rq >> 1)) & 3;  // rotated order: conflict-free 16-byte stores
                const int r = rq * 4 + j;
                const uint32_t off = kq * kLbo + (r >> 3) * 128 + (r & 7) * 16;
                const float4 v = make_float4(blk[j][0], blk[j][1], blk[j][2], blk[j][3]);
                if (EXACT) {
                    *reinterpret_cast<float4*>(hi + off) = v;
                } else {
                    float4 h, l;
                    split4(v, h, l);
                    *reinterpret_cast<float4*>(hi + off) = h;
                    *reinterpret_cast<float4*>(lo + off) = l;
                }
            }
        }
    }
}

using tc::TcEpi;
using tc::kTcStore;
using tc::kTcBiasRelu;
using tc::kTcBias;
using tc::kTcMask;
using tc::kTcStoreT;

template <int AM, int BMODE, int EPI>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_ts_kernel(GemmArgs p, int /*unused*/) {
    extern __shared__ __align__(1024) char smem[];
    char* raw = smem;                                  // 2 x (A raw, B raw)
    char* hl = smem + 4 * kRawTile;                    // 2 x (B_hi, B_lo)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * kRawTile + 4 * kTile);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 4 * kRawTile + 4 * kTile + 32);

    const int slot = p.slots[blockIdx.z];
    const int bs = (p.m_is_bs || p.k_is_bs) ? slot_bs(p, slot) : 0;
    const int M = p.m_is_bs ? bs : p.M;
    const int K = p.k_is_bs ? bs : p.K;
    const int N = p.N;
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
    if (m0 >= M || n0 >= N) return;
    const int nt = min(kBN, (N - n0 + 15) / 16 * 16);  // MMA N of this tile
    const int nlim = min(N, n0 + kBN);
    const bool a_exact = p.a.from_data != 0;  // synthetic data k/128 is exact in tf32
    const bool b_exact = p.b.from_data != 0;
    const bool b_direct = b_exact && BMODE == 0;

    const float* A = opnd_ptr(p.a, slot, p.st, p.n_train_mask);
    const float* B = opnd_ptr(p.b, slot, p.st, p.n_train_mask);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int quad = warp & 3, kpart = warp >> 2;
    const int arow = m0 + quad * 32 + lane;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_tf32(nt);
    const uint32_t raw_u32 = smem_u32(raw), hl_u32 = smem_u32(hl);

    const int nchunks = (K + kKC - 1) / kKC;
    auto issue_b = [&](int c) {
        const int b = c & 1;
        load_b<AM, false>(A, p.a.ld, m0, kBM, M, c * kKC, K, raw_u32 + b * 2 * kRawTile, 0);
        if (b_direct)
            load_b<BMODE, true>(B, p.b.ld, n0, nt, nlim, c * kKC, K, 0, hl_u32 + b * 2 * kTile);
        else
            load_b<BMODE, false>(B, p.b.ld, n0, nt, nlim, c * kKC, K, raw_u32 + b * 2 * kRawTile + kRawTile, 0);
    };
    issue_b(0);
    asm volatile("cp.async.commit_group;");
    if (nchunks > 1) issue_b(1);
    asm volatile("cp.async.commit_group;");
    float a_cur[kAK];

#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        const int b = c & 1;
        asm volatile("cp.async.wait_group 1;");
        if (c >= 2) mbar_wait(&bars[b], ((c - 2) >> 1) & 1);  // MMAs of chunk c-2 released buffer b
        __syncthreads();
        // A: raw smem -> registers -> split -> TMEM (lane = row, column = k)
        read_a<AM>(raw + b * 2 * kRawTile, quad * 32 + lane, kpart * kAK, a_cur);
        {
            float hi[kAK], lo[kAK];
#pragma unroll
            for (int i = 0; i < kAK; ++i) {
                hi[i] = a_exact ? a_cur[i] : tf32_rna(a_cur[i]);
                lo[i] = tf32_rna(__fsub_rn(a_cur[i], hi[i]));
            }
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + 128 + b * 64 + kpart * kAK;
            tmem_st8(ta, hi);
            if (!a_exact) tmem_st8(ta + 32, lo);
            asm volatile("tcgen05.wait::st.sync.aligned;");
        }
        // B: split the landed raw tile into hi/lo canonical tiles
        if (!b_direct) {
            char* h = hl + b * 2 * kTile;
            if (b_exact)
                split_b<BMODE, true>(raw + b * 2 * kRawTile + kRawTile, nt, h, h + kTile);
            else
                split_b<BMODE, false>(raw + b * 2 * kRawTile + kRawTile, nt, h, h + kTile);
        }
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (c + 2 < nchunks) issue_b(c + 2);  // raw[b] consumed (or hl[b] reused only after MMAs)
        asm volatile("cp.async.commit_group;");
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t bhi = hl_u32 + b * 2 * kTile, blo = bhi + kTile;
            const uint32_t ahi = tmem + 128 + b * 64, alo = ahi + 32;
            const int ksteps = (min(kKC, K - c * kKC) + 7) / 8;
#pragma unroll 1
            for (int s = 0; s < ksteps; ++s) {
                const uint32_t o = s * 2 * kLbo;
                const uint64_t dbh = smem_desc(bhi + o, kLbo, 128), dbl = smem_desc(blo + o, kLbo, 128);
                uint32_t acc = (c == 0 && s == 0) ? 0u : 1u;
                if (!a_exact) {
                    mma_ts(tmem, alo + s * 8, dbh, idesc, acc);
                    acc = 1u;
                }
                if (!b_exact) {
                    mma_ts(tmem, ahi + s * 8, dbl, idesc, acc);
                    acc = 1u;
                }
                mma_ts(tmem, ahi + s * 8, dbh, idesc, acc);
            }
            mma_commit(&bars[b]);
        }
    }
    const int last = nchunks - 1;
    mbar_wait(&bars[last & 1], (last >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // ---- epilogue: warp w reads TMEM lanes 32*(w%4).., column half w/4 of the tile
    const int m = arow;
    const int cols = nt / kParts;  // multiple of 4
    float* C = p.c + p.c_stride * slot;
    const float* mask = (EPI == kTcMask) ? p.mask + p.mask_stride * slot : nullptr;
    float* bias = reinterpret_cast<float*>(raw);  // the tile's bias slice, staged once in smem
    if (EPI == kTcBiasRelu || EPI == kTcBias) {
        const float* gb = p.bias + p.bias_stride * slot;
        for (int j = threadIdx.x; j < nt; j += kThreads) bias[j] = n0 + j < N ? gb[n0 + j] : 0.0f;
        __syncthreads();
    }
    for (int c0 = kpart * cols; c0 < (kpart + 1) * cols; c0 += 4) {
        uint32_t v[4];
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (m >= M) continue;
        const int nb = n0 + c0;
        float x[4], mk[4] = {1.f, 1.f, 1.f, 1.f};
        if (EPI == kTcMask) {
            const float* mp = mask + (long long)m * p.ldmask + nb;
            if (nb + 4 <= N && (p.ldmask & 3) == 0) {
                const float4 t4 = __ldg(reinterpret_cast<const float4*>(mp));
                mk[0] = t4.x; mk[1] = t4.y; mk[2] = t4.z; mk[3] = t4.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) mk[j] = nb + j < N ? mp[j] : 0.0f;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] = __uint_as_float(v[j]);
            if (EPI == kTcBiasRelu) {
                x[j] = __fadd_rn(x[j], bias[c0 + j]);
                x[j] = x[j] > 0.0f ? x[j] : 0.0f;
            } else if (EPI == kTcBias) {
                x[j] = __fadd_rn(x[j], bias[c0 + j]);
            } else if (EPI == kTcMask) {
                x[j] = mk[j] > 0.0f ? x[j] : 0.0f;
            }
        }
        if (EPI == kTcStoreT) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (nb + j < N) C[(long long)(nb + j) * p.ldc + m] = x[j];
        } else if (nb + 4 <= N && (p.ldc & 3) == 0) {
            *reinterpret_cast<float4*>(C + (long long)m * p.ldc + nb) = make_float4(x[0], x[1], x[2], x[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (nb + j < N) C[(long long)m * p.ldc + nb + j] = x[j];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace tc3
}  // namespace smx
