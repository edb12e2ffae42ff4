// Warp-specialised implicit-GEMM convolution on tcgen05 (3xTF32), the tensor-core path of the
// CNN (replaces the lock-step conv_tc_kernel structure: no CTA-wide barrier per K chunk).
//
//   warps 0-7   producers: gather the A tile (128 rows x 32 k) and the B tile (N x 32 k) of a K
//               chunk from global memory through the Op's implicit-GEMM address functions,
//               split each value into tf32 hi/lo, write A hi/lo to TMEM (tcgen05.st, lane = row)
//               and B hi/lo to shared memory in the UMMA K-major canonical layout, then arrive
//               on the stage's `full` mbarrier.  3-stage ring; K-contiguous A tiles are
//               staged by coalesced cp.async (3 deep) and read back row-wise.
//   warp 12     MMA issuer (one elected thread): per chunk 3 (2 when an operand is exact in tf32)
//               tcgen05.mma kind::tf32 per 8-k step into the tile's TMEM accumulator, commit
//               -> the stage's `empty` barrier; after a tile's last chunk commit -> `acc_full`.
//   warps 8-11  epilogue: tcgen05.ld the accumulator (lane quadrant = warp % 4), release it
//               (`acc_empty`), apply bias+ReLU / ReLU-mask / transposed partial store.
// Two TMEM accumulators alternate between consecutive accumulation units — M tiles, or for the
// weight gradients (Op::kSegChunks > 0) segments of kSegChunks chunks of one tile — so draining
// one unit overlaps the MMAs of the next.  Segmented units are added into an fp32 tile in shared
// memory with round-to-nearest adds: the tensor core's fp32 accumulation is not
// round-to-nearest, and over the 2048-row weight-gradient reductions its error grows to ~4e-5;
// promoting every 64 products keeps the result at fp32 accuracy.
// TMEM columns: acc0 [0,128), acc1 [128,256), A stages [256 + 64 s, +64) (hi at +0, lo at +32).
// Shared memory: 3 B stages (hi, lo; 32 KB) | 3 raw A tiles (18 KB) | barriers | segment sums (64 KB).
// Results depend only on the group's own operands and the fixed tile/chunk order: deterministic
// and grouping-invariant like every executor kernel.
#pragma once

#include <type_traits>

#include "cnn.cuh"

namespace smx {
namespace cnn {
namespace ws {

using namespace smx::tc3;

constexpr int kMaxStages = 4;                    // B smem / A TMEM ring (TMEM: 4 x 64 columns)
constexpr int kProducers = 256;                  // warps 0-7
constexpr int kEpiWarp0 = 8;                     // warps 8.. : Op::kEpiWarps epilogue warps (4 or 8),
                                                 // then the MMA warp
constexpr int kBTile = kKQ * 128 * 16;           // B hi (or lo) tile, compact K-major canonical, N <= 128
constexpr int kARawTile = kBM * kKC * 4;         // raw A tile, 16 KB: [128 rows][32 k] (16-B units
                                                 // XOR-swizzled by row) or [32 k][128 rows]

// Ops with kTmaOut (the input gradients): the epilogue adds a tile's segments straight into the
// segment-sum area laid out as the tile's TMA output boxes (Op::stage16; thread = row x 64
// columns), the segment completing a column masks it, and tensor stores write the tile
// (Op::store_tile)
template <class Op, class = void>
struct TmaOut {
    static constexpr bool value = false;
};
template <class Op>
struct TmaOut<Op, std::void_t<decltype(Op::kTmaOut)>> {
    static constexpr bool value = Op::kTmaOut;
};

// Ops with kANbrBox (the conv2 input gradient): chunk c of a tile reads output neighbour c % 4 of
// channels 32 (c / 4) ..; one TMA box (Op::kABoxBytes: the tile's rows + one row and column of
// neighbours) feeds those 4 chunks from one raw slot (Op::a_line(row, c) = the row's 128-byte
// line), released by the 8 producer warps after their last chunk of it.  Op::chunk_k0(c) is the
// chunk's reduction offset.
template <class Op, class = void>
struct ANbrBox {
    static constexpr bool value = false;
    static constexpr int bytes = 0;
};
template <class Op>
struct ANbrBox<Op, std::void_t<decltype(Op::kANbrBox)>> {
    static constexpr bool value = Op::kANbrBox;
    static constexpr int bytes = Op::kABoxBytes;
};
template <class Op>
__device__ __forceinline__ int chunk_k0(const Op& op, int c) {
    if constexpr (ANbrBox<Op>::value) return op.kbeg + Op::chunk_k0(c); else return op.kbeg + c * kKC;
}

// Shared-memory plan of one Op, sized by its N (the B tiles and the segment sums scale with it):
// kStages B stages | kARaw raw A tiles | barriers | segment sums.  The raw-A ring takes what is
// left of the 227 KB (at most 8 deep): the prefetch distance is kARaw - 1 chunks.
template <class Op>
struct WsPlan {
    static constexpr int N = Op::kMaxN;
    static constexpr int Stages = N >= 128 ? 3 : kMaxStages;
    static constexpr int BStage = N * 256;                          // hi + lo tiles
    static constexpr int Sacc = kBM * N * 4;                        // tile sums [row][N], 16-B units
                                                                    // XOR-swizzled by row
    // masked epilogues reading the ReLU mask as a bitmap stage the tile's words in shared memory
    static constexpr int MaskWords = (Op::EPI == 1 && Op::kMaskFromBits && !TmaOut<Op>::value) ? kBM * N / 32 : 0;
    static constexpr int BarBytes = TmaOut<Op>::value ? 1024 : 512;  // (a staged TMA box starts 1 KB-aligned)
    static constexpr int Fixed = Stages * BStage + BarBytes + Sacc + MaskWords * 4;
    // raw A slot: one chunk's tile, or (ANbrBox) one neighbour box of 4 chunks (1 KB-aligned)
    static constexpr int ARawTile = ANbrBox<Op>::value ? (ANbrBox<Op>::bytes + 1023) / 1024 * 1024 : kARawTile;
    static constexpr int ARawMax = (227 * 1024 - Fixed) / ARawTile;
    // two producer groups take alternate chunks; each prefetches ARaw/2 - 1 of its own chunks
    static constexpr int ARaw = ANbrBox<Op>::value ? (ARawMax > 8 ? 8 : ARawMax) : (ARawMax > 8 ? 8 : ARawMax) & ~1;
    static_assert(ARaw >= (ANbrBox<Op>::value ? 2 : 4), "shared memory plan");
    static constexpr int ARawOff = Stages * BStage;
    static constexpr int BarOff = ARawOff + ARaw * ARawTile;
    static constexpr int SaccOff = BarOff + BarBytes;
    static constexpr int MbitsOff = SaccOff + Sacc;
    static constexpr int Bytes = MbitsOff + MaskWords * 4;
    static_assert(!TmaOut<Op>::value || SaccOff % 1024 == 0, "staging box alignment");
    // epilogue: one warp per TMEM lane quadrant (4), or two each draining half the columns (8)
    static constexpr int EpiWarps = Op::kEpiWarps;
    static_assert(EpiWarps == 4 || EpiWarps == 8, "epilogue warps");
    static constexpr int EpiThreads = EpiWarps * 32;
    static constexpr int MmaWarp = kEpiWarp0 + EpiWarps;
    // TMA A operands: one more warp whose elected lane streams the A boxes of every chunk into the
    // raw ring as soon as the group that read a slot has released it
    static constexpr int TmaWarp = Op::A_TMA ? MmaWarp + 1 : -1;
    // TMA B operands (Op::B_TMA): one more warp whose elected lane loads each chunk's B tile
    // straight into its stage as soon as the stage's previous MMAs are done
    static constexpr int BTmaWarp = Op::B_TMA ? MmaWarp + 1 + (Op::A_TMA ? 1 : 0) : -1;
    static constexpr int Threads = (MmaWarp + 1 + (Op::A_TMA ? 1 : 0) + (Op::B_TMA ? 1 : 0)) * 32;
};
template <class Op>
constexpr int ws_smem() {
    return WsPlan<Op>::Bytes;
}
constexpr int kWsTmemCols = 512;

// Ops whose B tiles have all-zero row blocks for some K chunks (the sub-pixel input gradients: 7 of
// the 16 (parity class, output neighbour) blocks hold no tap) declare kColRanges and
// chunk_cols(k0, off, n): the chunk's MMAs then cover only accumulator columns [off, off + n)
// (a narrower N); the first chunk of every accumulation segment covers all the segment's columns,
// and the epilogue adds only those.
template <class Op, class = void>
struct ColRanges {
    static constexpr bool value = false;
};
template <class Op>
struct ColRanges<Op, std::void_t<decltype(Op::kColRanges)>> {
    static constexpr bool value = Op::kColRanges;
};
// Ops with kPool (the conv3 forward): the bias+ReLU epilogue emits per-sample channel sums (64
// rows = one sample, x 2^-6; a fixed order: 8 row classes r % 8, each ascending) and the tile's
// value > 0 bitmap instead of the activation tile itself
template <class Op, class = void>
struct PoolOp {
    static constexpr bool value = false;
};
template <class Op>
struct PoolOp<Op, std::void_t<decltype(Op::kPool)>> {
    static constexpr bool value = Op::kPool;
};
constexpr int kAcc = 128;                        // columns per accumulator
constexpr int kABase = 256;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ float4 ld4(const float* p) {
    return p ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
}

template <bool EXACT>
__device__ __forceinline__ void split1(float a, float& h, float& l) {
    h = EXACT ? a : tf32_rna(a);
    l = tf32_rna(__fsub_rn(a, h));
}

#ifdef SMX_DBG_NO_BREG
constexpr bool kDbgNoBreg = true;  // profiling variant: skip the register-path B operand
#else
constexpr bool kDbgNoBreg = false;
#endif

// MMA issue from a whole warp: descriptors stay warp-uniform (uniform registers, no per-MMA
// R2UR moves) and elect.sync picks the issuing lane.  Measured (profiles/micro/mma_rate.cu):
// 12 tf32 MMAs per chunk at N = 64 take 384 cycles this way vs ~870 from a single thread.
__device__ __forceinline__ void mma_ts_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_e(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(bytes));
}

// 1-D bulk async copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// hi = the fp32 value itself (the tensor core reads the top 19 bits of a kind::tf32 operand, i.e.
// truncates), lo = a - trunc_tf32(a) (exact; its own low bits are truncated again by the MMA):
// two instructions per element instead of rna/sub/rna.
__device__ __forceinline__ float lo_of(float a) { return __fsub_rn(a, __uint_as_float(__float_as_uint(a) & 0xFFFFE000u)); }

#ifdef SMX_DBG_TIMELINE
// profiling variant: clock64 timeline of one CTA ((0, 1, 1)) of the first launch after the host
// arms it (smx_dbg_timeline): producer lanes 0 of warps 0 / 4 per chunk [0, 1024), MMA lane per
// chunk [1024, 1536), epilogue warp 0 lane 0 per segment / tile [2048, 4096)
__device__ unsigned long long smx_tl[4096];
__device__ int smx_tl_armed;
#define SMX_TL(i, cond) do { if (tl_on && (cond) && (i) < 4096) smx_tl[(i)] = clock64(); } while (0)
#else
#define SMX_TL(i, cond) do { } while (0)
#endif

template <class Op>
__global__ void __launch_bounds__(WsPlan<Op>::Threads, 1) conv_ws_kernel(typename Op::Args p, int tiles) {
    extern __shared__ __align__(1024) char smem[];
    using Plan = WsPlan<Op>;
    constexpr int kBStage = Plan::BStage, kARaw = Plan::ARaw, kPre = Plan::ARaw - 1;  // prefetch distance
    constexpr int kStages = Plan::Stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Plan::BarOff);
    uint64_t* empty = full + kStages;
    uint64_t* accf = empty + kStages;
    uint64_t* acce = accf + 2;
    uint64_t* rawf = acce + 2;  // TMA A operands: raw slot filled (expect_tx) / released by the group's 4 warps
    uint64_t* rawe = rawf + 8;
    uint64_t* bfull = rawe + 8;  // TMA B operands: the stage's hi tile landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + kMaxStages);

    Op op;
    op.setup(p, blockIdx.z, blockIdx.x);
    const int M = op.M, N = op.N, K = op.K;
    const int tile0 = blockIdx.y * tiles;
    const int ntiles = min(tiles, (M + kBM - 1) / kBM - tile0);
    if (ntiles <= 0 || K <= 0) return;
    const int nt = (N + 15) / 16 * 16;
    const int lbo = nt * 16;  // B canonical: (row r, k) at (k/4)*lbo + (r/8)*128 + (r%8)*16 + (k%4)*4
    const int nchunks = (K + kKC - 1) / kKC;
    const int total = ntiles * nchunks;
    const int klim = op.kbeg + K;
    const int seg = Op::kSegChunks;  // 0: one accumulation unit per tile
    const int nseg = seg > 0 ? (nchunks + seg - 1) / seg : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kWsTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 128 + (Op::B_IMAGE ? 1 : 0));  // one producer group (+ the bulk copy)
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&accf[a], 1);
            mbar_init(&acce[a], Plan::EpiThreads);
        }
        if constexpr (Op::A_TMA)
            for (int r = 0; r < kARaw; ++r) {
                mbar_init(&rawf[r], 1);
                mbar_init(&rawe[r], ANbrBox<Op>::value ? 8 : 4);
            }
        if constexpr (Op::B_TMA)
            for (int st = 0; st < kStages; ++st) mbar_init(&bfull[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
#ifdef SMX_DBG_TIMELINE
    int& tl_flag = reinterpret_cast<int*>(tmem_slot)[1];  // spare word of the barrier area
    if (threadIdx.x == 0)
        tl_flag = (blockIdx.x == 0 && blockIdx.y == 1 && blockIdx.z == 1) ? atomicExch(&smx_tl_armed, 0) : 0;
    __syncthreads();
    const bool tl_on = tl_flag != 0;
    if (tl_on && threadIdx.x == 0) smx_tl[4095] = clock64();
#endif

    if (warp < kEpiWarp0) {
        // ================= producers =================
        // Two groups of four warps (one per TMEM lane quadrant) take alternate K chunks, so two
        // chunks are in flight; within a group warp q owns rows 32q..32q+31 and all 32 k.
        const int grp = warp >> 2, q = warp & 3;
        const int gt = threadIdx.x & 127;  // thread within the group
        constexpr int kDw = kARaw / 2 - 1; // own chunks prefetched ahead
        const uint32_t araw = smem_u32(smem + Plan::ARawOff);
        typename Op::RowInfo ri[8];
        // prefetch cursor over this group's chunks (g = grp, grp + 2, ...): tile, chunk, slot
        int pf_g = grp, pf_tile = 0, pf_chunk = grp, pf_slot = grp, ri_tile = -1;
        while (pf_chunk >= nchunks) { pf_chunk -= nchunks; ++pf_tile; }
        auto a_issue = [&]() {
            if (pf_g < total) {
                const int mm0 = (tile0 + pf_tile) * kBM, kk0 = op.kbeg + pf_chunk * kKC;
                const uint32_t dst = araw + pf_slot * kARawTile;
                if constexpr (Op::A_TMA) {
                    // issued by the TMA warp
                } else if constexpr (Op::AM == 0) {
                    // unit j: row 32q + lane/8 + 4j, k-quad lane%8 (8 lanes = one row's 128 bytes)
                    if (pf_tile != ri_tile) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) ri[j] = op.row_info(mm0 + q * 32 + (lane >> 3) + 4 * j);
                        ri_tile = pf_tile;
                    }
                    const int kq = lane & 7;
                    const auto tap = op.tap_info(kk0 + kq * 4);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int r = q * 32 + (lane >> 3) + 4 * j;
                        const float* src = op.a_ptr_tap(ri[j], tap);
#ifdef SMX_DBG_NO_LOAD
                        src = nullptr;
#endif
                        cp16(dst + r * 128 + ((kq ^ (r & 7)) << 4), src ? src : ctc::kZero16, src ? 16 : 0);
                    }
                } else {
                    // MN-contiguous A: unit j = (row quad 8q + lane%8, k = 8 (lane/8) + j): each lane walks
                    // 8 consecutive reduction indices (one decode, then a pointer stride)
                    const int rq = q * 8 + (lane & 7);
                    if (pf_tile != ri_tile) {
                        ri[0] = op.row_info(mm0 + rq * 4);
                        ri_tile = pf_tile;
                    }
                    const int kb = (lane >> 3) * 8;
                    const auto rd = op.red_info(kk0 + kb);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int k = kb + j;
                        const float* src = op.a_ptr_red_step(ri[0], rd, j);
#ifdef SMX_DBG_NO_LOAD
                        src = nullptr;
#endif
                        cp16(dst + k * 512 + rq * 16, src ? src : ctc::kZero16, src ? 16 : 0);
                    }
                }
            }
            if constexpr (!Op::A_TMA) asm volatile("cp.async.commit_group;");
            pf_g += 2;
            pf_chunk += 2;
            while (pf_chunk >= nchunks) { pf_chunk -= nchunks; ++pf_tile; }
            pf_slot += 2;
            if (pf_slot >= kARaw) pf_slot -= kARaw;
        };
#ifdef SMX_DBG_MMA_ONLY
        // profiling variant: producers only hand stages to the MMA (B image still copied)
        for (int g = grp; g < total; g += 2) {
            const int s = g % kStages, u = g / kStages;
            if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
            if constexpr (Op::B_IMAGE) {
                if (gt == 0) {
                    int cc = g % nchunks;
                    mbar_arrive_expect_tx(&full[s], nt * 256);
                    bulk_g2s(smem + s * kBStage, op.b_image(cc), nt * 256, &full[s]);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&full[s]);
        }
#else
        for (int j = 0; j < kDw; ++j) a_issue();
        int i = 0, c = grp, rd_slot = grp;
        while (c >= nchunks) { c -= nchunks; ++i; }
        for (int g = grp; g < total; g += 2) {
            const int s = g % kStages, u = g / kStages;
            SMX_TL(g * 8 + 0, gt == 0);
            const int m = (tile0 + i) * kBM + q * 32 + lane;
            const int k0 = chunk_k0(op, c);
            // B (register path, non-image Ops): the group's 128 threads cover the tile
            float4 b[8];
#ifdef SMX_DBG_NO_BREG
            if constexpr (false) {
#else
            if constexpr (!Op::B_IMAGE && Op::BMODE == 0) {
#endif
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int uu = gt + j * 128, r = uu % nt, kq = uu / nt, k = k0 + kq * 4;
                    b[j] = ld4(kq < kKQ && r < N && k < klim ? op.b_ptr(r, k) : nullptr);
                }
            } else if constexpr (!Op::B_IMAGE && !Op::B_TMA && !kDbgNoBreg) {
                // MN-contiguous B: unit (row r, k quad) = 4 scalar loads down the reduction index;
                // lanes = consecutive rows, so each load is one coalesced 128-byte line and the
                // unit is already the K-major 16-byte group (no transpose)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int uu = gt + j * 128, r = uu % nt, kq = uu / nt, k = k0 + kq * 4;
                    const bool ok = kq < kKQ && r < N;
                    b[j].x = ok && k < klim ? __ldg(op.b_ptr(r, k)) : 0.0f;
                    b[j].y = ok && k + 1 < klim ? __ldg(op.b_ptr(r, k + 1)) : 0.0f;
                    b[j].z = ok && k + 2 < klim ? __ldg(op.b_ptr(r, k + 2)) : 0.0f;
                    b[j].w = ok && k + 3 < klim ? __ldg(op.b_ptr(r, k + 3)) : 0.0f;
                }
            }
            // warm L2 with the B rows of this group's chunk kDw + 1 ahead (register-path B)
            if constexpr (!Op::B_IMAGE && !Op::B_TMA) {
                int pc = c + 2 * (kDw + 1);
                while (pc >= nchunks) pc -= nchunks;
                if (g + 2 * (kDw + 1) < total) {
                    const int pk = op.kbeg + pc * kKC;
                    if constexpr (Op::BMODE == 1) {  // rows = reduction index: 32 contiguous rows of the tile
                        const int kk = pk + (gt >> 2);
                        if (gt < 128 && kk < klim) prefetch_l2(op.b_ptr((gt & 3) * 32, kk));
                    } else {  // rows = n: one line per 32 k of each row
                        if (gt < nt && pk < klim) prefetch_l2(op.b_ptr(gt, pk));
                    }
                }
            }
            float a[32];
            // raw slot of this chunk (neighbour boxes: one per 4 chunks)
            const int a_slot = ANbrBox<Op>::value ? (g >> 2) % kARaw : rd_slot;
            if constexpr (ANbrBox<Op>::value)
                mbar_wait(&rawf[a_slot], ((g >> 2) / kARaw) & 1);
            else if constexpr (Op::A_TMA)
                mbar_wait(&rawf[rd_slot], ((((g - grp) >> 1) / (kARaw / 2)) & 1));
            else if constexpr (kDw > 1)
                asm volatile("cp.async.wait_group %0;" ::"n"(kDw - 1) : "memory");  // own copies of chunk g
            else
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            SMX_TL(g * 8 + 1, gt == 0);
            {
                const char* rawg = smem + Plan::ARawOff + a_slot * Plan::ARawTile;
                const int r = q * 32 + lane;
                if constexpr (ANbrBox<Op>::value) {
                    // the row's line of the neighbour box (128B-swizzled by line)
                    const int ln = op.a_line(r, c);
#pragma unroll
                    for (int kq = 0; kq < 8; ++kq) {
                        const float4 t = *reinterpret_cast<const float4*>(rawg + ln * 128 + ((kq ^ (ln & 7)) << 4));
                        a[4 * kq] = t.x; a[4 * kq + 1] = t.y; a[4 * kq + 2] = t.z; a[4 * kq + 3] = t.w;
                    }
                } else if constexpr (Op::AM == 0) {
#pragma unroll
                    for (int kq = 0; kq < 8; ++kq) {
                        const float4 t = *reinterpret_cast<const float4*>(rawg + r * 128 + ((kq ^ (r & 7)) << 4));
                        a[4 * kq] = t.x; a[4 * kq + 1] = t.y; a[4 * kq + 2] = t.z; a[4 * kq + 3] = t.w;
                    }
                } else if constexpr (Op::A_TMA) {
                    // [tap][pixel k][ci] boxes: lanes = consecutive channels (conflict-free)
                    const float* rp = reinterpret_cast<const float*>(rawg) + (r / Op::kTmaCi) * (32 * Op::kTmaCi) +
                                      r % Op::kTmaCi;
#pragma unroll
                    for (int k = 0; k < 32; ++k) a[k] = rp[k * Op::kTmaCi];
                } else {
                    const float* rp = reinterpret_cast<const float*>(rawg) + r;
#pragma unroll
                    for (int k = 0; k < 32; ++k) a[k] = rp[k * 128];
                }
            }
            __syncwarp();  // this warp's reads of the slot precede the refill below
            // (TMA operands: the slot is released only once the loaded registers have been
            // consumed by the TMEM stores below; an arrive right after the LDS instructions could
            // overtake loads still in flight, and the TMA warp would refill the slot under them)
            SMX_TL(g * 8 + 5, gt == 0);
            a_issue();
            rd_slot += 2;
            if (rd_slot >= kARaw) rd_slot -= kARaw;
            if (Op::kOnesRow >= 0 && m == Op::kOnesRow) {
#pragma unroll
                for (int j = 0; j < 32; ++j) a[j] = k0 + j < klim ? 1.0f : 0.0f;
            }
            if constexpr (Op::kInMaskBits) {
                if (uint32_t* wdst = op.in_bits_word(m, k0)) {
                    uint32_t wbits = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) wbits |= (a[j] > 0.0f ? 1u : 0u) << j;
                    *wdst = wbits;
                }
            }
            // ---- wait until the MMAs of this stage's previous use are done
            SMX_TL(g * 8 + 2, gt == 0);
            if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
            SMX_TL(g * 8 + 3, gt == 0);
            char* bh = smem + s * kBStage;
            char* bl = bh + nt * 128;
            if constexpr (Op::B_IMAGE) {
                if (gt == 0) {  // the weight image of this chunk: one bulk copy of hi | lo
#ifdef SMX_DBG_NO_BIMG  // profiling variant: no weight-image copies (B = whatever the stage holds)
                    mbar_arrive(&full[s]);
#else
                    mbar_arrive_expect_tx(&full[s], nt * 256);
                    bulk_g2s(bh, op.b_image(c), nt * 256, &full[s]);
#endif
                }
            }
            // A hi/lo -> TMEM (lane = row, column = k)
#ifndef SMX_DBG_NO_ASTORE
            {
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + kABase + s * 64;
                tmem_st16(ta, a);
                tmem_st16(ta + 16, a + 16);
                if (!Op::A_EXACT) {
                    float lo[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) lo[j] = lo_of(a[j]);
                    tmem_st16(ta + 32, lo);
                    tmem_st16(ta + 48, lo + 16);
                }
            }
#endif
            // B hi/lo -> smem canonical
            if constexpr (kDbgNoBreg) {
            } else if constexpr (Op::B_TMA) {
                // the TMA wrote the hi tile (the fp32 values: the MMA truncates them to tf32) in
                // the MN-major 128B/32B-atom swizzled layout; lo = b - trunc(b) element by
                // element lands at the same (swizzled) positions of the lo tile
                mbar_wait(&bfull[s], u & 1);
                const float4* hi4 = reinterpret_cast<const float4*>(bh);
                float4* lo4 = reinterpret_cast<float4*>(bl);
#pragma unroll 4
                for (int j = gt; j < nt * kKC / 4; j += 128) {
                    const float4 v = hi4[j];
                    lo4[j] = make_float4(lo_of(v.x), lo_of(v.y), lo_of(v.z), lo_of(v.w));
                }
            } else if constexpr (!Op::B_IMAGE) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int uu = gt + j * 128, r = uu % nt, kq = uu / nt;
                    if (kq < kKQ) {
                        const uint32_t off = kq * lbo + (r >> 3) * 128 + (r & 7) * 16;
                        *reinterpret_cast<float4*>(bh + off) = b[j];
                        *reinterpret_cast<float4*>(bl + off) =
                            make_float4(lo_of(b[j].x), lo_of(b[j].y), lo_of(b[j].z), lo_of(b[j].w));
                    }
                }
            }
            SMX_TL(g * 8 + 6, gt == 0);
            asm volatile("tcgen05.wait::st.sync.aligned;");
            SMX_TL(g * 8 + 4, gt == 0);
            if constexpr (Op::A_TMA) {
                __syncwarp();
                if (lane == 0 && (!ANbrBox<Op>::value || (g & 3) >= 2)) mbar_arrive(&rawe[a_slot]);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;");
            asm volatile("fence.proxy.async.shared::cta;");
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&full[s]);
            c += 2;
            while (c >= nchunks) { c -= nchunks; ++i; }
        }
#endif
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else if (warp == Plan::TmaWarp) {
        // ================= TMA producer of the A operands (one elected lane) =================
        // chunk g (group g % 2) goes to raw slot g % ARaw; the slot's previous chunk g - ARaw
        // must have been released by the 4 warps of its group
        if constexpr (Op::A_TMA) {
            if (lane == 0) {
                constexpr int kBoxBytes = kARawTile / Op::kBoxes;
                const uint32_t araw = smem_u32(smem + Plan::ARawOff);
                if constexpr (ANbrBox<Op>::value) {
                    // one neighbour box per 4 chunks of a tile
                    const int per_tile = nchunks / 4;
                    for (int u = 0; u < total / 4; ++u) {
                        const int slot = u % kARaw, use = u / kARaw;
                        if (use > 0) mbar_wait(&rawe[slot], (use - 1) & 1);
                        const uint32_t bar = smem_u32(&rawf[slot]), dst = araw + slot * Plan::ARawTile;
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                                     "r"(ANbrBox<Op>::bytes));
                        int cc[4];
                        op.a_box(tile0 + u / per_tile, u % per_tile, cc);
                        asm volatile(
                            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
                            "l"(op.tmap), "r"(cc[0]), "r"(cc[1]), "r"(cc[2]), "r"(cc[3]), "r"(bar)
                            : "memory");
                    }
                } else {
                int tile = 0, c = 0;
                for (int g = 0; g < total; ++g) {
                    const int slot = g % kARaw, use = g / kARaw;
                    if (use > 0) mbar_wait(&rawe[slot], (use - 1) & 1);
                    const int nbox = op.a_nbox(tile0 + tile);  // boxes past the operand are skipped
                    const uint32_t bar = smem_u32(&rawf[slot]), dst = araw + slot * kARawTile;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                                 "r"(nbox * kBoxBytes));
                    for (int b = 0; b < nbox; ++b) {
                        int cc[4];
                        op.a_coords(tile0 + tile, op.kbeg + c * kKC, b, cc);
                        asm volatile(
                            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst + b * kBoxBytes),
                            "l"(op.tmap), "r"(cc[0]), "r"(cc[1]), "r"(cc[2]), "r"(cc[3]), "r"(bar)
                            : "memory");
                    }
                    if (++c == nchunks) { c = 0; ++tile; }
                }
                }
            }
            __syncwarp();
        }
    } else if (warp == Plan::BTmaWarp) {
        // ================= TMA producer of the B operands (one elected lane) =================
        // chunk g's B tile (nt channels x 32 reduction rows, nt / 32 swizzled 4 KB boxes) goes to
        // stage g % kStages once the MMAs of the stage's previous chunk have completed
        if constexpr (Op::B_TMA) {
            if (lane == 0) {
                int c = 0;
                for (int g = 0; g < total; ++g) {
                    const int s = g % kStages, u = g / kStages;
                    if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
                    const uint32_t bar = smem_u32(&bfull[s]), dst = smem_u32(smem + s * kBStage);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nt * kKC * 4));
                    const int row = op.kbeg + c * kKC;
                    for (int b = 0; b < nt / 32; ++b)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + b * 4096),
                            "l"(op.btmap), "r"(32 * b), "r"(row), "r"(bar)
                            : "memory");
                    if (++c == nchunks) c = 0;
                }
            }
            __syncwarp();
        }
    } else if (warp == Plan::MmaWarp) {
        // ================= MMA issuer (whole warp, elected lane issues) =================
        {
            // TMA B operands are MN-major (instruction descriptor bit 16)
            const uint32_t idesc = idesc_tf32(nt) | (Op::B_TMA ? (1u << 16) : 0u);
            const uint32_t smem_base = smem_u32(smem);
            int g = 0, un = 0;
            for (int i = 0; i < ntiles; ++i) {
                uint32_t dacc = 0;
                int acc_i = 0;
                for (int c = 0; c < nchunks; ++c, ++g) {
                    const bool unit_start = c == 0 || (seg > 0 && c % seg == 0);
                    const bool unit_end = c == nchunks - 1 || (seg > 0 && c % seg == seg - 1);
                    if (unit_start) {
                        acc_i = un & 1;
                        const int use = un >> 1;
                        if (use > 0) mbar_wait(&acce[acc_i], (use - 1) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        dacc = tmem + acc_i * kAcc;
                    }
                    const int s = g % kStages, u = g / kStages;
                    SMX_TL(1024 + g * 4 + 0, lane == 0);
                    mbar_wait(&full[s], u & 1);
                    SMX_TL(1024 + g * 4 + 1, lane == 0);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t bhi = smem_base + s * kBStage, blo = bhi + nt * 128;
                    const uint32_t ahi = tmem + kABase + s * 64, alo = ahi + 32;
                    const int ksteps = (min(kKC, klim - chunk_k0(op, c)) + 7) / 8;
                    // accumulator columns of this chunk (all of them unless the Op skips zero blocks)
                    int coff = 0, cn = nt;
                    if constexpr (ColRanges<Op>::value) op.chunk_cols(chunk_k0(op, c), coff, cn);
                    const uint32_t idc = ColRanges<Op>::value ? idesc_tf32(cn) | (Op::B_TMA ? (1u << 16) : 0u) : idesc;
                    const uint32_t dac = dacc + coff;
                    // descriptors built once per chunk; a k-step of 8 tf32 advances the B tiles by
                    // 2 LBO (the 14-bit address field cannot overflow below 256 KB of smem)
                    // (TMA B: MN-major SWIZZLE_128B_BASE32B -- LBO = 4 KB between 32-column atoms,
                    // SBO = 512 B between 4-row k groups; a k-step of 8 rows advances 1 KB)
                    // (a column range starts coff rows into the K-major B tile: + coff x 16 bytes)
                    const uint64_t dbh0 = (Op::B_TMA ? smem_desc_mn32(bhi, 4096, 512) : smem_desc(bhi, lbo, 128)) + coff;
                    const uint64_t dbl0 = (Op::B_TMA ? smem_desc_mn32(blo, 4096, 512) : smem_desc(blo, lbo, 128)) + coff;
                    const uint64_t dstep = Op::B_TMA ? (uint64_t)(1024 >> 4) : (uint64_t)((2 * lbo) >> 4);
#ifndef SMX_DBG_NO_MMA
                    if (ksteps == 4) {
#pragma unroll
                        for (int st = 0; st < 4; ++st) {
                            const uint64_t dbh = dbh0 + st * dstep, dbl = dbl0 + st * dstep;
                            const uint32_t a_off = st * 8;
                            if (!Op::A_EXACT) mma_ts_e(dac, alo + a_off, dbh, idc, (unit_start && st == 0) ? 0u : 1u);
                            if (!Op::B_EXACT)
                                mma_ts_e(dac, ahi + a_off, dbl, idc, (unit_start && st == 0 && Op::A_EXACT) ? 0u : 1u);
                            mma_ts_e(dac, ahi + a_off, dbh, idc,
                                   (unit_start && st == 0 && Op::A_EXACT && Op::B_EXACT) ? 0u : 1u);
                        }
                    } else {
                        for (int st = 0; st < ksteps; ++st) {
                            const uint64_t dbh = dbh0 + st * dstep, dbl = dbl0 + st * dstep;
                            uint32_t accum = (unit_start && st == 0) ? 0u : 1u;
                            if (!Op::A_EXACT) {
                                mma_ts_e(dac, alo + st * 8, dbh, idc, accum);
                                accum = 1u;
                            }
                            if (!Op::B_EXACT) {
                                mma_ts_e(dac, ahi + st * 8, dbl, idc, accum);
                                accum = 1u;
                            }
                            mma_ts_e(dac, ahi + st * 8, dbh, idc, accum);
                        }
                    }
#endif
                    SMX_TL(1024 + g * 4 + 2, lane == 0);
                    mma_commit_e(&empty[s]);
                    if (unit_end) {
                        mma_commit_e(&accf[acc_i]);
                        ++un;
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue =================
        const int q = warp & 3, ch = (warp - kEpiWarp0) >> 2;  // lane quadrant, column half
        static_assert(Op::kSegChunks > 0, "the epilogue stages every tile in shared memory");
        float* sacc = reinterpret_cast<float*>(smem + Plan::SaccOff);  // [row][PN], 16-B units swizzled
        constexpr int PN = Plan::N;
        // float4 unit (row r, column quad c4) of the tile sums
        auto s4 = [&](int r, int c4) -> float4* { return reinterpret_cast<float4*>(sacc + r * PN) + (c4 ^ (r & 7)); };
        const int row = q * 32 + lane;
        const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..EpiThreads-1
        // this warp's accumulator columns: half of the tile (all of it below 32 columns)
        const bool halves = Plan::EpiWarps == 8 && nt >= 32;
        const int cw = halves ? nt / 2 : (ch == 0 ? nt : 0), cbeg = halves ? ch * cw : 0;
        constexpr int kCW = Plan::EpiWarps == 8 ? Plan::N / 2 : Plan::N;  // most columns a warp drains
        // (register sums only where the register budget allows: the 13-warp kernels)
        constexpr bool kRegSum = Plan::EpiWarps == 4 && kCW <= 64 && kCW % 16 == 0;
        static_assert(!(kRegSum && ColRanges<Op>::value), "column ranges need the shared-memory segment sums");
        // TmaOut: which 32-column class blocks each segment writes (bit = block; its first chunk's
        // range, all blocks for the first segment) and the last segment writing each block
        uint32_t seg_cols = 0, last_seg = 0;  // 4 bits per segment (<= 8) / per block
        if constexpr (TmaOut<Op>::value) {
            static_assert(Plan::N == 128, "4 class blocks");
            for (int j = 0; j < nseg && j < 8; ++j) {
                int slo = 0, sn = nt;
                if constexpr (ColRanges<Op>::value)
                    if (j > 0) op.chunk_cols(chunk_k0(op, j * seg), slo, sn);
                for (int bb = 0; bb < 4; ++bb)
                    if (32 * bb < slo + sn && 32 * bb + 32 > slo) {
                        seg_cols |= 1u << (4 * j + bb);
                        last_seg = (last_seg & ~(15u << (4 * bb))) | ((uint32_t)j << (4 * bb));
                    }
            }
        }
        int un = 0;
        for (int i = 0; i < ntiles; ++i) {
            const int mt0 = (tile0 + i) * kBM;
            if constexpr (TmaOut<Op>::value) {
                // ---- segments summed straight into the staged output box, one TMA store per tile
                static_assert(Plan::EpiWarps == 8 && Plan::N == 128, "TMA-out epilogue mapping");
                const int m = mt0 + row;
                uint32_t mw[2];
#pragma unroll
                for (int cb = 0; cb < 2; ++cb) mw[cb] = m < M ? op.mask_word(m, cbeg + 32 * cb) : 0u;
                char* stg = smem + Plan::SaccOff;
                // the previous tile's store has finished reading the staging area
                if (et == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");
                for (int j = 0; j < nseg; ++j, ++un) {
                    const int acc_i = un & 1, use = un >> 1;
                    SMX_TL(2048 + un * 4 + 0, et == 0);
                    mbar_wait(&accf[acc_i], use & 1);
                    SMX_TL(2048 + un * 4 + 1, et == 0);
                    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
                    for (int cb = 0; cb < 2; ++cb) {
                        if (!((seg_cols >> (4 * j + 2 * ch + cb)) & 1u)) continue;
                        const int c0 = cbeg + 32 * cb;
                        const bool last = ((last_seg >> (4 * (2 * ch + cb))) & 15u) == (uint32_t)j;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint32_t r[16];
                            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc_i * kAcc + c0 + 16 * h, r);
                            asm volatile("tcgen05.wait::ld.sync.aligned;");
#ifndef SMX_DBG_NO_EPI
                            op.stage16(stg, row, c0 + 16 * h, r, j == 0, last, cb ? mw[1] : mw[0]);
#endif
                        }
                    }
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    mbar_arrive(&acce[acc_i]);
                }
                SMX_TL(3072 + i * 2 + 0, et == 0);
                asm volatile("fence.proxy.async.shared::cta;");  // generic stores -> the TMA's async proxy
                asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");
#ifndef SMX_DBG_NO_EPI
                if (et == 0) {
                    op.store_tile(smem_u32(stg), tile0 + i);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
#endif
                SMX_TL(3072 + i * 2 + 1, et == 0);
            } else {
            // bitmap masks: the tile's words are loaded now (in flight during the drains) and staged
            // in shared memory before the scatter
            constexpr int kMW = Plan::MaskWords > 0 ? Plan::MaskWords / Plan::EpiThreads : 1;
            uint32_t mword[kMW];
            if constexpr (Plan::MaskWords > 0) {
                static_assert(Plan::MaskWords % Plan::EpiThreads == 0, "mask-word mapping");
                constexpr int WPR = Plan::N / 32;  // words per row
#pragma unroll
                for (int j = 0; j < kMW; ++j) {
                    const int w = et + j * Plan::EpiThreads, m = mt0 + w / WPR;
                    mword[j] = m < M ? op.mask_word(m, 32 * (w % WPR)) : 0u;
                }
            } else if constexpr (Op::EPI == ctc::kEpiMask) {
                // warm L2 with the tile's ReLU-mask lines (one 128-byte line per 32 columns of a row)
                const int m = mt0 + row;
                if (m < M)
                    for (int col = 32 * ch; col < N; col += 32 * (Plan::EpiWarps / 4)) prefetch_l2(op.mask_at(m, col));
            } else if constexpr (Op::kSgd) {
                // SGD epilogue: warm L2 with the tile's parameters and momenta while the MMAs run
                const int m = mt0 + row;
                if (m < M)
                    for (int col = 32 * ch; col < N; col += 32 * (Plan::EpiWarps / 4)) {
                        prefetch_l2(op.w_at(m, col));
                        prefetch_l2(op.w_at(m, col) + op.m_off);
                    }
            }
            // sum the tile's segments (round-to-nearest fp32 adds, fixed order): in registers when
            // a warp drains at most 64 columns, then once into sacc; otherwise in sacc directly
            if constexpr (kRegSum) {
                float sum[kCW];
                for (int j = 0; j < nseg; ++j, ++un) {
                    const int acc_i = un & 1, use = un >> 1;
                    SMX_TL(2048 + un * 4 + 0, et == 0);
                    mbar_wait(&accf[acc_i], use & 1);
                    SMX_TL(2048 + un * 4 + 1, et == 0);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (cw == 0) {
                        asm volatile("tcgen05.fence::before_thread_sync;");
                        mbar_arrive(&acce[acc_i]);
                    }
#pragma unroll
                    for (int b16 = 0; b16 < kCW / 16; ++b16) {
                        if (16 * b16 < cw) {
                            uint32_t r[16];
                            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc_i * kAcc + cbeg + 16 * b16, r);
                            asm volatile("tcgen05.wait::ld.sync.aligned;");
                            if (16 * b16 + 16 >= cw) {
                                asm volatile("tcgen05.fence::before_thread_sync;");
                                mbar_arrive(&acce[acc_i]);
                            }
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj)
                                sum[16 * b16 + jj] = j == 0 ? __uint_as_float(r[jj]) : __fadd_rn(sum[16 * b16 + jj], __uint_as_float(r[jj]));
                        }
                    }
                }
                if constexpr (Op::EPI == ctc::kEpiPartT) {
#ifndef SMX_DBG_NO_EPI
                    // transposed outputs straight from registers: lanes = consecutive rows of one
                    // column (coalesced)
                    const int m = mt0 + row;
                    if (m < M) {
#pragma unroll
                        for (int cc = 0; cc < kCW; ++cc)
                            if (cc < cw && cbeg + cc < N) *op.ct_at(cbeg + cc, m) = sum[cc];
                    }
#endif
                    continue;
                } else {
#pragma unroll
                    for (int c4 = 0; c4 < kCW / 4; ++c4)
                        if (4 * c4 < cw)
                            *s4(row, (cbeg >> 2) + c4) = make_float4(sum[4 * c4], sum[4 * c4 + 1], sum[4 * c4 + 2], sum[4 * c4 + 3]);
                }
            } else {
                for (int j = 0; j < nseg; ++j, ++un) {
                    const int acc_i = un & 1, use = un >> 1;
                    SMX_TL(2048 + un * 4 + 0, et == 0);
                    mbar_wait(&accf[acc_i], use & 1);
                    SMX_TL(2048 + un * 4 + 1, et == 0);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (cw == 0) {  // nothing to drain for this warp: release at once
                        asm volatile("tcgen05.fence::before_thread_sync;");
                        mbar_arrive(&acce[acc_i]);
                    }
                    // columns written in this segment (Ops skipping zero blocks: the first chunk's range)
                    int slo = 0, shi = nt;
                    if constexpr (ColRanges<Op>::value) {
                        int sn;
                        op.chunk_cols(chunk_k0(op, j * seg), slo, sn);
                        shi = slo + sn;
                    }
                    // 32 columns per TMEM round trip (two loads in flight before one wait)
                    for (int c0 = cbeg; c0 < cbeg + cw; c0 += 32) {
                        uint32_t r[32];
                        const bool two = c0 + 16 < cbeg + cw;
                        const bool use = !ColRanges<Op>::value || (c0 < shi && c0 + 32 > slo);
                        if (use) {
                            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc_i * kAcc + c0, r);
                            if (two) tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc_i * kAcc + c0 + 16, r + 16);
                            asm volatile("tcgen05.wait::ld.sync.aligned;");
                        }
                        if (c0 + 32 >= cbeg + cw) {
                            asm volatile("tcgen05.fence::before_thread_sync;");
                            mbar_arrive(&acce[acc_i]);
                        }
                        if (!use) continue;
#pragma unroll
                        for (int jj = 0; jj < 32; jj += 4) {
                            if (jj >= 16 && !two) break;
                            float4* sp = s4(row, (c0 + jj) >> 2);
                            const float4 nv = make_float4(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1]),
                                                          __uint_as_float(r[jj + 2]), __uint_as_float(r[jj + 3]));
                            if (j == 0) {
                                *sp = nv;
                            } else {
                                float4 o = *sp;
                                o.x = __fadd_rn(o.x, nv.x);
                                o.y = __fadd_rn(o.y, nv.y);
                                o.z = __fadd_rn(o.z, nv.z);
                                o.w = __fadd_rn(o.w, nv.w);
                                *sp = o;
                            }
                        }
                    }
                }
            }
            SMX_TL(3072 + i * 2 + 0, et == 0);
#ifndef SMX_DBG_NO_EPI
            if constexpr (Op::EPI == ctc::kEpiBiasRelu || Op::EPI == ctc::kEpiBias || Op::EPI == ctc::kEpiStore) {
                // row-major output tile: cooperative, coalesced write-out, consecutive threads =
                // consecutive 16 bytes of a row
                asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");  // the whole tile is in sacc
                const int q4 = N / 4;
                // the thread's column quad is fixed when the stride is a multiple of the row
                // length: its bias quad is then loaded once per tile
                const bool fixed_c4 = Plan::EpiThreads % q4 == 0;
                float4 bfix = make_float4(0.f, 0.f, 0.f, 0.f);
                if constexpr (Op::EPI != ctc::kEpiStore)
                    if (fixed_c4) bfix = op.bias4(4 * (et % q4));
                if constexpr (Op::kSgd) {
                    // K3+K5: the tile is the weight gradient; apply the update to w | m in place,
                    // U quads per thread with their loads issued before any use
                    constexpr int U = 4;
                    if ((op.ldc & 3) == 0 && (N & 3) == 0) {
                        for (int e0 = et; e0 < kBM * q4; e0 += U * Plan::EpiThreads) {
                            float4 wv[U], mv[U];
                            float* wp[U];
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                const int e = e0 + u * Plan::EpiThreads, r = e / q4, c4 = e % q4, m = mt0 + r;
                                wp[u] = (e < kBM * q4 && m < M) ? op.w_at(m, 4 * c4) : nullptr;
                                if (wp[u]) {
                                    wv[u] = *reinterpret_cast<const float4*>(wp[u]);
                                    mv[u] = *reinterpret_cast<const float4*>(wp[u] + op.m_off);
                                }
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                if (!wp[u]) continue;
                                const int e = e0 + u * Plan::EpiThreads, r = e / q4, c4 = e % q4;
                                op.sgd4(wv[u], mv[u], *s4(r, c4));
                                *reinterpret_cast<float4*>(wp[u]) = wv[u];
                                *reinterpret_cast<float4*>(wp[u] + op.m_off) = mv[u];
                            }
                        }
                    } else {
                        for (int e = et; e < kBM * q4; e += Plan::EpiThreads) {
                            const int r = e / q4, c4 = e % q4, m = mt0 + r;
                            if (m < M && 4 * c4 < N) op.store4(m, 4 * c4, *s4(r, c4));
                        }
                    }
                } else if constexpr (PoolOp<Op>::value) {
                    // conv3 forward: bias + ReLU, then per-sample channel sums and the value > 0
                    // bitmap (no activation store).  Thread = column quad c4 = lane, rows warp + 8 i:
                    // a warp holds one whole row per step (ballots give its bitmap words) and each
                    // thread sums its 8 rows of each sample; the 8 row classes are added in a fixed
                    // order through shared memory.
                    static_assert(Plan::N == 128 && Plan::EpiThreads == 256, "pooling epilogue mapping");
                    const int c4 = et & 31, w8 = et >> 5;
                    float4 ps[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
#pragma unroll
                    for (int ii = 0; ii < 16; ++ii) {
                        const int r = w8 + 8 * ii, m = mt0 + r;
                        if (m >= M) break;  // rows >= M only in the last tile, past its last sample
                        float4 x = *s4(r, c4);
                        x.x = __fadd_rn(x.x, bfix.x); x.y = __fadd_rn(x.y, bfix.y);
                        x.z = __fadd_rn(x.z, bfix.z); x.w = __fadd_rn(x.w, bfix.w);
                        x = make_float4(x.x > 0.0f ? x.x : 0.0f, x.y > 0.0f ? x.y : 0.0f, x.z > 0.0f ? x.z : 0.0f,
                                        x.w > 0.0f ? x.w : 0.0f);
                        float4& pp = ps[ii >> 3];
                        pp.x = __fadd_rn(pp.x, x.x); pp.y = __fadd_rn(pp.y, x.y);
                        pp.z = __fadd_rn(pp.z, x.z); pp.w = __fadd_rn(pp.w, x.w);
                        // bitmap word q (channels 32 q .. 32 q + 31) = the nibbles of lanes 8 q .. 8 q + 7
                        uint32_t v = ((x.x > 0.0f ? 1u : 0u) | (x.y > 0.0f ? 2u : 0u) | (x.z > 0.0f ? 4u : 0u) |
                                      (x.w > 0.0f ? 8u : 0u)) << (4 * (c4 & 7));
                        v |= __shfl_xor_sync(0xffffffffu, v, 1);
                        v |= __shfl_xor_sync(0xffffffffu, v, 2);
                        v |= __shfl_xor_sync(0xffffffffu, v, 4);
                        if ((c4 & 7) == 0) op.mk_out[(long long)m * 4 + (c4 >> 3)] = v;
                    }
                    asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");  // sacc reads done
                    float4* part = reinterpret_cast<float4*>(sacc);  // [row class w8][sample][c4]
                    part[(w8 * 2 + 0) * 32 + c4] = ps[0];
                    part[(w8 * 2 + 1) * 32 + c4] = ps[1];
                    asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");
                    {  // thread = (sample, channel): row classes 0..7 in order, x 2^-6
                        const int smp = et >> 7, ch = et & 127;
                        if (mt0 + 64 * smp < M) {
                            float sum = 0.0f;
#pragma unroll
                            for (int w = 0; w < 8; ++w)
                                sum = __fadd_rn(sum, reinterpret_cast<const float*>(&part[(w * 2 + smp) * 32 + (ch >> 2)])[ch & 3]);
                            op.gout[(long long)((mt0 + 64 * smp) / 64) * 128 + ch] = __fmul_rn(sum, 0.015625f);
                        }
                    }
                } else
                for (int e = et; e < kBM * q4; e += Plan::EpiThreads) {
                    const int r = e / q4, c4 = e % q4, m = mt0 + r;
                    if (m >= M) continue;
                    if (4 * c4 >= N) continue;
                    float4 x = *s4(r, c4);
                    if constexpr (Op::EPI != ctc::kEpiStore) {
                        const float4 b = fixed_c4 ? bfix : op.bias4(4 * c4);
                        x.x = __fadd_rn(x.x, b.x); x.y = __fadd_rn(x.y, b.y);
                        x.z = __fadd_rn(x.z, b.z); x.w = __fadd_rn(x.w, b.w);
                    }
                    if constexpr (Op::EPI == ctc::kEpiBiasRelu)
                        x = make_float4(x.x > 0.0f ? x.x : 0.0f, x.y > 0.0f ? x.y : 0.0f, x.z > 0.0f ? x.z : 0.0f,
                                        x.w > 0.0f ? x.w : 0.0f);
                    op.store4(m, 4 * c4, x);
                }
                asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");  // sacc free for the next tile
                SMX_TL(3072 + i * 2 + 1, et == 0);
            } else if constexpr (Op::EPI == ctc::kEpiPartT) {
                // transposed outputs: lanes = consecutive rows of one column (coalesced)
                const int m = mt0 + row;
                if (m < M)  // each warp writes the columns it drained (no barrier needed)
                    for (int col = cbeg; col < min(N, cbeg + cw); ++col)
                        *op.ct_at(col, m) = sacc[row * PN + (((col >> 2) ^ (row & 7)) << 2) + (col & 3)];
            } else {
                // ReLU-masked scatter to the 4 sub-pixels, cooperative: thread = fixed float4 column
                // (class, 4 channels), rows r0, r0 + 4, ...; a warp covers one row's N columns =
                // whole 128-byte pixel segments.  Mask loads are issued 8 rows ahead of their use.
                constexpr int Q4 = Plan::N / 4, RSTEP = Plan::EpiThreads / Q4, PER = kBM / RSTEP, U = 8;
                static_assert(Plan::EpiThreads % Q4 == 0 && PER % U == 0, "epilogue mapping");
                uint32_t* sbits = reinterpret_cast<uint32_t*>(smem + Plan::MbitsOff);
                if constexpr (Plan::MaskWords > 0) {
#pragma unroll
                    for (int j = 0; j < kMW; ++j) sbits[et + j * Plan::EpiThreads] = mword[j];
                }
                asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");  // the whole tile is in sacc
                const int c4 = et % Q4, r0 = et / Q4;
                if constexpr (Plan::MaskWords > 0) {
                    // bits of the thread's 4 channels: word (row, column / 32), bit column % 32
                    constexpr int WPR = Plan::N / 32;
                    const int wc = (4 * c4) >> 5, sh = (4 * c4) & 31;
#pragma unroll 4
                    for (int ii = 0; ii < PER; ++ii) {
                        const int r = r0 + RSTEP * ii, m = mt0 + r;
                        if (m >= M || 4 * c4 >= N) continue;
                        const uint32_t b = sbits[r * WPR + wc] >> sh;
                        const float4 x = *s4(r, c4);
                        op.store_masked(m, 4 * c4, op.mask_off(m, 4 * c4),
                                        make_float4((b & 1u) ? x.x : 0.0f, (b & 2u) ? x.y : 0.0f, (b & 4u) ? x.z : 0.0f,
                                                    (b & 8u) ? x.w : 0.0f));
                    }
                } else
                for (int i0 = 0; i0 < PER; i0 += U) {
                    float4 mk[U];
                    long long off[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int m = mt0 + r0 + RSTEP * (i0 + u);
                        off[u] = (m < M && 4 * c4 < N) ? op.mask_off(m, 4 * c4) : -1;
                        mk[u] = off[u] >= 0 ? op.mask4(off[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (off[u] < 0) continue;
                        const float4 x = *s4(r0 + RSTEP * (i0 + u), c4);
                        op.store_masked(mt0 + r0 + RSTEP * (i0 + u), 4 * c4, off[u],
                            make_float4(mk[u].x > 0.0f ? x.x : 0.0f, mk[u].y > 0.0f ? x.y : 0.0f,
                                        mk[u].z > 0.0f ? x.z : 0.0f, mk[u].w > 0.0f ? x.w : 0.0f));
                    }
                }
                asm volatile("bar.sync 2, %0;" ::"n"(Plan::EpiThreads) : "memory");  // sacc free for the next tile
                SMX_TL(3072 + i * 2 + 1, et == 0);
            }
#endif
            }  // !TmaOut
        }
        if constexpr (TmaOut<Op>::value)
            if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the last tile's store
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
#ifdef SMX_DBG_TIMELINE
    if (tl_on && threadIdx.x == 0) smx_tl[4094] = clock64();
#endif
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kWsTmemCols));
}

}  // namespace ws
}  // namespace cnn
}  // namespace smx
