// conv2 weight gradient, all taps per CTA (tensor-core mode; replaces conv_ws_kernel<Wgrad<2>>).
//
//   part[split][co][k] = sum_{m in split} im2col(a1)[m][k] * d2[m][co],   k = (tap, ci) < 288,
//   k = 288: the bias gradient (an all-ones im2col row) -- the partial layout wgrad_reduce<2> sums.
//
// The per-tap kernel (one CTA per 128-row M tile = 4 taps) fetched, per 32 output pixels, a
// 16 KB tap box of a1 for its tile and the 8 KB d2 tile: three CTAs read the same d2 rows and
// overlapping a1 windows (60 KB of L2 -> shared-memory traffic per 32 pixels, 80 KB of shared-
// memory traffic per 12 MMAs), so it ran at ~42 % of its MMA floor, bound by shared-memory
// bandwidth and load latency (profiles/r02/SUMMARY.md).  Here one CTA owns a 2048-pixel range of
// the reduction for ALL three M tiles:
//
//   per K chunk (32 output pixels = 2 output rows of one sample):
//     TMA warp   one 4-D box of the chunk's input window (5 input rows x 33 columns (-1..31) x
//                32 channels, zero fill = the convolution's padding; 21 KB) + the d2 tile (two
//                32 x 32 MN-major 128B/32B-atom swizzled boxes, 8 KB) into the stage
//     producers  (warps 0-3, warp q = TMEM lane quadrant q; tile 2 by warps 12 / 13): for each M tile t the im2col rows of tap 4t + q (lane =
//                input channel) straight from the window (input (2r + kh, 2ow + kw) for pixel
//                (r, ow): one conflict-free LDS per k), split hi / lo, tcgen05.st to a TMEM A slot
//                (5-slot ring; tile 2 quadrant 1 lane 0 = the all-ones bias row)
//     MMA warp   per tile 4 k-steps x 3 kind::tf32 MMAs (3xTF32) into the tile's accumulator
//     epilogue   (warps 4-13, one per lane quadrant holding outputs; warps 4-11 also write B lo =
//                b - trunc(b) next to the TMA'd hi tile): every 4 chunks drain the tile's accumulator and
//                add it into fp32 register sums (round-to-nearest, fixed order: §3b.5), write the
//                tile's partial rows at the end
//   = 29 KB of L2 traffic and ~150 KB of shared-memory traffic per 36 MMAs.
//
// Accumulators are single-buffered (3 x 64 TMEM columns): a tile's drain overlaps the other two
// tiles' MMAs of the next chunk.  TMEM: [0, 192) accumulators, [192, 512) five A slots of 64
// columns (hi at +0, lo at +32).  Arithmetic per output = the per-tap kernel's (same MMA order,
// same segments, same bias row), so results are deterministic and grouping invariant.
#pragma once

#include "conv_ws.cuh"

namespace smx {
namespace cnn {
namespace wg2 {

using namespace smx::tc3;
using ws::lo_of;
using ws::mbar_arrive;
using ws::mma_commit_e;
using ws::mma_ts_e;
using ws::tmem_ld16;
using ws::tmem_st16;

using G = Geo<2>;
constexpr int kStages = 6;
constexpr int kWinRows = 5, kWinCols = 33;                       // input rows 2 oh0 - 1 .. 2 oh0 + 3, cols -1 .. 31
constexpr int kWinBytes = kWinRows * kWinCols * G::Ci * 4;         // 21120
constexpr int kBBytes = 32 * G::Co * 4;                            // 8192 (hi or lo)
constexpr int kStageBytes = (2 * kBBytes + kWinBytes + 1023) / 1024 * 1024;  // 37888
constexpr int kBarOff = kStages * kStageBytes;
constexpr int kSmem = kBarOff + 512;
constexpr int kASlots = 5;
constexpr int kAccCols = 64, kABase = 3 * kAccCols;
// warps: 0-3 producers, 4-7 / 8-11 epilogue of tiles 0 / 1, 12-13 epilogue of tile 2 (only its lane
// quadrants 0 (tap 8) and 1 (the bias row) hold outputs), 14 MMA, 15 TMA: 16 warps = 128 registers
constexpr int kProdWarps = 4, kEpiWarp0 = 4, kMmaWarp = 14, kTmaWarp = 15;
constexpr int kBloThreads = 256;  // the epilogue warps of tiles 0 / 1 also split each chunk's B tile
constexpr int kThreads = 16 * 32;
constexpr int kSeg = SMX_SEG_CHUNKS;
static_assert(kABase + kASlots * 64 == 512, "TMEM plan");
static_assert(kSmem <= 227 * 1024, "shared-memory plan");

// A work item = (slot, 2048-pixel split); the grid is persistent (one CTA per SM) and CTA b takes
// items b, b + gridDim.x, ...  Every role walks the same item sequence; chunk and segment counters
// run on across items, so the pipeline never drains between them.
struct Item {
    int slot, split, kbeg, nchunks;
};
__device__ __forceinline__ bool item_at(const ConvArgs& p, int j, int splits, Item& it) {
    const int z = j / splits;
    it.split = j % splits;
    it.slot = p.slots[z];
    const int total = conv_bs(p, it.slot) * G::OH * G::OH;  // a multiple of 256
    it.kbeg = it.split * kSplitRows;
    it.nchunks = min(kSplitRows, total - it.kbeg) / 32;
    return it.nchunks > 0;
}

// One warp's 32 rows of an A slot: tap < 9 -> the tap's im2col rows (lane = input channel) read
// from the chunk's window, split hi / lo; tap == 9 -> the all-ones bias row (lane 0) and zeros.
__device__ __forceinline__ void build_rows(int tap, uint32_t ta, const float* win, int lane) {
    if (tap < 9) {
        const float* src = win + ((tap / 3) * kWinCols + tap % 3) * G::Ci + lane;
        float x[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
#ifdef WG2_DBG_NO_WIN  // profiling variant: no window reads
            x[k] = __int_as_float(0x3f000000 + lane + k);
#else
            x[k] = src[((k >> 4) * 2 * kWinCols + 2 * (k & 15)) * G::Ci];
#endif
        }
        tmem_st16(ta, x);
        tmem_st16(ta + 16, x + 16);
        float lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) lo[k] = lo_of(x[k]);
        tmem_st16(ta + 32, lo);
        tmem_st16(ta + 48, lo + 16);
    } else {
        float x[16], z[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x[k] = lane == 0 ? 1.0f : 0.0f;
            z[k] = 0.0f;
        }
        tmem_st16(ta, x);
        tmem_st16(ta + 16, x);
        tmem_st16(ta + 32, z);
        tmem_st16(ta + 48, z);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
}

// The 12 MMAs of one (tile, chunk): 4 k-steps x (A_lo B_hi, A_hi B_lo, A_hi B_hi), one elect and
// all operand arithmetic inside one asm block (A: +8 TMEM columns, B: +1 KB = 64 descriptor units
// per k-step), so the issuing warp spends few instructions per MMA.
__device__ __forceinline__ void mma12(uint32_t d, uint32_t ahi, uint64_t bh, uint64_t bl, uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t.reg .b32 al, ah;\n\t.reg .b64 h, l;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "add.u32 al, %1, 32;\n\tmov.b32 ah, %1;\n\tmov.b64 h, %2;\n\tmov.b64 l, %3;\n\t"
#ifndef WG2_DBG_NO_LO
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], h, %4, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], l, %4, t;\n\t"
#else
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], l, %4, p;\n\t"
#endif
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], h, %4, t;\n\t"
        "add.u32 al, al, 8;\n\tadd.u32 ah, ah, 8;\n\tadd.u64 h, h, 64;\n\tadd.u64 l, l, 64;\n\t"
#ifndef WG2_DBG_NO_LO
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], h, %4, t;\n\t"
#endif
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], l, %4, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], h, %4, t;\n\t"
        "add.u32 al, al, 8;\n\tadd.u32 ah, ah, 8;\n\tadd.u64 h, h, 64;\n\tadd.u64 l, l, 64;\n\t"
#ifndef WG2_DBG_NO_LO
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], h, %4, t;\n\t"
#endif
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], l, %4, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], h, %4, t;\n\t"
        "add.u32 al, al, 8;\n\tadd.u32 ah, ah, 8;\n\tadd.u64 h, h, 64;\n\tadd.u64 l, l, 64;\n\t"
#ifndef WG2_DBG_NO_LO
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], h, %4, t;\n\t"
#endif
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], l, %4, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], h, %4, t;\n\t"
        "}\n" ::"r"(d), "r"(ahi), "l"(bh), "l"(bl), "r"(idesc), "r"(acc0));
}

__device__ __forceinline__ void mbar_arrive2(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0], 2;\n\t}" ::"r"(smem_u32(bar)));
}

__global__ void __launch_bounds__(kThreads, 1) wgrad2_at_kernel(ConvArgs p, int splits, int nitems) {
    extern __shared__ __align__(1024) char smem[];
    uint64_t* tfull = reinterpret_cast<uint64_t*>(smem + kBarOff);  // stage landed (TMA tx)
    uint64_t* empty = tfull + kStages;                              // stage's MMAs done
    uint64_t* afull = empty + kStages;                              // A slot written (+ B lo)
    uint64_t* aempty = afull + kASlots;                             // A slot's MMAs done
    uint64_t* accf = aempty + kASlots;                              // tile accumulator segment done
    uint64_t* acce = accf + 3;                                      // tile accumulator drained
    uint64_t* bready = acce + 3;                                    // stage's B lo written
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bready + kStages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&bready[s], kBloThreads);
        }
        for (int a = 0; a < kASlots; ++a) {
            mbar_init(&afull[a], kProdWarps * 32);
            mbar_init(&aempty[a], 1);
        }
        for (int t = 0; t < 3; ++t) {
            mbar_init(&accf[t], 1);
            mbar_init(&acce[t], t == 2 ? 64 : 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    Item it;

    if (warp < kProdWarps) {
        // ================= producers =================
        const int q = warp;
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
        int gg = 0;  // chunks processed by this CTA
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, splits, it)) continue;
            for (int g = 0; g < it.nchunks; ++g, ++gg) {
                const int s = gg % kStages;
                mbar_wait(&tfull[s], (gg / kStages) & 1);
                char* st = smem + s * kStageBytes;
                const float* win = reinterpret_cast<const float*>(st + 2 * kBBytes);
                // tiles 0 / 1 (taps q, 4 + q); tile 2 (tap 8, the bias row) is built by warps 12 / 13
#pragma unroll 1
                for (int t = 0; t < 2; ++t) {
                    const int i = 3 * gg + t, a = i % kASlots;
                    if (i >= kASlots) mbar_wait(&aempty[a], ((i / kASlots) - 1) & 1);
                    build_rows(4 * t + q, tq + kABase + a * 64, win, lane);
                    mbar_arrive(&afull[a]);
                }
            }
        }
    } else if (warp == kTmaWarp) {
        // ================= TMA producer (one elected lane) =================
        if (lane == 0) {
            int gg = 0;
            for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
                if (!item_at(p, j, splits, it)) continue;
                const CUtensorMap* wmap = p.tmaps + (long long)it.slot * kTmapKinds + kTmWg2;
                const CUtensorMap* bmap = p.tmaps + (long long)it.slot * kTmapKinds + kTmWgB2;
                for (int g = 0; g < it.nchunks; ++g, ++gg) {
                    const int s = gg % kStages;
                    if (gg >= kStages) mbar_wait(&empty[s], ((gg / kStages) - 1) & 1);
                    const uint32_t bar = smem_u32(&tfull[s]), dst = smem_u32(smem + s * kStageBytes);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                                 "r"(2 * 4096 + kWinBytes));
                    const int pix = it.kbeg + 32 * g;
                    const int n = pix / (G::OH * G::OH), oh0 = (pix % (G::OH * G::OH)) / G::OH;
                    for (int b = 0; b < 2; ++b)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + b * 4096),
                            "l"(bmap), "r"(32 * b), "r"(pix), "r"(bar)
                            : "memory");
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst + 2 * kBBytes),
                        "l"(wmap), "r"(0), "r"(-1), "r"(2 * oh0 - 1), "r"(n), "r"(bar)
                        : "memory");
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer (whole warp, elected lane issues) =================
        const uint32_t idesc = idesc_tf32(G::Co) | (1u << 16);  // B MN-major
        int gg = 0, sg = 0;  // chunks / accumulation segments started by this CTA
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, splits, it)) continue;
            for (int g = 0; g < it.nchunks; ++g, ++gg) {
                const int s = gg % kStages;
                const bool seg_start = g % kSeg == 0, seg_end = g % kSeg == kSeg - 1 || g == it.nchunks - 1;
                const uint32_t bhi = smem_u32(smem + s * kStageBytes), blo = bhi + kBBytes;
                const uint64_t dbh0 = smem_desc_mn32(bhi, 4096, 512), dbl0 = smem_desc_mn32(blo, 4096, 512);
                for (int t = 0; t < 3; ++t) {
                    const int i = 3 * gg + t, a = i % kASlots;
                    if (seg_start && sg > 0) mbar_wait(&acce[t], (sg - 1) & 1);
                    if (t == 0) mbar_wait(&bready[s], (gg / kStages) & 1);
                    mbar_wait(&afull[a], (i / kASlots) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t dacc = tmem + t * kAccCols, ahi = tmem + kABase + a * 64;
                    mma12(dacc, ahi, dbh0, dbl0, idesc, seg_start ? 0u : 1u);
                    mma_commit_e(&aempty[a]);
                    if (seg_end) mma_commit_e(&accf[t]);
                }
                mma_commit_e(&empty[s]);
                if (seg_end) ++sg;
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: one warp per lane quadrant holding outputs =================
        // The warps of tiles 0 / 1 also write each chunk's B lo (= b - trunc(b) at the TMA'd hi
        // tile's swizzled positions), one chunk ahead of the drains, so a drain never holds up
        // the next chunk's MMAs.
        const int t = (warp - kEpiWarp0) >> 2, q = warp & 3;
        const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + t * kAccCols;
        const int m = 128 * t + 32 * q + lane;
        const bool blo_role = t < 2;
        const int bt = threadIdx.x - kEpiWarp0 * 32;
        int total = 0;  // chunks of this CTA
        for (int j = blockIdx.x; j < nitems; j += gridDim.x)
            if (item_at(p, j, splits, it)) total += it.nchunks;
        auto blo_chunk = [&](int c) {
            const int s = c % kStages;
            mbar_wait(&tfull[s], (c / kStages) & 1);
            char* st = smem + s * kStageBytes;
            const float4* hi4 = reinterpret_cast<const float4*>(st);
            float4* lo4 = reinterpret_cast<float4*>(st + kBBytes);
#pragma unroll
            for (int u = bt; u < kBBytes / 16; u += kBloThreads) {
#ifdef WG2_DBG_NO_BLO  // profiling variant: B lo not computed
                break;
#endif
                const float4 b = hi4[u];
                lo4[u] = make_float4(lo_of(b.x), lo_of(b.y), lo_of(b.z), lo_of(b.w));
            }
            asm volatile("fence.proxy.async.shared::cta;");  // B lo -> the MMA's async proxy
            mbar_arrive(&bready[s]);
        };
        if (blo_role && total > 0) blo_chunk(0);
        int gg = 0, sg = 0;
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, splits, it)) continue;
            float sum[64];
            for (int g = 0; g < it.nchunks; ++g, ++gg) {
                if (blo_role && gg + 1 < total) blo_chunk(gg + 1);
                if (t == 2) {  // tile 2's rows: tap 8 (quadrant 0), the bias row (quadrant 1)
                    const int s = gg % kStages, i = 3 * gg + 2, a = i % kASlots;
                    mbar_wait(&tfull[s], (gg / kStages) & 1);
                    if (i >= kASlots) mbar_wait(&aempty[a], ((i / kASlots) - 1) & 1);
                    build_rows(8 + q, tmem + ((uint32_t)(q * 32) << 16) + kABase + a * 64,
                               reinterpret_cast<const float*>(smem + s * kStageBytes + 2 * kBBytes), lane);
                    mbar_arrive2(&afull[a]);  // 64 threads x 2 = the slot's 128 arrivals
                }
                if (g % kSeg != kSeg - 1 && g != it.nchunks - 1) continue;
                const bool first = g < kSeg;
                mbar_wait(&accf[t], sg & 1);
                ++sg;
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t r[32];
                    tmem_ld16(tacc + 32 * h, r);
                    tmem_ld16(tacc + 32 * h + 16, r + 16);
                    asm volatile("tcgen05.wait::ld.sync.aligned;");
                    if (h == 1) {
                        asm volatile("tcgen05.fence::before_thread_sync;");
                        mbar_arrive(&acce[t]);
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        sum[32 * h + c] = first ? __uint_as_float(r[c]) : __fadd_rn(sum[32 * h + c], __uint_as_float(r[c]));
                }
            }
            if (m < Part<2>::Rows) {
                float* out = p.act + p.al.stride * it.slot + p.al.p2 + (long long)it.split * G::Co * Part<2>::Ld + m;
#pragma unroll
                for (int co = 0; co < 64; ++co) out[(long long)co * Part<2>::Ld] = sum[co];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace wg2
}  // namespace cnn
}  // namespace smx
