// conv1 on the tensor cores (tensor-core mode).  conv1 (3x3, 3 -> 32, stride 1) has K = 27 and
// N = 32, far too thin for a 128-row tile in its natural im2col form; both kernels here reshape it.
//
// ---------------------------------------------------------------------------------------------
// Weight gradient (round 1 ran it on a packed-FFMA2 CUDA-core kernel, FMA-pipe bound at ~57 %):
//
//   dW1[co][kh][kw][ci] = sum_{n, h, w} dA1[n][h][w][co] * X[n][h + kh - 1][w + kw - 1][ci]
//
// A K chunk is 4 consecutive image rows h0 .. h0 + 3 of one sample (128 pixels); within it the
// reduction index is the column w (32 per row).  The four rows sit in the four TMEM lane quadrants
// of A and in four diagonal blocks of B:
//   A[(b, co)][w]            = dA1[n][h0 + b][w][co]                    M = 4 rows x 32 co = 128
//   B[(b, kh, kw, ci)][w]    = X[n][h0 + b + kh - 1][w + kw - 1][ci]     N = 4 blocks x 48 = 192
//                              (per block 36 taps x channels incl. the zero channel, the all-ones
//                              bias row 36, rows 37-47 zero: blocks start at 16-column multiples)
//   D[(b, co)][(b, ...)]     = row h0 + b's contribution to dW1[co][...]  (only the diagonal
//                              blocks are read: 1/4 of the MMA's columns, but every A element is
//                              read once per k-step by an N = 160 MMA instead of three times by
//                              N = 16 MMAs -- an A-from-TMEM MMA costs ~25 + 0.3 N cycles)
// Roles (384 threads, one CTA per SM, all 512 TMEM columns):
//   warp 6      TMA: per chunk the 4 dA1 rows (16 KB, contiguous) + the input rows h0 - 1 .. h0 + 4
//               (clipped to the image) into a 4-entry ring
//   warps 0-3   A builders (warp b = TMEM lane quadrant, lane = co): dA1 row h0 + b, hi = the value
//               (the MMA truncates to tf32) and lo = a - trunc(a), tcgen05.st into a 2-slot ring
//   warps 4-5   B builders (lane = w): blocks 2 (warp - 4) and 2 (warp - 4) + 1, the shifted input
//               rows into a K-major SWIZZLE_NONE tile (LBO 3088 B: conflict-free stores); lo
//               tiles too when the data is not tf32-exact
//   warp 7      MMA: 4 k-steps x (A_lo B_hi [, A_hi B_lo], A_hi B_hi) per chunk, N = 192
//   warps 8-11  epilogue (quadrant b): drain the block's 37 columns every kSeg chunks (128 products
//               per TMEM segment, §3b.5), fp32 round-to-nearest sums in registers; at the end of a
//               work item (kImgs samples of one slot) the four blocks are added in order b = 0..3
//               into the item's partial row part[item][co * 28 + (kh * 3 + kw) * 3 + ci] (+ 27: bias)
//               that conv1_wgrad_reduce sums.
// Work items (slot, group of kImgs samples) are walked by a persistent grid; every role walks the
// same sequence, so ring / slot / segment counters run on across items.
#pragma once

#include "conv_ws.cuh"

namespace smx {
namespace cnn {
namespace c1 {

using namespace smx::tc3;
using ws::lo_of;
using ws::mbar_arrive;
using ws::mma_commit_e;
using ws::tmem_ld16;
using ws::tmem_st16;

constexpr int kImgs = 4;                       // samples per work item (= per partial row)
constexpr int kRing = 4;                       // chunk ring entries
constexpr int kDBytes = 4 * 32 * 32 * 4;       // 4 dA1 rows: 16 KB
constexpr int kXRows = 6;                      // input rows h0 - 1 .. h0 + 4
constexpr int kEntry = kDBytes + kXRows * 512;  // 19456
constexpr int kASlots = 2, kBSlots = 2;
constexpr int kN = 192, kBlk = 48;            // blocks start at 16-column multiples
constexpr int kLbo = 3088, kSbo = 128;         // B tile: (r, k) at (k/4)*3088 + (r/8)*128 + (r%8)*16 + (k%4)*4
constexpr int kBTile = 8 * kLbo;               // 24704 (192 rows x 32 k)
constexpr int kBOff = kRing * kEntry;          // 77824
constexpr int kRedOff = kBOff + kBSlots * 2 * kBTile;  // 176640: item-end block sums [4][32][48]
constexpr int kBarOff = kRedOff + 4 * 32 * kBlk * 4;   // 201216
constexpr int kSmem = kBarOff + 256;
constexpr int kAccCol = kASlots * 64;          // TMEM: [0, 128) A slots (hi +0, lo +32), [128, 512) two accumulators
constexpr int kTmemCols = 512;
constexpr int kTmaWarp = 6, kMmaWarp = 7, kEpiWarp0 = 8;
constexpr int kThreads = 12 * 32;
constexpr int kSeg = SMX_SEG_CHUNKS;
static_assert(kAccCol + 2 * kN <= kTmemCols, "TMEM plan");
static_assert(kSmem <= 227 * 1024, "shared-memory plan");

struct Item {
    int slot, part, n0, n1;  // samples [n0, n1) of slot
};
__device__ __forceinline__ bool item_at(const ConvArgs& p, int j, int parts, Item& it) {
    const int z = j / parts;
    it.part = j % parts;
    it.slot = p.slots[z];
    const int bs = conv_bs(p, it.slot);
    it.n0 = it.part * kImgs;
    it.n1 = min(bs, it.n0 + kImgs);
    return it.n0 < it.n1;
}

__device__ __forceinline__ int boff(int r, int k) { return ((k >> 2) * kLbo + (r >> 3) * kSbo + (r & 7) * 16) / 4 + (k & 3); }

template <bool XEXACT>
__global__ void __launch_bounds__(kThreads, 1) conv1_wgrad_tc_kernel(ConvArgs p, int parts, int nitems) {
    extern __shared__ __align__(1024) char smem[];
    uint64_t* rfull = reinterpret_cast<uint64_t*>(smem + kBarOff);  // ring entry landed (tx)
    uint64_t* rempty = rfull + kRing;                               // entry read by the 6 builder warps
    uint64_t* afull = rempty + kRing;                               // A slot written (128 threads)
    uint64_t* aempty = afull + kASlots;                             // A slot's MMAs done
    uint64_t* bfull = aempty + kASlots;                             // B tile written (2 warps)
    uint64_t* bempty = bfull + kBSlots;                             // B tile's MMAs done
    uint64_t* accf = bempty + kBSlots;                              // accumulator segment done
    uint64_t* acce = accf + 2;                                      // accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 4 || warp == 5) {  // constant B rows: the zero channel, the ones rows, rows 37-39
        for (int t = 0; t < 2 * kBSlots; ++t) {
            float* bt = reinterpret_cast<float*>(smem + kBOff + t * kBTile);
            for (int b = 2 * (warp - 4); b < 2 * (warp - 4) + 2; ++b)
                for (int i = 0; i < kBlk; ++i) {
                    if (i < 36 && (i & 3) != 3) continue;
                    bt[boff(b * kBlk + i, lane)] = (i == 36 && t % 2 == 0) ? 1.0f : 0.0f;  // lo tiles: 0
                }
        }
        asm volatile("fence.proxy.async.shared::cta;");
    }
    if (threadIdx.x == 0) {
        for (int e = 0; e < kRing; ++e) {
            mbar_init(&rfull[e], 1);
            mbar_init(&rempty[e], 6);
        }
        for (int a = 0; a < kASlots; ++a) {
            mbar_init(&afull[a], 128);
            mbar_init(&aempty[a], 1);
        }
        for (int b = 0; b < kBSlots; ++b) {
            mbar_init(&bfull[b], 2);
            mbar_init(&bempty[b], 1);
        }
        for (int u = 0; u < 2; ++u) {
            mbar_init(&accf[u], 1);
            mbar_init(&acce[u], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    Item it;

    if (warp < 4) {
        // ================= A builders: warp b = row h0 + b, lane co =================
        const int b = warp;
        const uint32_t tq = tmem + ((uint32_t)(b * 32) << 16);
        int g = 0;  // chunks of this CTA
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, parts, it)) continue;
            for (int c = 0; c < (it.n1 - it.n0) * 8; ++c, ++g) {
                const int a = g % kASlots, e = g % kRing;
                if (g >= kASlots) mbar_wait(&aempty[a], ((g / kASlots) - 1) & 1);
                mbar_wait(&rfull[e], (g / kRing) & 1);
                const float* src = reinterpret_cast<const float*>(smem + e * kEntry) + b * 1024 + lane;
                float x[32];
#pragma unroll
                for (int w = 0; w < 32; ++w) x[w] = src[w * 32];
                const uint32_t ta = tq + a * 64;
                tmem_st16(ta, x);
                tmem_st16(ta + 16, x + 16);
                float lo[32];
#pragma unroll
                for (int w = 0; w < 32; ++w) lo[w] = lo_of(x[w]);
                tmem_st16(ta + 32, lo);
                tmem_st16(ta + 48, lo + 16);
                asm volatile("tcgen05.wait::st.sync.aligned;");
                asm volatile("tcgen05.fence::before_thread_sync;");
                mbar_arrive(&afull[a]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&rempty[e]);
            }
        }
    } else if (warp < 6) {
        // ================= B builders: lane w, blocks 2 (warp - 4) .. + 1 =================
        const int b0 = 2 * (warp - 4);
        int g = 0;
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, parts, it)) continue;
            for (int c = 0; c < (it.n1 - it.n0) * 8; ++c, ++g) {
                const int s = g % kBSlots, e = g % kRing, h0 = (c & 7) * 4;
                mbar_wait(&rfull[e], (g / kRing) & 1);
                if (g >= kBSlots) mbar_wait(&bempty[s], ((g / kBSlots) - 1) & 1);
                const float4* xr = reinterpret_cast<const float4*>(smem + e * kEntry + kDBytes);
                float* hi = reinterpret_cast<float*>(smem + kBOff + (2 * s) * kBTile);
                // input rows h0 + b0 - 1 .. h0 + b0 + 2 feed blocks b0, b0 + 1 (entry row = ih - h0 + 1)
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int ih = h0 + b0 - 1 + rr;
                    float4 xc = make_float4(0.f, 0.f, 0.f, 0.f);
                    if ((unsigned)ih < 32u) xc = xr[(ih - h0 + 1) * 32 + lane];
                    float4 xl, xq;
                    xl.x = __shfl_up_sync(0xffffffffu, xc.x, 1);
                    xl.y = __shfl_up_sync(0xffffffffu, xc.y, 1);
                    xl.z = __shfl_up_sync(0xffffffffu, xc.z, 1);
                    xq.x = __shfl_down_sync(0xffffffffu, xc.x, 1);
                    xq.y = __shfl_down_sync(0xffffffffu, xc.y, 1);
                    xq.z = __shfl_down_sync(0xffffffffu, xc.z, 1);
                    if (lane == 0) xl = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (lane == 31) xq = make_float4(0.f, 0.f, 0.f, 0.f);
                    const float v[9] = {xl.x, xl.y, xl.z, xc.x, xc.y, xc.z, xq.x, xq.y, xq.z};  // (kw, ci)
#pragma unroll
                    for (int bb = 0; bb < 2; ++bb) {
                        const int kh = rr - bb;  // block b0 + bb reads input row h0 + b0 + bb + kh - 1
                        if (kh < 0 || kh > 2) continue;
#pragma unroll
                        for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                            for (int ci = 0; ci < 3; ++ci) {
                                const int r = (b0 + bb) * kBlk + (kh * 3 + kw) * 4 + ci;
                                hi[boff(r, lane)] = v[kw * 3 + ci];
                                if constexpr (!XEXACT) hi[kBTile / 4 + boff(r, lane)] = lo_of(v[kw * 3 + ci]);
                            }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;");  // generic stores -> the MMA's async proxy
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&bfull[s]);
                    mbar_arrive(&rempty[e]);
                }
            }
        }
    } else if (warp == kTmaWarp) {
        // ================= TMA: 4 dA1 rows + the input rows per chunk =================
        if (lane == 0) {
            int g = 0;
            for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
                if (!item_at(p, j, parts, it)) continue;
                const SlotView v = slot_view(p, it.slot);
                const float* dy = layer_dout<1>(p, v);
                const float* x = layer_in<1>(p, v);
                for (int c = 0; c < (it.n1 - it.n0) * 8; ++c, ++g) {
                    const int e = g % kRing, n = it.n0 + (c >> 3), h0 = (c & 7) * 4;
                    if (g >= kRing) mbar_wait(&rempty[e], ((g / kRing) - 1) & 1);
                    const int r0 = max(0, h0 - 1), r1 = min(32, h0 + 5);
                    ws::mbar_arrive_expect_tx(&rfull[e], kDBytes + (r1 - r0) * 512);
                    ws::bulk_g2s(smem + e * kEntry, dy + ((long long)n * 1024 + h0 * 32) * 32, kDBytes, &rfull[e]);
                    ws::bulk_g2s(smem + e * kEntry + kDBytes + (r0 - h0 + 1) * 512, x + (long long)n * kSample + r0 * 128,
                                 (r1 - r0) * 512, &rfull[e]);
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer =================
        const uint32_t idesc = idesc_tf32(kN);
        int g = 0, sg = 0;
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, parts, it)) continue;
            const int nch = (it.n1 - it.n0) * 8;
            for (int c = 0; c < nch; ++c, ++g) {
                const int a = g % kASlots, s = g % kBSlots, buf = sg & 1;
                const bool seg_start = c % kSeg == 0, seg_end = c % kSeg == kSeg - 1 || c == nch - 1;
                if (seg_start && sg >= 2) mbar_wait(&acce[buf], ((sg >> 1) - 1) & 1);
                mbar_wait(&afull[a], (g / kASlots) & 1);
                mbar_wait(&bfull[s], (g / kBSlots) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + kAccCol + buf * kN, ah = tmem + a * 64, al = ah + 32;
                const uint32_t bh = smem_u32(smem + kBOff + (2 * s) * kBTile), bl = bh + kBTile;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t dh = smem_desc(bh + 2 * k * kLbo, kLbo, kSbo);
                    const uint32_t acc = (seg_start && k == 0) ? 0u : 1u;
                    ws::mma_ts_e(d, al + 8 * k, dh, idesc, acc);
                    if constexpr (!XEXACT) ws::mma_ts_e(d, ah + 8 * k, smem_desc(bl + 2 * k * kLbo, kLbo, kSbo), idesc, 1u);
                    ws::mma_ts_e(d, ah + 8 * k, dh, idesc, 1u);
                }
                mma_commit_e(&aempty[a]);
                mma_commit_e(&bempty[s]);
                if (seg_end) {
                    mma_commit_e(&accf[buf]);
                    ++sg;
                }
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: warp 8 + b, lane co =================
        const int b = warp - kEpiWarp0;
        const uint32_t tq = tmem + ((uint32_t)(b * 32) << 16) + kAccCol + b * kBlk;
        float* red = reinterpret_cast<float*>(smem + kRedOff);
        const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..127
        int sg = 0;
        for (int j = blockIdx.x; j < nitems; j += gridDim.x) {
            if (!item_at(p, j, parts, it)) continue;
            const int nseg = ((it.n1 - it.n0) * 8 + kSeg - 1) / kSeg;
            float sum[37];
            for (int s = 0; s < nseg; ++s, ++sg) {
                const int buf = sg & 1;
                mbar_wait(&accf[buf], (sg >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                uint32_t r[kBlk];
                tmem_ld16(tq + buf * kN, r);
                tmem_ld16(tq + buf * kN + 16, r + 16);
                ws::tmem_ld16(tq + buf * kN + 32, r + 32);
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                asm volatile("tcgen05.fence::before_thread_sync;");
                mbar_arrive(&acce[buf]);
#pragma unroll
                for (int q = 0; q < 37; ++q)
                    sum[q] = s == 0 ? __uint_as_float(r[q]) : __fadd_rn(sum[q], __uint_as_float(r[q]));
            }
            // the four row blocks' sums, added in order b = 0..3
            asm volatile("bar.sync 1, 128;" ::: "memory");  // the previous item's reads of red are done
#pragma unroll
            for (int q = 0; q < 37; ++q) red[(b * 32 + lane) * kBlk + q] = sum[q];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const SlotView v = slot_view(p, it.slot);
            float* part = v.act + p.al.w1p + (long long)it.part * kL1Outs;
            for (int i = et; i < kL1Outs; i += 128) {
                const int co = i / 28, jj = i % 28;
                const int q = jj < 27 ? (jj / 3) * 4 + jj % 3 : 36;
                float t = red[co * kBlk + q];
#pragma unroll
                for (int bb = 1; bb < 4; ++bb) t = __fadd_rn(t, red[(bb * 32 + co) * kBlk + q]);
                part[i] = t;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------------------------------------
// conv1 forward on the tensor cores (tensor-core mode; round 1 used a packed-FFMA2 kernel,
// FMA-pipe bound at ~66 %).  An HBM-bound implicit GEMM: a 128-pixel tile (4 image rows of 32) =
// M, N = 32 output channels, K = 9 taps x 4 channels (the fourth is the zero pad) + 4 zeros = 40,
// 5 k-steps; the weight operand is the pre-split hi / lo image of weight_image_kernel<1> (K-major
// canonical, 2 chunks of 32 k), bulk-copied into shared memory once per slot run.
//
//   warp 8      TMA: per tile the 6 input rows h0 - 1 .. h0 + 4 (512 B each, clipped to the image)
//               into a 4-entry ring; per slot run the 16 KB weight image into one of two buffers
//   warps 0-3   A builders (warp q = TMEM lane quadrant = tile row q, lane = column w): the pixel's
//               3 x 3 x 4 neighbourhood (nine 16-byte loads, zero outside the image) -> 40 TMEM
//               columns (+ 40 lo columns when the data is not tf32-exact)
//   warp 9      MMA: 5 k-steps x (A_hi W_hi, A_hi W_lo [, A_lo W_hi]) into one of two accumulators
//   warps 4-7   epilogue (quadrant q): + bias, ReLU, the pixel's 32 channels (128 B) into a
//               per-warp 128-byte-swizzled staging tile (conflict-free), one 4 KB TMA tensor store
//               per warp and tile row (kTmA1), and the pixel's a1 > 0 bitmap word (mk1)
// Items (slot, sample) are split into contiguous per-CTA ranges (a CTA stays on one slot, so the
// weight image is reloaded only when the slot changes).
namespace f1 {

constexpr int kXRing = 4, kXEntry = 6 * 512;       // 6 input rows x 32 pixels x 4 channels
constexpr int kWImg = 2 * 2 * 32 * 32 * 4;         // 2 K chunks x (hi, lo) x 32 rows x 32 k = 16 KB
constexpr int kWOff = kXRing * kXEntry;            // 12288
constexpr int kStOff = kWOff + 2 * kWImg;          // 45056: staging, 4 warps x 2 x 4 KB
constexpr int kBarOff = kStOff + 4 * 2 * 4096;     // 77824
constexpr int kSmem = kBarOff + 256;
constexpr int kACols = 80;                         // A slot: hi [0, 40), lo [40, 80)
constexpr int kAccCol = 2 * kACols;                // two accumulators of 32 columns at 160, 192
constexpr int kTmemCols = 256;
constexpr int kTmaWarp = 8, kMmaWarp = 9, kEpiWarp0 = 4;
constexpr int kThreads = 10 * 32;

// contiguous item range of this CTA
__device__ __forceinline__ void item_range(int nitems, int& j0, int& j1) {
    const int per = (nitems + gridDim.x - 1) / gridDim.x;
    j0 = min(nitems, (int)blockIdx.x * per);
    j1 = min(nitems, j0 + per);
}
// item j = (slot z, sample n); false if n >= the slot's batch size
__device__ __forceinline__ bool f1_item(const ConvArgs& p, int j, int mb, int& slot, int& n) {
    slot = p.slots[j / mb];
    n = j % mb;
    return n < conv_bs(p, slot);
}

template <bool XEXACT>
__global__ void __launch_bounds__(kThreads, 2) conv1_fwd_tc_kernel(ConvArgs p, int mb, int nitems) {
    extern __shared__ __align__(1024) char smem[];
    uint64_t* xfull = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint64_t* xempty = xfull + kXRing;
    uint64_t* wfull = xempty + kXRing;
    uint64_t* wempty = wfull + 2;
    uint64_t* afull = wempty + 2;
    uint64_t* aempty = afull + 2;
    uint64_t* accf = aempty + 2;
    uint64_t* acce = accf + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int e = 0; e < kXRing; ++e) {
            mbar_init(&xfull[e], 1);
            mbar_init(&xempty[e], 4);
        }
        for (int u = 0; u < 2; ++u) {
            mbar_init(&wfull[u], 1);
            mbar_init(&wempty[u], 1);
            mbar_init(&afull[u], 128);
            mbar_init(&aempty[u], 1);
            mbar_init(&accf[u], 1);
            mbar_init(&acce[u], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    int j0, j1;
    item_range(nitems, j0, j1);
    int slot, n;

    if (warp < 4) {
        // ================= A builders: warp q = tile row, lane w =================
        const int q = warp;
        const uint32_t ta0 = tmem + ((uint32_t)(q * 32) << 16);
        int t = 0;
        for (int j = j0; j < j1; ++j) {
            if (!f1_item(p, j, mb, slot, n)) continue;
            for (int tr = 0; tr < 8; ++tr, ++t) {
                const int e = t % kXRing, a = t & 1, h0 = tr * 4;
                mbar_wait(&xfull[e], (t / kXRing) & 1);
                if (t >= 2) mbar_wait(&aempty[a], ((t >> 1) - 1) & 1);
                const float4* ent = reinterpret_cast<const float4*>(smem + e * kXEntry);
                float v[40];
#pragma unroll
                for (int kh = 0; kh < 3; ++kh) {
                    const int ih = h0 + q + kh - 1;  // entry row ih - (h0 - 1)
#pragma unroll
                    for (int kw = 0; kw < 3; ++kw) {
                        const int iw = lane + kw - 1;
                        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                        if ((unsigned)ih < 32u && (unsigned)iw < 32u) x = ent[(q + kh) * 32 + iw];
                        const int k = (kh * 3 + kw) * 4;
                        v[k] = x.x; v[k + 1] = x.y; v[k + 2] = x.z; v[k + 3] = x.w;
                    }
                }
#pragma unroll
                for (int k = 36; k < 40; ++k) v[k] = 0.0f;
                const uint32_t ta = ta0 + a * kACols;
#ifndef F1_DBG_NO_AST
                tmem_st16(ta, v);
                tmem_st16(ta + 16, v + 16);
                tmem_st8(ta + 32, v + 32);
#else
                if (v[0] == 12345.0f && v[39] == 1.0f) tmem_st16(ta, v);
#endif
                if constexpr (!XEXACT) {
                    float lo[40];
#pragma unroll
                    for (int k = 0; k < 40; ++k) lo[k] = lo_of(v[k]);
                    tmem_st16(ta + 40, lo);
                    tmem_st16(ta + 56, lo + 16);
                    tmem_st8(ta + 72, lo + 32);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;");
                asm volatile("tcgen05.fence::before_thread_sync;");
                mbar_arrive(&afull[a]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&xempty[e]);
            }
        }
    } else if (warp == kTmaWarp) {
        // ================= TMA: weight image per slot run, input rows per tile =================
        if (lane == 0) {
            int t = 0, u = -1, cur = -1;
            for (int j = j0; j < j1; ++j) {
                if (!f1_item(p, j, mb, slot, n)) continue;
                const SlotView v = slot_view(p, slot);
                if (slot != cur) {
                    cur = slot;
                    ++u;
                    const int b = u & 1;
                    if (u >= 2) mbar_wait(&wempty[b], ((u >> 1) - 1) & 1);
                    ws::mbar_arrive_expect_tx(&wfull[b], kWImg);
                    ws::bulk_g2s(smem + kWOff + b * kWImg, v.act + p.al.wf1, kWImg, &wfull[b]);
                }
                const float* img = layer_in<1>(p, v) + (long long)n * kSample;
                for (int tr = 0; tr < 8; ++tr, ++t) {
                    const int e = t % kXRing, h0 = tr * 4;
                    if (t >= kXRing) mbar_wait(&xempty[e], ((t / kXRing) - 1) & 1);
                    const int r0 = max(0, h0 - 1), r1 = min(32, h0 + 5);
                    ws::mbar_arrive_expect_tx(&xfull[e], (r1 - r0) * 512);
                    ws::bulk_g2s(smem + e * kXEntry + (r0 - (h0 - 1)) * 512, img + r0 * 128, (r1 - r0) * 512, &xfull[e]);
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer =================
        const uint32_t idesc = idesc_tf32(32);
        int t = 0, u = -1, cur = -1;
        for (int j = j0; j < j1; ++j) {
            if (!f1_item(p, j, mb, slot, n)) continue;
            if (slot != cur) {
                if (u >= 0) mma_commit_e(&wempty[u & 1]);  // the previous run's tiles are all issued
                cur = slot;
                ++u;
                mbar_wait(&wfull[u & 1], (u >> 1) & 1);
            }
            const uint32_t wb = smem_u32(smem + kWOff + (u & 1) * kWImg);
            for (int tr = 0; tr < 8; ++tr, ++t) {
                const int a = t & 1;
                mbar_wait(&afull[a], (t >> 1) & 1);
                if (t >= 2) mbar_wait(&acce[a], ((t >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + kAccCol + a * 32, ah = tmem + a * kACols;
#ifndef F1_DBG_NO_MMA
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const uint32_t bh = wb + (k >> 2) * 8192 + (k & 3) * 1024;
                    const uint64_t dh = smem_desc(bh, 512, 128), dl = smem_desc(bh + 4096, 512, 128);
                    ws::mma_ts_e(d, ah + 8 * k, dh, idesc, k == 0 ? 0u : 1u);
                    ws::mma_ts_e(d, ah + 8 * k, dl, idesc, 1u);
                    if constexpr (!XEXACT) ws::mma_ts_e(d, ah + 40 + 8 * k, dh, idesc, 1u);
                }
#else
                (void)d; (void)ah; (void)wb; (void)idesc;
#endif
                mma_commit_e(&aempty[a]);
                mma_commit_e(&accf[a]);
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: warp 4 + q, lane w =================
        const int q = warp - kEpiWarp0;
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + kAccCol;
        float* stg = reinterpret_cast<float*>(smem + kStOff + q * 8192);
        int t = 0;
        for (int j = j0; j < j1; ++j) {
            if (!f1_item(p, j, mb, slot, n)) continue;
            const SlotView v = slot_view(p, slot);
            float bias[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) bias[c] = __ldg(v.w + Geo<1>::OffB + c);
            const CUtensorMap* omap = p.tmaps + (long long)slot * kTmapKinds + kTmA1;
            uint32_t* mk1 = reinterpret_cast<uint32_t*>(v.act + p.al.mk1);
            for (int tr = 0; tr < 8; ++tr, ++t) {
                const int a = t & 1;
                mbar_wait(&accf[a], (t >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                uint32_t r[32];
                tmem_ld16(tq + a * 32, r);
                tmem_ld16(tq + a * 32 + 16, r + 16);
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                asm volatile("tcgen05.fence::before_thread_sync;");
                mbar_arrive(&acce[a]);
                // staging row `lane` of buffer a (its bulk store of two tiles ago has read it)
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                // 128-byte swizzle (16-byte chunk c of row p at c ^ (p % 8)): conflict-free stores,
                // and the layout the TMA store un-swizzles
                float4* row = reinterpret_cast<float4*>(stg + a * 1024 + lane * 32);
                uint32_t bits = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int c4 = i;
                    float4 o;
                    o.x = fmaxf(__fadd_rn(__uint_as_float(r[4 * c4 + 0]), bias[4 * c4 + 0]), 0.0f);
                    o.y = fmaxf(__fadd_rn(__uint_as_float(r[4 * c4 + 1]), bias[4 * c4 + 1]), 0.0f);
                    o.z = fmaxf(__fadd_rn(__uint_as_float(r[4 * c4 + 2]), bias[4 * c4 + 2]), 0.0f);
                    o.w = fmaxf(__fadd_rn(__uint_as_float(r[4 * c4 + 3]), bias[4 * c4 + 3]), 0.0f);
                    row[c4 ^ (lane & 7)] = o;
                    bits |= ((o.x > 0.0f ? 1u : 0u) | (o.y > 0.0f ? 2u : 0u) | (o.z > 0.0f ? 4u : 0u) |
                             (o.w > 0.0f ? 8u : 0u)) << (4 * c4);
                }
                // the pixel's a1 > 0 bitmap word (the conv2 input gradient's ReLU mask)
                mk1[(long long)n * 1024 + (tr * 4 + q) * 32 + lane] = bits;
                asm volatile("fence.proxy.async.shared::cta;");
                __syncwarp();
#ifdef F1_DBG_NO_STORE
                if (lane == 0 && omap == nullptr) {
#else
                if (lane == 0) {
#endif
                    const int y = n * 1024 + (tr * 4 + q) * 32;  // first pixel of the tile row
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(omap),
                                 "r"(0), "r"(y), "r"(smem_u32(stg + a * 1024))
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace f1
}  // namespace c1
}  // namespace cnn
}  // namespace smx
