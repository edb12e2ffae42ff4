// CNN model of the stage executor (SMX_MODEL_CNN, SURVEY §8d "small CNN"):
//   conv3x3 3->32 s1 -> ReLU -> conv3x3 32->64 s2 -> ReLU -> conv3x3 64->128 s2 -> ReLU
//   -> global average pool -> FC 128->10 -> softmax-CE;  PyTorch SGD (K5, shared with the MLP).
//
// Layout (HBM): images NHWC 32x32x4 (channel 3 == 0), activations NHWC per slot, conv weights
// [Cout][kh*3+kw][Cin_pad].  Exact mode runs the SIMT kernels below (one thread per output, the
// fmaf chain order of oracle/cnn.c); tensor-core mode runs conv2/conv3 as implicit GEMMs on
// tcgen05 through the Op policies below and the warp-specialised kernel of conv_ws.cuh: forward
// M = pixels, K = (tap, cin); input gradient as one sub-pixel GEMM; weight gradient with the
// reduction over (sample, pixel) split into fixed 2048-row ranges reduced in order by
// wgrad_reduce_kernel (deterministic, grouping invariant) and the bias gradient as an extra
// all-ones row of the im2col operand.  conv1 (K = 27) uses fp32 SIMT kernels in both modes.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded on the host through the runtime's driver entry point)

#include "common.cuh"
#include "gemm_tc.cuh"
#include "step_kernels.cuh"

// chunks (of 32 products) per TMEM accumulation segment before the fp32 promotion (§3b.5)
#ifndef SMX_SEG_CHUNKS
#define SMX_SEG_CHUNKS 4
#endif
// the input gradients' segments: 4 chunks = 128 products, as every other conv.  8-chunk segments
// (one drain per conv2 tile) measured Dgrad2 562 -> 518 us and Dgrad3 457 -> 419 us at bs 128, but
// their dA1 / dA2 errors reach the conv1 bias gradient -- a bs x 1024-term sum with cancellation --
// at 2.1-3.4e-5 (90th-percentile channel, bs 5) against the 2e-5 bound (the fp32 oracle: 3e-6);
// with 4-chunk segments batch sizes 1 / 5 / 16 / 37 / 64 are all within it
// (tests/test_cnn_gpu.py::test_tc_first_step_gradient).
#ifndef SMX_DGR_SEG_CHUNKS
#define SMX_DGR_SEG_CHUNKS 4
#endif

namespace smx {
namespace cnn {

constexpr int kImg = 32, kChReal = 3, kChPad = 4, kSample = kImg * kImg * kChPad;  // floats per image
constexpr int kNC = 10, kNCP = 16, kFeat = 128;

template <int L>
struct Geo;
template <>
struct Geo<1> {
    static constexpr int H = 32, Ci = 4, Cr = 3, Co = 32, S = 1, OH = 32;
    static constexpr long long OffW = 0, OffB = 1152;
};
template <>
struct Geo<2> {
    static constexpr int H = 32, Ci = 32, Cr = 32, Co = 64, S = 2, OH = 16;
    static constexpr long long OffW = 1184, OffB = 19616;
};
template <>
struct Geo<3> {
    static constexpr int H = 16, Ci = 64, Cr = 64, Co = 128, S = 2, OH = 8;
    static constexpr long long OffW = 19680, OffB = 93408;
};
constexpr long long kOffW4 = 93536, kOffB4 = kOffW4 + kNCP * kFeat, kPEnd = kOffB4 + kNCP;
constexpr long long kPAlloc = (kPEnd + 63) / 64 * 64;  // 95616
constexpr long long kPAlgo = 32LL * 27 + 32 + 64LL * 288 + 64 + 128LL * 576 + 128 + 10LL * 128 + 10;  // 94538
static_assert(Geo<1>::OffB == Geo<1>::OffW + 32 * 9 * 4 && Geo<2>::OffW == Geo<1>::OffB + 32, "layout");
static_assert(Geo<2>::OffB == Geo<2>::OffW + 64 * 9 * 32 && Geo<3>::OffW == Geo<2>::OffB + 64, "layout");
static_assert(Geo<3>::OffB == Geo<3>::OffW + 128 * 9 * 64 && kOffW4 == Geo<3>::OffB + 128, "layout");

// weight-gradient split of the (sample, pixel) reduction: fixed 2048-row ranges
constexpr int kSplitRows = 2048;
template <int L>
struct Part {
    static constexpr int Rows = 9 * Geo<L>::Ci + 1;            // im2col rows + the all-ones (bias) row
    static constexpr int Ld = (Rows + 3) / 4 * 4;               // floats per partial row
    static constexpr int MaxSplit = (256 * Geo<L>::OH * Geo<L>::OH + kSplitRows - 1) / kSplitRows;
    static constexpr long long Size = (long long)MaxSplit * Geo<L>::Co * Ld;
};

// layer-1 weight-gradient outputs: 32 co x 27 (tap, ci) + 32 bias
constexpr int kL1Outs = 32 * 28;

// Per-slot activation scratch: offsets in floats, tensors [max_batch][...] (computed on host).
struct ActLayout {
    long long a1, a2, a3, d1, d2, d3, g, z, dz, dg, rl, p1, p2, p3, wf1, wf2, wf3, wd2, wd3, w1p, stride;
    long long mk1, mk2;  // tensor-core mode: ReLU-mask bitmaps of a1 / a2, bit e = (a[e] > 0)
    long long mk3;       // tensor-core mode: bitmap of a3 > 0 (written by the conv3 forward epilogue, read by head_dg)
};

// Tensor-core B operands that are weights are pre-split once per lockstep into "images": per K
// chunk of 32, the tf32 hi tile then the lo tile, each in the UMMA K-major canonical layout
// ((row r, k) at (k/4)*16*nt + (r/8)*128 + (r%8)*16 + (k%4)*4 bytes), so a stage is one bulk
// async copy of nt*256 bytes.  Forward: rows co, K = (tap, ci); input gradient: rows ci, K per
// parity class = (dense tap, co), classes back to back.
template <int L>
struct WImg {
    static constexpr int FwdChunks = (9 * Geo<L>::Ci + 31) / 32;
    static constexpr int FwdFloats = FwdChunks * Geo<L>::Co * 64;
    // input gradient as a sub-pixel GEMM: N = 4 parity classes x Ci (in tiles of <= 128 rows),
    // K = 2x2 output neighbourhood x Co
    static constexpr int DgrN = 4 * Geo<L>::Ci;
    static constexpr int DgrNTile = DgrN < 128 ? DgrN : 128;
    static constexpr int DgrChunks = 4 * Geo<L>::Co / 32;
    static constexpr int DgrFloats = DgrChunks * DgrN * 64;
    // first chunk of parity class c (taps 1, 2, 2, 4)
    static __host__ __device__ constexpr int class_chunk0(int c) {
        return (c == 0 ? 0 : c == 1 ? 1 : c == 2 ? 3 : 5) * Geo<L>::Co / 32;
    }
};
inline ActLayout act_layout(int max_batch) {
    ActLayout L{};
    long long o = 0;
    auto take = [&](long long per_sample) {
        const long long at = o;
        o += (per_sample * max_batch + 63) / 64 * 64;
        return at;
    };
    L.a1 = take(1024 * 32);
    L.a2 = take(256 * 64);
    L.a3 = take(64 * 128);
    L.d1 = take(1024 * 32);
    L.d2 = take(256 * 64);
    L.d3 = take(64 * 128);
    L.g = take(kFeat);
    L.z = take(kNCP);
    L.dz = take(kNCP);
    L.dg = take(kFeat);
    L.rl = take(1);
    L.w1p = take(kL1Outs);
    L.mk1 = take(1024 * 32 / 32);
    L.mk2 = take(256 * 64 / 32);
    L.mk3 = take(64 * 128 / 32);
    L.p1 = o;
    o += Part<1>::Size;
    L.p2 = o;
    o += Part<2>::Size;
    L.p3 = o;
    o += Part<3>::Size;
    L.wf1 = o;
    o += WImg<1>::FwdFloats;
    L.wf2 = o;
    o += WImg<2>::FwdFloats;
    L.wf3 = o;
    o += WImg<3>::FwdFloats;
    L.wd2 = o;
    o += WImg<2>::DgrFloats;
    L.wd3 = o;
    o += WImg<3>::DgrFloats;
    L.stride = (o + 63) / 64 * 64;
    return L;
}

// TMA tensor maps of the tensor-core convolutions' A operands, per slot (NHWC fp32, dims
// innermost first: channel, column, row, sample = max_batch; 128-byte swizzle; zero fill out of
// bounds): the conv2 / conv3 forward inputs (a1 / a2, loaded with a column and row traversal
// stride of 2), the conv2 / conv3 output gradients (d2 / d3) of the sub-pixel input gradients, and
// the weight gradients' im2col operands (a1 / a2 again, one box of 32 output pixels x all input
// channels per tap).
enum { kTmFwd2 = 0, kTmFwd3 = 1, kTmDgr2 = 2, kTmDgr3 = 3, kTmWg2 = 4, kTmWg3 = 5, kTmWgB2 = 6, kTmWgB3 = 7, kTmA1 = 8, kTmD1 = 9, kTmD2 = 10, kTmapKinds = 11 };
// kTmWgB2 / kTmWgB3: the weight gradients' B operand (the layer's output gradient d2 / d3 as a
// 2-D [sample x pixel][Co] tensor): 32 x 32 boxes with the 128-byte / 32-byte-atom swizzle = the
// UMMA MN-major tf32 layout (SWIZZLE_128B_BASE32B), loaded straight into the B stage.
// kTmA1: a1 as a 2-D [sample x pixel][32] tensor, boxes of one image row (32 pixels x 128 B) with
// the 128-byte swizzle: the conv1 forward's output tiles leave shared memory by TMA stores.

struct ConvArgs {
    const int* slots;
    const SlotState* st;
    const float* hp;
    int hp_cap;
    int n_train_mask;
    const float* x;      // image rows (train or validation set)
    int x_from_slot;     // 1: first row = slot data offset (training); 0: x_row0 (eval chunk)
    int x_row0;
    int fixed_bs;        // > 0: batch size override (eval chunks)
    int fuse_update;     // tensor-core lockstep: the weight-gradient reductions apply K5 in place
    int pooled;          // tensor-core mode: the conv3 forward epilogue wrote g (pooled) and the a3 > 0 bitmap
                         // instead of a3; the head kernels read those
    float* slab;
    long long slab_stride;
    float* act;
    ActLayout al;
    float* grad;
    long long grad_stride;
    const int* labels;   // training labels (slot offset) or validation labels (x_row0)
    const CUtensorMap* tmaps;  // [slot][kTmapKinds]: TMA maps of the implicit-GEMM A operands
    float* loss_hist;
    float* zout;         // eval: logits [group][n_val][16]
    long long z_stride;
};

__device__ __forceinline__ int conv_bs(const ConvArgs& p, int slot) {
    if (p.fixed_bs > 0) return p.fixed_bs;
    return (int)p.hp[((long long)slot * p.hp_cap + p.st[slot].step) * 4 + 3];
}
__device__ __forceinline__ long long conv_row0(const ConvArgs& p, int slot) {
    return p.x_from_slot ? (long long)(p.st[slot].offset & p.n_train_mask) : (long long)p.x_row0;
}

// ---- K8/K10 for images ----------------------------------------------------------------
// x[r][h][w][c] = k/128, k = (hash(seed, stream, r mod n, (h*32+w)*3+c) & 0xFF) - 128; c = 3 -> 0.
__global__ void gen_img_kernel(float* x, long long rows, int n, uint64_t seed, uint64_t stream) {
    const long long total = rows * kSample;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / kSample;
        const int e = (int)(i - r * kSample);
        const int pix = e >> 2, ch = e & 3;
        float v = 0.0f;
        if (ch < kChReal) {
            const uint64_t h = ckey(seed, stream, (uint64_t)(r % n), (uint64_t)(pix * kChReal + ch));
            v = (float)((int)(h & 0xFF) - 128) * 0.0078125f;
        }
        x[i] = v;
    }
}

// label = argmax_c sum_{h,w,ch} k * T[ch*16 + (h/8)*4 + w/8][c] (exact int32), ties -> smallest c.
__global__ void gen_img_labels_kernel(const float* x, int* y, long long rows, uint64_t seed) {
    __shared__ signed char T[kChReal * 16 * kNC];
    for (int i = threadIdx.x; i < kChReal * 16 * kNC; i += blockDim.x) {
        const int b = i / kNC, c = i % kNC;
        T[i] = (signed char)((int)((ckey(seed, 7, (uint64_t)c, (uint64_t)b) >> 8) & 7) - 4);
    }
    __syncthreads();
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
         r += (long long)gridDim.x * blockDim.x) {
        int acc[kNC];
#pragma unroll
        for (int c = 0; c < kNC; ++c) acc[c] = 0;
        const float* xr = x + r * kSample;
        for (int pix = 0; pix < kImg * kImg; ++pix) {
            const int h = pix >> 5, w = pix & 31;
            for (int ch = 0; ch < kChReal; ++ch) {
                const int k = (int)(xr[pix * 4 + ch] * 128.0f);
                const int b = ch * 16 + (h >> 3) * 4 + (w >> 3);
#pragma unroll
                for (int c = 0; c < kNC; ++c) acc[c] += k * (int)T[b * kNC + c];
            }
        }
        int best = 0;
#pragma unroll
        for (int c = 1; c < kNC; ++c)
            if (acc[c] > acc[best]) best = c;
        y[r] = best;
    }
}

// He-uniform init (stream 8), identical for every root; padded entries stay 0.
__global__ void cnn_init_kernel(float* w, float* m, uint64_t seed, float s1, float s2, float s3, float s4) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < kPAlloc;
         i += (long long)gridDim.x * blockDim.x) {
        int layer = 0, o = 0, in = 0;
        float sc = 0.0f;
        if (i < Geo<1>::OffB) {
            const int r = (int)i;
            o = r / 36; const int t = (r % 36) / 4, ci = r % 4;
            if (ci < 3) { layer = 1; in = t * 3 + ci; sc = s1; }
        } else if (i >= Geo<2>::OffW && i < Geo<2>::OffB) {
            const int r = (int)(i - Geo<2>::OffW);
            layer = 2; o = r / 288; in = r % 288; sc = s2;
        } else if (i >= Geo<3>::OffW && i < Geo<3>::OffB) {
            const int r = (int)(i - Geo<3>::OffW);
            layer = 3; o = r / 576; in = r % 576; sc = s3;
        } else if (i >= kOffW4 && i < kOffW4 + (long long)kNC * kFeat) {
            const int r = (int)(i - kOffW4);
            layer = 4; o = r / kFeat; in = r % kFeat; sc = s4;
        }
        float v = 0.0f;
        if (layer) {
            const uint64_t h = ckey(seed, 8, ((uint64_t)layer << 16) | (uint64_t)o, (uint64_t)in);
            const int s = (int)((h >> 40) & 0xFFFFFF) - 8388608;
            v = __fmul_rn((float)s, sc);
        }
        w[i] = v;
        m[i] = 0.0f;
    }
}

// ---- per-slot tensor addressing ---------------------------------------------------------
struct SlotView {
    int slot, bs;
    const float* w;
    float* act;
};
__device__ __forceinline__ SlotView slot_view(const ConvArgs& p, int slot) {
    SlotView v;
    v.slot = slot;
    v.bs = conv_bs(p, slot);
    v.w = p.slab + p.slab_stride * slot;
    v.act = p.act + p.al.stride * slot;
    return v;
}
template <int L>
__device__ __forceinline__ const float* layer_in(const ConvArgs& p, const SlotView& v) {
    if (L == 1) return p.x + conv_row0(p, v.slot) * kSample;
    return v.act + (L == 2 ? p.al.a1 : p.al.a2);
}
template <int L>
__device__ __forceinline__ float* layer_out(const ConvArgs& p, const SlotView& v) {
    return v.act + (L == 1 ? p.al.a1 : L == 2 ? p.al.a2 : p.al.a3);
}
template <int L>
__device__ __forceinline__ float* layer_dout(const ConvArgs& p, const SlotView& v) {  // dL/d(out of L)
    return v.act + (L == 1 ? p.al.d1 : L == 2 ? p.al.d2 : p.al.d3);
}

// ---- exact mode: SIMT convolutions in the oracle's order ---------------------------------
// out[n][p][co] = relu(b[co] + sum_{t valid asc} sum_{ci < Cr asc} in * W[co][t][ci])
template <int L>
__global__ void __launch_bounds__(256) conv_fwd_simt(ConvArgs p) {
    using G = Geo<L>;
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const long long total = (long long)v.bs * G::OH * G::OH * G::Co;
    const float* in = layer_in<L>(p, v);
    float* out = layer_out<L>(p, v);
    const float* W = v.w + G::OffW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int co = (int)(i % G::Co);
        const long long m = i / G::Co;
        const int n = (int)(m / (G::OH * G::OH)), pix = (int)(m % (G::OH * G::OH));
        const int oh = pix / G::OH, ow = pix % G::OH;
        float acc = 0.0f;
        for (int t = 0; t < 9; ++t) {
            const int ih = oh * G::S + t / 3 - 1, iw = ow * G::S + t % 3 - 1;
            if (ih < 0 || ih >= G::H || iw < 0 || iw >= G::H) continue;
            const float* xin = in + (((long long)n * G::H + ih) * G::H + iw) * G::Ci;
            const float* wr = W + ((long long)co * 9 + t) * G::Ci;
            for (int ci = 0; ci < G::Cr; ++ci) acc = __fmaf_rn(xin[ci], wr[ci], acc);
        }
        const float r = __fadd_rn(acc, v.w[G::OffB + co]);
        out[m * G::Co + co] = r > 0.0f ? r : 0.0f;
    }
}

// gW[co][t][ci] = sum_{n asc, p asc, valid} dy * in;  gb[co] = sum dy (sequential)
template <int L>
__global__ void __launch_bounds__(128) conv_wgrad_simt(ConvArgs p) {
    using G = Geo<L>;
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int nw = G::Co * 9 * G::Ci;
    if (i >= nw + G::Co) return;
    const float* in = layer_in<L>(p, v);
    const float* dy = layer_dout<L>(p, v);
    float* g = p.grad + p.grad_stride * v.slot;
    const int npix = G::OH * G::OH;
    if (i >= nw) {
        const int co = i - nw;
        float s = 0.0f;
        for (long long m = 0; m < (long long)v.bs * npix; ++m) s = __fadd_rn(s, dy[m * G::Co + co]);
        g[G::OffB + co] = s;
        return;
    }
    const int co = i / (9 * G::Ci), t = (i / G::Ci) % 9, ci = i % G::Ci;
    float acc = 0.0f;
    if (ci < G::Cr) {
        const int kh = t / 3, kw = t % 3;
        for (int n = 0; n < v.bs; ++n)
            for (int pix = 0; pix < npix; ++pix) {
                const int oh = pix / G::OH, ow = pix % G::OH;
                const int ih = oh * G::S + kh - 1, iw = ow * G::S + kw - 1;
                if (ih < 0 || ih >= G::H || iw < 0 || iw >= G::H) continue;
                acc = __fmaf_rn(dy[((long long)n * npix + pix) * G::Co + co],
                                in[(((long long)n * G::H + ih) * G::H + iw) * G::Ci + ci], acc);
            }
    }
    g[G::OffW + i] = acc;
}

// dx[n][q][ci] = (act > 0) ? sum_{t asc valid} sum_{co asc} dy * W[co][t][ci] : 0
template <int L>
__global__ void __launch_bounds__(256) conv_dgrad_simt(ConvArgs p) {
    using G = Geo<L>;
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const long long total = (long long)v.bs * G::H * G::H * G::Ci;
    const float* dy = layer_dout<L>(p, v);
    const float* act = layer_out<L - 1>(p, v);
    float* dx = layer_dout<L - 1>(p, v);
    const float* W = v.w + G::OffW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int ci = (int)(i % G::Ci);
        const long long q = i / G::Ci;
        const int n = (int)(q / (G::H * G::H)), pix = (int)(q % (G::H * G::H));
        const int ih = pix / G::H, iw = pix % G::H;
        float acc = 0.0f;
        for (int t = 0; t < 9; ++t) {
            const int nh = ih + 1 - t / 3, nw = iw + 1 - t % 3;
            if (nh < 0 || nw < 0 || nh % G::S || nw % G::S) continue;
            const int oh = nh / G::S, ow = nw / G::S;
            if (oh >= G::OH || ow >= G::OH) continue;
            const float* d = dy + (((long long)n * G::OH + oh) * G::OH + ow) * G::Co;
            const float* wr = W + (long long)t * G::Ci + ci;
            for (int co = 0; co < G::Co; ++co) acc = __fmaf_rn(d[co], wr[(long long)co * 9 * G::Ci], acc);
        }
        dx[i] = act[i] > 0.0f ? acc : 0.0f;
    }
}

// ---- head (both modes): pool + FC + softmax-CE, loss, FC grads, dA3 --------------------------
// grid (max_batch, groups), block 128: one sample per block.
// g[c] = (sum_{p asc} a3[p][c]) * 2^-6;  z[k] = fmaf chain over c of g[c]*W4[k][c], + b4[k]
// train: dz = (softmax - onehot) / B, row loss, then the sample's dA3 (pool / ReLU backward);
// eval (zout != null): logits to zout.
__global__ void __launch_bounds__(128) head_fwd_kernel(ConvArgs p) {
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const int n = blockIdx.x;
    if (n >= v.bs) return;
    __shared__ float g[kFeat];
    __shared__ float z[kNCP];
    const int c = threadIdx.x;
    if (p.pooled) {  // pooled by the conv3 forward epilogue (same order and scaling)
        g[c] = v.act[p.al.g + (long long)n * kFeat + c];
    } else {
        const float* a3 = v.act + p.al.a3 + (long long)n * 64 * kFeat;
        float s = 0.0f;
#pragma unroll 16
        for (int pix = 0; pix < 64; ++pix) s = __fadd_rn(s, __ldg(a3 + pix * kFeat + c));  // loads run ahead
        g[c] = __fmul_rn(s, 0.015625f);
        if (!p.zout) v.act[p.al.g + (long long)n * kFeat + c] = g[c];
    }
    __syncthreads();
    if (p.pooled) {
        // tensor-core mode: warp w computes z[4w .. 4w + 3], lane = 4 strided channels, then a
        // fixed shuffle tree (instead of one 128-long fmaf chain per output: the head is latency-bound)
        const int lane = c & 31, w = c >> 5;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int k = 4 * w + kk;
            const float* wr = v.w + kOffW4 + k * kFeat;
            float acc = 0.0f;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc = __fmaf_rn(g[lane + 32 * j], __ldg(wr + lane + 32 * j), acc);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
            if (lane == 0) {
                z[k] = __fadd_rn(acc, v.w[kOffB4 + k]);
                if (p.zout) p.zout[p.z_stride * blockIdx.y + ((long long)p.x_row0 + n) * kNCP + k] = z[k];
            }
        }
    } else if (c < kNCP) {  // exact mode: the oracle's chain
        const float* wr = v.w + kOffW4 + c * kFeat;
        float acc = 0.0f;
        for (int i = 0; i < kFeat; ++i) acc = __fmaf_rn(g[i], wr[i], acc);
        z[c] = __fadd_rn(acc, v.w[kOffB4 + c]);
        if (p.zout) p.zout[p.z_stride * blockIdx.y + ((long long)p.x_row0 + n) * kNCP + c] = z[c];
    }
    __syncthreads();
    if (p.zout) return;
    __shared__ float dzs[kNCP];
    if (c == 0) {
        const int y = p.labels[conv_row0(p, v.slot) + n];
        float dz[kNC];
        const float l = softmax_ce_row(z, y, dz, nullptr);
        v.act[p.al.rl + n] = l;
        float* dzo = v.act + p.al.dz + (long long)n * kNCP;
        const float fb = (float)v.bs;
        for (int k = 0; k < kNC; ++k) dzs[k] = dzo[k] = __fdiv_rn(dz[k], fb);
        for (int k = kNC; k < kNCP; ++k) dzs[k] = dzo[k] = 0.0f;
    }
    // the pool / ReLU backward of this sample (formerly head_dg_kernel, same arithmetic):
    // dg[c] = (fmaf chain over k < 16 of dz * W4[k][c]) * 2^-6; d3[n][p][c] = (a3 > 0) ? dg[c] : 0
    __shared__ float dgs[kFeat];
    __shared__ uint32_t mks[64 * (kFeat / 32)];
    const uint32_t* mk = reinterpret_cast<const uint32_t*>(v.act + p.al.mk3) + (long long)n * 64 * (kFeat / 32);
    if (p.pooled)  // a3 > 0 as the bitmap the conv3 forward epilogue wrote: word (n, pix, c / 32), staged coalesced
        for (int i = c; i < 64 * (kFeat / 32); i += 128) mks[i] = __ldg(mk + i);
    __syncthreads();
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < kNCP; ++k) acc = __fmaf_rn(dzs[k], v.w[kOffW4 + k * kFeat + c], acc);
    dgs[c] = __fmul_rn(acc, 0.015625f);
    __syncthreads();
    // thread = 4 channels (cq) x 16 pixels (pg): 16-byte stores, a warp writes 512 contiguous bytes
    const int cq = c & 31, pg = c >> 5;
    const float4 dg4 = reinterpret_cast<const float4*>(dgs)[cq];
    float4* d3 = reinterpret_cast<float4*>(v.act + p.al.d3 + (long long)n * 64 * kFeat) + cq;
    const float4* a3 = reinterpret_cast<const float4*>(v.act + p.al.a3 + (long long)n * 64 * kFeat) + cq;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
        const int pix = pg * 16 + i;
        bool m0, m1, m2, m3;
        if (p.pooled) {
            const uint32_t w = mks[pix * (kFeat / 32) + (cq >> 3)] >> ((cq & 7) * 4);
            m0 = w & 1u; m1 = (w >> 1) & 1u; m2 = (w >> 2) & 1u; m3 = (w >> 3) & 1u;
        } else {
            const float4 a = __ldg(a3 + pix * (kFeat / 4));
            m0 = a.x > 0.0f; m1 = a.y > 0.0f; m2 = a.z > 0.0f; m3 = a.w > 0.0f;
        }
        d3[pix * (kFeat / 4)] = make_float4(m0 ? dg4.x : 0.0f, m1 ? dg4.y : 0.0f, m2 ? dg4.z : 0.0f, m3 ? dg4.w : 0.0f);
    }
}

// grid (groups), block 256: loss = (sum_n rl) / B; gW4[k][c] = fmaf chain over n; gb4[k] = sum_n dz
// grid (17, groups), block 128: one output per thread (the chains are sequential in n, so the
// parallelism is across outputs; the loads are independent of the chain and unrolled ahead).
__global__ void __launch_bounds__(128) head_grad_kernel(ConvArgs p) {
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const float* dz = v.act + p.al.dz;
    const float* g = v.act + p.al.g;
    float* gr = p.grad + p.grad_stride * v.slot;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kNCP * kFeat) {
        const int k = i / kFeat, c = i % kFeat;
        float acc = 0.0f;
#pragma unroll 8
        for (int n = 0; n < v.bs; ++n) acc = __fmaf_rn(__ldg(dz + n * kNCP + k), __ldg(g + n * kFeat + c), acc);
        gr[kOffW4 + i] = acc;
    } else if (i < kNCP * kFeat + kNCP) {
        const int k = i - kNCP * kFeat;
        float s = 0.0f;
#pragma unroll 8
        for (int n = 0; n < v.bs; ++n) s = __fadd_rn(s, __ldg(dz + n * kNCP + k));
        gr[kOffB4 + k] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        float s = 0.0f;
        for (int n = 0; n < v.bs; ++n) s = __fadd_rn(s, v.act[p.al.rl + n]);
        p.loss_hist[(long long)v.slot * p.hp_cap + p.st[v.slot].step] = __fdiv_rn(s, (float)v.bs);
    }
}

// ---- tensor-core mode: implicit-GEMM Op policies for conv_ws.cuh ---------------------------
// Each Op describes one GEMM-shaped conv pass: its per-group setup, the implicit-GEMM address
// functions of the A operand (row decode once per tile, tap decode once per K chunk), the B
// operand (pre-split weight image or register gather) and the epilogue target.
namespace ctc {
using namespace smx::tc3;

enum { kEpiBiasRelu = 0, kEpiMask = 1, kEpiPartT = 2, kEpiBias = 3, kEpiStore = 4 };

// source of zero-filled 16-byte copies (cp.async reads 0 bytes from it)
__device__ __align__(16) float kZero16[4] = {0.0f, 0.0f, 0.0f, 0.0f};

// Forward: C[m = (n, oh, ow)][co] = relu(b + sum_{k = (t, ci)} im2col(in)[m][k] W[co][k])
template <int L>
struct Fwd {
    using G = Geo<L>;
    static constexpr int AM = 0, BMODE = 0, EPI = kEpiBiasRelu, kMaxN = G::Co;
    static constexpr bool A_EXACT = (L == 1), B_EXACT = false, B_IMAGE = true, B_TMA = false;
    static constexpr bool A_TMA = (L >= 2);  // A tile = one strided TMA box per chunk
    static constexpr int kOnesRow = -1, kPartLd = 0, kSegChunks = SMX_SEG_CHUNKS, kEpiWarps = L == 3 ? 8 : 4;
    static constexpr int kRowsPerSample = G::OH * G::OH;
    // the ReLU masks the input gradients read are bitmaps: a1's is written by the conv1 forward
    // epilogue, a3's by the pooled conv3 epilogue, and a2's by the conv3 forward producers (the taps
    // (kh, kw) in {1, 2}^2 of a stride-2 conv visit every input pixel exactly once, and a producer
    // thread holds 32 consecutive channels of it).  (The conv2 forward epilogue writing a2's bits
    // instead made that 4-warp epilogue the kernel's bottleneck: 470 -> 620 us.)
    static constexpr bool kInMaskBits = (L == 3), kMaskFromBits = false, kSgd = false;
    // conv3: the epilogue pools each sample's 64 output pixels into g (the head's input, in
    // head_fwd's order) and writes the a3 > 0 bitmap for head_dg instead of storing a3 itself
    static constexpr bool kPool = (L == 3);
    float* gout;
    uint32_t* mk_out;
    uint32_t* in_bits;
    const CUtensorMap* tmap;
    const float* in;
    const float* w;
    const float* bias;
    float* out;
    const float* img;
    int M, N, K, kbeg, m0, split;
    struct RowInfo {
        const float* ptr;  // input element (top-left of the 3x3 window, channel 0); may be out of range
        uint32_t vmask;    // bit t: tap t of the window lies inside the image (0 for rows >= M)
    };
    using Args = ConvArgs;
    __device__ __forceinline__ float4 bias4(int col) const { return __ldg(reinterpret_cast<const float4*>(bias + col)); }
    __device__ __forceinline__ void store4(int m, int col, float4 x) const {
        *reinterpret_cast<float4*>(out + (long long)m * G::Co + col) = x;
    }
    __device__ void setup(const ConvArgs& p, int z, int tile_y) {
        const SlotView v = slot_view(p, p.slots[z]);
        img = v.act + (L == 1 ? p.al.wf1 : L == 2 ? p.al.wf2 : p.al.wf3);
        tmap = p.tmaps + (long long)v.slot * kTmapKinds + (L == 3 ? kTmFwd3 : kTmFwd2);
        in_bits = reinterpret_cast<uint32_t*>(v.act + (L == 3 ? p.al.mk2 : p.al.mk1));
        gout = v.act + p.al.g;
        mk_out = reinterpret_cast<uint32_t*>(v.act + p.al.mk3);
        in = layer_in<L>(p, v);
        w = v.w + G::OffW;
        bias = v.w + G::OffB;
        out = layer_out<L>(p, v);
        M = v.bs * G::OH * G::OH;
        N = G::Co;
        K = 9 * G::Ci;
        kbeg = 0;
        split = 0;
        (void)tile_y;
    }
    __device__ __forceinline__ const float* a_ptr(int m, int k) const {
        const int n = m / (G::OH * G::OH), pix = m % (G::OH * G::OH);
        const int t = k / G::Ci, ci = k % G::Ci;
        const int ih = (pix / G::OH) * G::S + t / 3 - 1, iw = (pix % G::OH) * G::S + t % 3 - 1;
        if (ih < 0 || ih >= G::H || iw < 0 || iw >= G::H) return nullptr;
        return in + (((long long)n * G::H + ih) * G::H + iw) * G::Ci + ci;
    }
    __device__ __forceinline__ RowInfo row_info(int m) const {
        if (m >= M) return RowInfo{in, 0u};
        const int n = m / (G::OH * G::OH), pix = m % (G::OH * G::OH);
        const int ih0 = (pix / G::OH) * G::S - 1, iw0 = (pix % G::OH) * G::S - 1;
        uint32_t mask = 0;
#pragma unroll
        for (int t = 0; t < 9; ++t)
            if ((unsigned)(ih0 + t / 3) < (unsigned)G::H && (unsigned)(iw0 + t % 3) < (unsigned)G::H) mask |= 1u << t;
        return RowInfo{in + (n * G::H * G::H + ih0 * G::H + iw0) * G::Ci, mask};
    }
    // per-chunk decode of a producer's k (shared by its 4 rows), then per-row pointer
    struct TapInfo {
        int off, bit;  // element offset from the window origin; mask bit (31: k beyond K)
    };
    __device__ __forceinline__ TapInfo tap_info(int k) const {
        const int t = k / G::Ci;
        return k < K ? TapInfo{((t / 3) * G::H + t % 3) * G::Ci + k % G::Ci, t} : TapInfo{0, 31};
    }
    __device__ __forceinline__ const float* a_ptr_tap(const RowInfo& r, const TapInfo& t) const {
        return (r.vmask >> t.bit) & 1u ? r.ptr + t.off : nullptr;
    }
    __device__ __forceinline__ const float* b_image(int c) const { return img + (long long)c * N * 64; }
    // TMA box origin (channel, column, row, sample) of M tile `tile`, reduction chunk k0: output
    // rows (n, oh, ow) -> input (2 oh + kh - 1, 2 ow + kw - 1), one tap and 32 channels per chunk
    static constexpr int kBoxes = 1;
    __device__ __forceinline__ int a_nbox(int) const { return 1; }
    __device__ __forceinline__ void a_coords(int tile, int k0, int, int* c) const {
        const int m0 = tile * kBM, t = k0 / G::Ci;
        const int n = m0 / kRowsPerSample, oh0 = (m0 % kRowsPerSample) / G::OH;
        c[0] = k0 % G::Ci;
        c[1] = t % 3 - 1;
        c[2] = G::S * oh0 + t / 3 - 1;
        c[3] = n;
    }
    __device__ __forceinline__ const float* b_ptr(int co, int k) const { return w + (long long)co * 9 * G::Ci + k; }
    // bitmap word of row m's input pixel for reduction chunk k0 (nullptr: not a recording tap)
    __device__ __forceinline__ uint32_t* in_bits_word(int m, int k0) const {
        const int t = k0 / G::Ci, kh = t / 3, kw = t % 3;
        if (kh == 0 || kw == 0 || m >= M) return nullptr;
        const int n = m / kRowsPerSample, pix = m % kRowsPerSample;
        const int ih = G::S * (pix / G::OH) + kh - 1, iw = G::S * (pix % G::OH) + kw - 1;
        return in_bits + ((((long long)n * G::H + ih) * G::H + iw) * G::Ci + k0 % G::Ci) / 32;
    }
    __device__ __forceinline__ float* c_row(int m) const { return out + (long long)m * G::Co; }
    __device__ __forceinline__ float* c_at(int m, int col) const { return out + (long long)m * G::Co + col; }
    __device__ __forceinline__ const float* mask_row(int) const { return nullptr; }
    __device__ __forceinline__ const float* mask_at(int, int) const { return nullptr; }
};

// Input gradient of a stride-2 layer as one dense "sub-pixel" GEMM: row r = (n, a, b) stands
// for the 2x2 input block (2a + pi, 2b + pj), column = (class pi*2+pj, ci), reduction k =
// (output neighbour (a + da, b + db), co).  An input pixel of class (pi, pj) receives tap
// kh = (pi ? (da ? 0 : 2) : 1) from output row a + da (da = 0 only for pi = 0), likewise kw, so
// B[(cls, ci)][(da, db, co)] = W[co][kh][kw][ci] or 0: 9 of the 16 (class, neighbour) pairs are
// taps.  Versus one GEMM per parity class this gathers each output-gradient block once for 4
// input pixels (4/9 of the gather work) with N = 4 Ci instead of Ci.
// blockIdx.x selects the 128-column half of N when 4 Ci > 128.
template <int L>
struct Dgrad {
    using G = Geo<L>;
    static_assert(G::S == 2, "sub-pixel decomposition is for stride 2");
    static constexpr int AM = 0, BMODE = 0, EPI = kEpiMask, kMaxN = WImg<L>::DgrNTile;
    static constexpr bool A_EXACT = false, B_EXACT = false, B_IMAGE = true, B_TMA = false;
    static constexpr bool A_TMA = true;  // A tile = one shifted TMA box of dy per chunk
    static constexpr bool kInMaskBits = false, kMaskFromBits = true, kSgd = false;
    static constexpr int kOnesRow = -1, kPartLd = 0, kSegChunks = SMX_DGR_SEG_CHUNKS, kEpiWarps = 8;
    static constexpr int HH = G::H / 2;  // == OH
    // The tile's output is staged in shared memory in the 128B-swizzled layout of TMA boxes and
    // written by tensor stores (conv_ws TmaOut): conv2 = 16 input rows x 32 columns x 32 channels
    // of one sample (64 KB contiguous in d1, one kTmD1 box); conv3 = the N tile's parity row pi of
    // 2 samples (8 rows x 16 columns x 64 channels each), two kTmD2 boxes of 32 channels
    static constexpr bool kTmaOut = true;
    // conv2: chunk c = output neighbour c % 4 x channels 32 (c / 4) ..; the 4 neighbours' A tiles
    // are windows of one TMA box of dy (the tile's 8 output rows + 1 x 16 columns + 1, zero
    // filled past the image: 9 x 17 pixels x 32 channels) read from one raw slot (conv_ws ANbrBox).
    // The reduction order changes with it: a 4-chunk accumulation segment = one 32-channel group
    // over all neighbours.
    static constexpr bool kANbrBox = (L == 2);
    static constexpr int kABoxBytes = 32 * 17 * 9 * 4;
    __host__ __device__ static constexpr int chunk_k0(int c) {
        return L == 2 ? (c & 3) * G::Co + (c >> 2) * 32 : c * 32;
    }
    // line (pixel) of the neighbour box holding row r's A values for chunk c
    __device__ __forceinline__ int a_line(int r, int c) const {
        const int nb = c & 3;
        return ((r / HH) + (nb >> 1)) * 17 + (r % HH) + (nb & 1);
    }
    // neighbour box origin (channel, column, row, sample) of tile `tile`, channel group cu
    __device__ __forceinline__ void a_box(int tile, int cu, int* c) const {
        const int m0 = tile * kBM;
        c[0] = cu * 32;
        c[1] = 0;
        c[2] = (m0 % (HH * HH)) / HH;
        c[3] = m0 / (HH * HH);
    }
    // Column position -> parity class.  conv2 orders its 4 classes 0, 1, 3, 2 so that the classes
    // fed by each output neighbour (da, db) -- those with (pi or !da) and (pj or !db) -- are
    // contiguous: (0,0) all, (0,1) {1, 3}, (1,0) {3, 2}, (1,1) {3}; the MMAs of a K chunk then
    // cover only those columns (conv_ws ColRanges): 9 of the 16 class x neighbour blocks are issued.
    static constexpr bool kColRanges = true;
    static __host__ __device__ constexpr int cls_at(int pos) { return (L == 2 && pos >= 2) ? (pos ^ 1) : pos; }
    __device__ __forceinline__ void chunk_cols(int k0, int& off, int& n) const { chunk_cols_at(col0, k0, off, n); }
    __host__ __device__ static void chunk_cols_at(int col0, int k0, int& off, int& n) {
        const int nb = k0 / G::Co, da = nb >> 1, db = nb & 1;
        constexpr int P = WImg<L>::DgrNTile / G::Ci;  // class positions per N tile
        int lo = P, hi = -1;
#pragma unroll
        for (int pp = 0; pp < P; ++pp) {
            const int cls = cls_at(col0 / G::Ci + pp), pi = cls >> 1, pj = cls & 1;
            if ((pi || !da) && (pj || !db)) {
                lo = min(lo, pp);
                hi = pp;
            }
        }
        off = lo * G::Ci;
        n = (hi - lo + 1) * G::Ci;
    }
    const CUtensorMap* tmap;
    const CUtensorMap* omap;  // kTmaOut: the output box map
    const float* dy;
    const float* w;
    const uint32_t* mbits;  // ReLU mask of the layer input as a bitmap (written by this layer's forward)
    float* dx;
    const float* img;
    int M, N, K, kbeg, m0, split;
    int col0;  // first (class, ci) column of this N tile
    struct RowInfo {
        const float* ptr;  // dy at output pixel (a, b), channel 0
        uint32_t vmask;    // bit 2 da + db: neighbour (a + da, b + db) exists (0 for rows >= M)
    };
    using Args = ConvArgs;
    __device__ void setup(const ConvArgs& p, int z, int half) {
        const SlotView v = slot_view(p, p.slots[z]);
        dy = layer_dout<L>(p, v);
        tmap = p.tmaps + (long long)v.slot * kTmapKinds + (L == 2 ? kTmDgr2 : kTmDgr3);
        omap = p.tmaps + (long long)v.slot * kTmapKinds + (L == 2 ? kTmD1 : kTmD2);
        w = v.w + G::OffW;
        mbits = reinterpret_cast<const uint32_t*>(v.act + (L == 2 ? p.al.mk1 : p.al.mk2));
        dx = layer_dout<L - 1>(p, v);
        N = WImg<L>::DgrNTile;
        col0 = half * N;
        img = v.act + (L == 2 ? p.al.wd2 : p.al.wd3) + (long long)half * WImg<L>::DgrChunks * N * 64;
        M = v.bs * HH * HH;
        // an N tile of one parity row pi (conv3: 2 classes x 64 cin) has no taps from the
        // neighbours below (da = 1) when pi = 0: its reduction stops after (da = 0, db = 0 / 1)
        K = (N == 2 * G::Ci && half == 0) ? 2 * G::Co : 4 * G::Co;
        kbeg = 0;
        split = 0;
    }
    __device__ __forceinline__ RowInfo row_info(int r) const {
        if (r >= M) return RowInfo{dy, 0u};
        const int n = r / (HH * HH), q = r % (HH * HH);
        const int a = q / HH, b = q % HH;
        const uint32_t mask = 1u | (b + 1 < G::OH ? 2u : 0u) | (a + 1 < G::OH ? 4u : 0u) |
                              (a + 1 < G::OH && b + 1 < G::OH ? 8u : 0u);
        return RowInfo{dy + ((n * G::OH + a) * G::OH + b) * G::Co, mask};
    }
    struct TapInfo {
        int off, bit;
    };
    __device__ __forceinline__ TapInfo tap_info(int k) const {
        const int nb = k / G::Co;  // neighbour (da, db) = (nb >> 1, nb & 1)
        return k < K ? TapInfo{((nb >> 1) * G::OH + (nb & 1)) * G::Co + k % G::Co, nb} : TapInfo{0, 31};
    }
    __device__ __forceinline__ const float* a_ptr_tap(const RowInfo& r, const TapInfo& t) const {
        return (r.vmask >> t.bit) & 1u ? r.ptr + t.off : nullptr;
    }
    __device__ __forceinline__ const float* b_image(int c) const { return img + (long long)c * N * 64; }
    // TMA box origin (channel, column, row, sample): rows (n, a, b) of M tile `tile` read dy at
    // (a + da, b + db), channels co0 .. co0 + 31 of chunk k0 = (neighbour, co0)
    static constexpr int kBoxes = 1;
    __device__ __forceinline__ int a_nbox(int) const { return 1; }
    __device__ __forceinline__ void a_coords(int tile, int k0, int, int* c) const {
        const int m0 = tile * kBM, nb = k0 / G::Co;
        c[0] = k0 % G::Co;
        c[1] = nb & 1;
        c[2] = (m0 % (HH * HH)) / HH + (nb >> 1);
        c[3] = m0 / (HH * HH);
    }
    // epilogue column c (0..N-1) -> (class, ci); rows write 4 input pixels
    __device__ __forceinline__ long long pix_off(int r, int col) const {
        const int cc = col0 + col, cls = cls_at(cc / G::Ci);
        const int n = r / (HH * HH), q = r % (HH * HH);
        const int ih = 2 * (q / HH) + (cls >> 1), iw = 2 * (q % HH) + (cls & 1);
        return (((long long)n * G::H + ih) * G::H + iw) * G::Ci + cc % G::Ci;
    }
    __device__ __forceinline__ float* c_at(int r, int col) const { return dx + pix_off(r, col); }
    __device__ __forceinline__ const void* mask_at(int r, int col) const { return mbits + (pix_off(r, col) >> 5); }
    // masked epilogue: the output element's offset (input pixel, channel) is also its mask bit;
    // the 4 channels of a float4 lie in one 32-bit word
    __device__ __forceinline__ long long mask_off(int r, int col) const { return pix_off(r, col); }
    __device__ __forceinline__ uint32_t mask_word(int r, int col) const { return __ldg(mbits + (pix_off(r, col) >> 5)); }
    __device__ __forceinline__ void store_masked(int, int, long long off, float4 x) const {
        __stcs(reinterpret_cast<float4*>(dx + off), x);  // streaming: read next by another kernel
    }
    // kTmaOut staging of tile row `row`, 16 columns [col, col + 16) (4 channel quads of one class),
    // r = their values of one accumulation segment: the first segment writes them, later ones add
    // (round-to-nearest), and the segment that completes the columns applies the ReLU mask (word
    // mw: the pixel's 32 channel bits of these columns).  A box line (128 bytes) holds 32 channels
    // of one input pixel; conv2: line (2 a + pi) x 32 + 2 b + pj, conv3: box ci / 32, line
    // (sample x 8 + a) x 16 + 2 b + pj.  16-byte unit u sits at u ^ (line & 7) (SWIZZLE_128B).
    // Lanes b and b + 4 would share units, so lanes with bit 2 of b set take the units of each pair
    // in the order u ^ 1: every 8 lanes then cover the 8 units of a bank row (4 wavefronts per
    // warp store).
    __device__ __forceinline__ void stage16(char* stg, int row, int col, const uint32_t* r, bool first, bool last,
                                            uint32_t mw) const {
        const int b = row % HH, rot = (b >> 2) & 1;
        const int cls = cls_at((col0 + col) / G::Ci), pi = cls >> 1, pj = cls & 1, ci = (col0 + col) % G::Ci;
        int Ln;
        char* box = stg;
        if constexpr (L == 2) {
            Ln = (2 * (row / HH) + pi) * 32 + 2 * b + pj;
        } else {
            Ln = ((row / (HH * HH)) * HH + (row / HH) % HH) * 16 + 2 * b + pj;
            box += (ci >> 5) * 32768;
        }
        char* line = box + Ln * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int u = (((ci & 31) >> 2) + j) ^ rot;  // channel quad written by this step
            float4 v;
            v.x = __uint_as_float(rot ? r[4 * (j ^ 1)] : r[4 * j]);
            v.y = __uint_as_float(rot ? r[4 * (j ^ 1) + 1] : r[4 * j + 1]);
            v.z = __uint_as_float(rot ? r[4 * (j ^ 1) + 2] : r[4 * j + 2]);
            v.w = __uint_as_float(rot ? r[4 * (j ^ 1) + 3] : r[4 * j + 3]);
            float4* dst = reinterpret_cast<float4*>(line + ((u ^ (Ln & 7)) << 4));
            if (!first) {
                const float4 o = *dst;
                v.x = __fadd_rn(o.x, v.x);
                v.y = __fadd_rn(o.y, v.y);
                v.z = __fadd_rn(o.z, v.z);
                v.w = __fadd_rn(o.w, v.w);
            }
            if (last) {
                const uint32_t bits = mw >> (4 * u);
                v.x = (bits & 1u) ? v.x : 0.0f;
                v.y = (bits & 2u) ? v.y : 0.0f;
                v.z = (bits & 4u) ? v.z : 0.0f;
                v.w = (bits & 8u) ? v.w : 0.0f;
            }
            *dst = v;
        }
    }
    // the staged tile -> dx.  conv2: d1 rows 2 a0 .. 2 a0 + 15 of its sample (kTmD1: {32 channels,
    // 32 columns, max_batch x 32 rows}, box {32, 32, 16}).  conv3: d2 as {64 channels, 16 columns,
    // 2 row parities, 8 row pairs, max_batch} (kTmD2), boxes {32, 16, 1, 8, 2} at channels 0 / 32,
    // parity pi of this N tile, samples 2 tile, 2 tile + 1 (a partial last tile writes zeros into
    // sample bs < max_batch, which the step never reads, or is clipped at max_batch)
    __device__ __forceinline__ void store_tile(uint32_t stg, int tile) const {
        if constexpr (L == 2) {
            const int m0 = tile * kBM, n = m0 / (HH * HH), a0 = (m0 % (HH * HH)) / HH;
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(omap),
                         "r"(0), "r"(0), "r"(n * G::H + 2 * a0), "r"(stg)
                         : "memory");
        } else {
            const int pi = cls_at(col0 / G::Ci) >> 1;
#pragma unroll
            for (int bx = 0; bx < 2; ++bx)
                asm volatile(
                    "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(omap),
                    "r"(32 * bx), "r"(0), "r"(pi), "r"(0), "r"(2 * tile), "r"(stg + bx * 32768)
                    : "memory");
        }
    }
};

// Weight gradient, split s of the reduction: part[s][co][k] = sum_{m in split} im2col(in)[m][k] dy[m][co]
// (k = 9*Ci is the all-ones row: the bias gradient).
template <int L>
struct Wgrad {
    using G = Geo<L>;
    static constexpr int AM = 1, BMODE = 1, EPI = kEpiPartT, kMaxN = G::Co;
    static constexpr bool A_EXACT = (L == 1), B_EXACT = false, B_IMAGE = false, A_TMA = (L >= 2);
    // B = dY[m][co] (co contiguous: MN-major) by TMA, 32 co x 32 m boxes (SWIZZLE_128B_BASE32B)
    static constexpr bool B_TMA = (L >= 2);
    const CUtensorMap* btmap;
    static constexpr bool kInMaskBits = false, kMaskFromBits = false, kSgd = false;
    // TMA: a tile's 128 rows are 128 / Ci taps x Ci channels; one box per tap = 32 output pixels
    // (the chunk's reduction indices) x Ci channels, stored [tap][pixel][ci]
    static constexpr int kBoxes = 128 / G::Ci, kTmaCi = G::Ci;
    const CUtensorMap* tmap;
    __device__ __forceinline__ int a_nbox(int tile) const {
        const int t0 = tile * kBoxes;
        return t0 >= 9 ? 0 : (9 - t0 < kBoxes ? 9 - t0 : kBoxes);
    }
    __device__ __forceinline__ void a_coords(int tile, int k0, int b, int* c) const {
        const int t = tile * kBoxes + b;
        const int n = k0 / (G::OH * G::OH), oh0 = (k0 % (G::OH * G::OH)) / G::OH;
        c[0] = 0;
        c[1] = t % 3 - 1;
        c[2] = G::S * oh0 + t / 3 - 1;
        c[3] = n;
    }
    struct RowInfo {
        int kh, kw, ci;  // tap and first channel of a row quad (kh = -1000: padding rows)
    };
    // rows row..row+3 = (tap, 4 consecutive channels)
    __device__ __forceinline__ RowInfo row_info(int row) const {
        if (row >= kOnesRow) return RowInfo{-1000, 0, 0};
        const int t = row / G::Ci;
        return RowInfo{t / 3 - 1, t % 3 - 1, row % G::Ci};
    }
    // per-chunk decode of a reduction index (sample, output pixel), then the row quad's pointer
    struct RedInfo {
        int base, ih, iw, left;  // first pixel of a run; `left` reduction indices remain in range
    };
    __device__ __forceinline__ RedInfo red_info(int m) const {
        if (m >= kbeg + K) return RedInfo{0, -1000, -1000, 0};
        const int n = m / (G::OH * G::OH), pix = m % (G::OH * G::OH);
        return RedInfo{n * G::H * G::H * G::Ci, (pix / G::OH) * G::S, (pix % G::OH) * G::S, kbeg + K - m};
    }
    __device__ __forceinline__ const float* a_ptr_red(const RowInfo& ri, const RedInfo& rd) const {
        return a_ptr_red_step(ri, rd, 0);
    }
    // reduction index m + j of a run of 8 that starts at a multiple of 8 (same output row: OH % 8 == 0)
    __device__ __forceinline__ const float* a_ptr_red_step(const RowInfo& ri, const RedInfo& rd, int j) const {
        const int ih = rd.ih + ri.kh, iw = rd.iw + G::S * j + ri.kw;
        if (j >= rd.left || (unsigned)ih >= (unsigned)G::H || (unsigned)iw >= (unsigned)G::H) return nullptr;
        return in + (rd.base + (ih * G::H + iw) * G::Ci + ri.ci);
    }
    // the 4 rows of `ri` at reduction index m (sample, output pixel)
    __device__ __forceinline__ const float* a_ptr_ri(const RowInfo& ri, int m) const {
        const int n = m / (G::OH * G::OH), pix = m % (G::OH * G::OH);
        const int ih = (pix / G::OH) * G::S + ri.kh, iw = (pix % G::OH) * G::S + ri.kw;
        if ((unsigned)ih >= (unsigned)G::H || (unsigned)iw >= (unsigned)G::H || m >= kbeg + K) return nullptr;
        return in + ((n * G::H + ih) * G::H + iw) * G::Ci + ri.ci;
    }
    __device__ __forceinline__ const float* b_image(int) const { return nullptr; }
    static constexpr int kOnesRow = 9 * G::Ci, kPartLd = Part<L>::Ld, kSegChunks = SMX_SEG_CHUNKS, kEpiWarps = 4;
    const float* in;
    const float* dy;
    float* part;
    int M, N, K, kbeg, m0, split;
    using Args = ConvArgs;
    __device__ __forceinline__ float* ct_at(int col, int m) const {
        return part + ((long long)split * N + col) * kPartLd + m;
    }
    __device__ void setup(const ConvArgs& p, int z, int s) {
        const SlotView v = slot_view(p, p.slots[z]);
        in = layer_in<L>(p, v);
        dy = layer_dout<L>(p, v);
        tmap = p.tmaps + (long long)v.slot * kTmapKinds + (L == 3 ? kTmWg3 : kTmWg2);
        btmap = p.tmaps + (long long)v.slot * kTmapKinds + (L == 3 ? kTmWgB3 : kTmWgB2);
        part = v.act + (L == 1 ? p.al.p1 : L == 2 ? p.al.p2 : p.al.p3);
        const int total = v.bs * G::OH * G::OH;
        split = s;
        kbeg = s * kSplitRows;
        K = max(0, min(kSplitRows, total - kbeg));
        M = Part<L>::Rows;
        N = G::Co;
    }
    // A(row = (t, ci), reduction m): 4 consecutive ci contiguous
    __device__ __forceinline__ const float* a_ptr(int row, int m) const {
        const int t = row / G::Ci, ci = row % G::Ci;
        const int n = m / (G::OH * G::OH), pix = m % (G::OH * G::OH);
        const int ih = (pix / G::OH) * G::S + t / 3 - 1, iw = (pix % G::OH) * G::S + t % 3 - 1;
        if (ih < 0 || ih >= G::H || iw < 0 || iw >= G::H) return nullptr;
        return in + (((long long)n * G::H + ih) * G::H + iw) * G::Ci + ci;
    }
    __device__ __forceinline__ const float* b_ptr(int co, int m) const { return dy + (long long)m * G::Co + co; }
    __device__ __forceinline__ float* c_row(int) const { return nullptr; }
    __device__ __forceinline__ float* c_at(int, int) const { return nullptr; }
    __device__ __forceinline__ const float* mask_row(int) const { return nullptr; }
    __device__ __forceinline__ const float* mask_at(int, int) const { return nullptr; }
};

}  // namespace ctc

// Weight images (see WImg): one thread per 16-byte unit of the hi tile (and its lo twin).
// grid (blocks, groups), block 256.
__device__ __forceinline__ float tf32_rna_h(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
template <int L>
__device__ __forceinline__ void weight_image_body(const ConvArgs& p, int bx, int nbx) {
    using G = Geo<L>;
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const float* W = v.w + G::OffW;
    const int fwd_units = WImg<L>::FwdChunks * 8 * G::Co;
    const int dgr_units = (L >= 2) ? WImg<L>::DgrChunks * 8 * WImg<L>::DgrN : 0;
    for (int u = bx * blockDim.x + threadIdx.x; u < fwd_units + dgr_units; u += nbx * blockDim.x) {
        float val[4];
        float* dst;
        int nt;
        if (u < fwd_units) {  // rows co, k = (tap, ci)
            nt = G::Co;
            const int c = u / (8 * nt), kq = (u / nt) % 8, r = u % nt;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = c * 32 + kq * 4 + e;
                val[e] = k < 9 * G::Ci ? W[r * 9 * G::Ci + k] : 0.0f;
            }
            dst = v.act + (L == 1 ? p.al.wf1 : L == 2 ? p.al.wf2 : p.al.wf3) + (long long)c * nt * 64 +
                  (kq * nt * 16 + (r >> 3) * 128 + (r & 7) * 16) / 4;
        } else {  // rows (class, ci), k = (neighbour (da, db), co)
            const int uu = u - fwd_units;
            constexpr int NT = WImg<L>::DgrNTile;
            const int half = uu / (WImg<L>::DgrChunks * 8 * NT);
            const int rem = uu % (WImg<L>::DgrChunks * 8 * NT);
            const int c = rem / (8 * NT), kq = (rem / NT) % 8, r = rem % NT;
            nt = NT;
            // rows outside the chunk's column range are never read (the MMAs of a K chunk cover only
            // the classes its neighbour feeds, conv_ws ColRanges): not written
            {
                int off, n;
                ctc::Dgrad<(L >= 2 ? L : 2)>::chunk_cols_at(half * NT, ctc::Dgrad<(L >= 2 ? L : 2)>::chunk_k0(c), off, n);
                if (r < off || r >= off + n) continue;
            }
            const int cc = half * NT + r, cls = ctc::Dgrad<(L >= 2 ? L : 2)>::cls_at(cc / G::Ci), ci = cc % G::Ci;
            const int pi = cls >> 1, pj = cls & 1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = ctc::Dgrad<(L >= 2 ? L : 2)>::chunk_k0(c) + kq * 4 + e;
                const int nb = k / G::Co, co = k % G::Co, da = nb >> 1, db = nb & 1;
                const int kh = pi ? (da ? 0 : 2) : (da ? -1 : 1);
                const int kw = pj ? (db ? 0 : 2) : (db ? -1 : 1);
                val[e] = (kh >= 0 && kw >= 0) ? W[(co * 9 + kh * 3 + kw) * G::Ci + ci] : 0.0f;
            }
            dst = v.act + (L == 2 ? p.al.wd2 : p.al.wd3) + (long long)half * WImg<L>::DgrChunks * NT * 64 +
                  (long long)c * NT * 64 + (kq * NT * 16 + (r >> 3) * 128 + (r & 7) * 16) / 4;
        }
        float4 hi, lo;
        hi.x = tf32_rna_h(val[0]); lo.x = tf32_rna_h(__fsub_rn(val[0], hi.x));
        hi.y = tf32_rna_h(val[1]); lo.y = tf32_rna_h(__fsub_rn(val[1], hi.y));
        hi.z = tf32_rna_h(val[2]); lo.z = tf32_rna_h(__fsub_rn(val[2], hi.z));
        hi.w = tf32_rna_h(val[3]); lo.w = tf32_rna_h(__fsub_rn(val[3], hi.w));
        *reinterpret_cast<float4*>(dst) = hi;
        *reinterpret_cast<float4*>(dst + nt * 32) = lo;  // lo tile follows the hi tile (nt*128 bytes)
    }
}

template <int L>
constexpr int wimg_units() {
    return WImg<L>::FwdChunks * 8 * Geo<L>::Co + (L >= 2 ? WImg<L>::DgrChunks * 8 * WImg<L>::DgrN : 0);
}
constexpr int kWImgBlocks1 = (wimg_units<1>() + 255) / 256, kWImgBlocks2 = (wimg_units<2>() + 255) / 256,
              kWImgBlocks3 = (wimg_units<3>() + 255) / 256;
// all three layers' images in one launch: grid (kWImgBlocks1 + 2 + 3, groups), block 256
__global__ void __launch_bounds__(256) weight_image_kernel(ConvArgs p) {
    const int b = blockIdx.x;
    if (b < kWImgBlocks1)
        weight_image_body<1>(p, b, kWImgBlocks1);
    else if (b < kWImgBlocks1 + kWImgBlocks2)
        weight_image_body<2>(p, b - kWImgBlocks1, kWImgBlocks2);
    else
        weight_image_body<3>(p, b - kWImgBlocks1 - kWImgBlocks2, kWImgBlocks3);
}

// ---- layer 1 in tensor-core mode: the tcgen05 kernels are in conv1_tc.cuh (round 1 ran conv1 on
// packed-FFMA2 CUDA-core kernels: FMA-pipe bound at 57-66 %, 331 + 434 us per 64-slot lockstep
// against 193 + 288 us now; profiles/r02/SUMMARY.md).  The partial rows they write are summed here.

// Sum the partial rows (one per `per_part` consecutive samples) in order into the gradient slab,
// or (fuse_update) apply K5 to the parameter in place.  grid (7, groups), block 128.
__global__ void __launch_bounds__(128) conv1_wgrad_reduce(ConvArgs p, int per_part) {
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    const float* part = v.act + p.al.w1p;
    float* g = p.grad + p.grad_stride * v.slot;
    float* w = p.slab + p.slab_stride * v.slot;
    float* m = w + p.slab_stride / 2;
    const SgdRow h = sgd_row(p.hp, p.hp_cap, p.st, v.slot);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kL1Outs; i += gridDim.x * blockDim.x) {
        float s_ = 0.0f;
#pragma unroll 8
        for (int n = 0; n < (v.bs + per_part - 1) / per_part; ++n) s_ = __fadd_rn(s_, __ldg(part + (long long)n * kL1Outs + i));
        const int co = i / 28, j = i % 28;
        const long long at = j < 27 ? Geo<1>::OffW + (co * 9 + j / 3) * 4 + j % 3 : Geo<1>::OffB + co;
        if (p.fuse_update)
            sgd_apply(w, m, at, s_, h);
        else
            g[at] = s_;
    }
    // the padded input channel's weights stay exactly zero (gradient 0; w = m = 0 untouched)
    if (blockIdx.x == 0 && !p.fuse_update)
        for (int i = threadIdx.x; i < 32 * 9; i += blockDim.x) g[Geo<1>::OffW + i * 4 + 3] = 0.0f;
}

// Weight-gradient reduction: grad[W][co][k] = sum_{s asc} part[s][co][k] (k < 9 Ci), grad[b][co]
// from the all-ones row; with fuse_update the sum is the gradient K5 applies in place (K3+K5:
// no gradient slab round trip).  grid (Co [+ kFcBlocks for L = 3 fused], groups), block 128.
// The fused L = 3 launch also updates the FC layer (W4 | b4, gradients from head_grad_kernel):
// it runs on the weight-gradient branch after head_dg_kernel, the last reader of W4.
constexpr int kFcParams = kNCP * kFeat + kNCP, kFcBlocks = (kFcParams + 127) / 128;
template <int L>
__global__ void __launch_bounds__(128) wgrad_reduce_kernel(ConvArgs p) {
    using G = Geo<L>;
    using P = Part<L>;
    const SlotView v = slot_view(p, p.slots[blockIdx.y]);
    float* w = p.slab + p.slab_stride * v.slot;
    float* m = w + p.slab_stride / 2;
    float* g = p.grad + p.grad_stride * v.slot;
    const SgdRow h = sgd_row(p.hp, p.hp_cap, p.st, v.slot);
    if ((int)blockIdx.x >= G::Co) {  // L = 3, fused: the FC parameters
        const int i = (blockIdx.x - G::Co) * 128 + threadIdx.x;
        if (i < kFcParams) sgd_apply(w, m, kOffW4 + i, __ldcs(g + kOffW4 + i), h);
        return;
    }
    const int co = blockIdx.x;
    const int nsplit = (v.bs * G::OH * G::OH + kSplitRows - 1) / kSplitRows;
    const float* part = v.act + (L == 1 ? p.al.p1 : L == 2 ? p.al.p2 : p.al.p3) + (long long)co * P::Ld;
    // all of the thread's elements at once (parameter / momentum loads issued first, then split by
    // split), each summed over the splits in ascending order
    constexpr int KI = (P::Rows + 127) / 128;
    static_assert(KI <= 8, "elements per thread");
    float s[KI], wv[KI], mv[KI];
    long long at[KI];
#pragma unroll
    for (int j = 0; j < KI; ++j) {
        const int k = threadIdx.x + 128 * j;
        at[j] = k >= P::Rows ? -1 : k < 9 * G::Ci ? G::OffW + (long long)co * 9 * G::Ci + k : G::OffB + co;
        s[j] = 0.0f;
        if (p.fuse_update && at[j] >= 0) {
            wv[j] = w[at[j]];
            mv[j] = m[at[j]];
        }
    }
    for (int i = 0; i < nsplit; ++i)
#pragma unroll
        for (int j = 0; j < KI; ++j)
            if (at[j] >= 0) s[j] = __fadd_rn(s[j], part[(long long)i * G::Co * P::Ld + threadIdx.x + 128 * j]);
#pragma unroll
    for (int j = 0; j < KI; ++j) {
        if (at[j] < 0) continue;
        if (p.fuse_update) {  // sgd_apply on the preloaded values
            const float mn = __fmaf_rn(h.mu, mv[j], __fmaf_rn(h.wd, wv[j], s[j]));
            m[at[j]] = mn;
            w[at[j]] = __fmaf_rn(h.nlr, mn, wv[j]);
        } else {
            g[at[j]] = s[j];
        }
    }
}

}  // namespace cnn
}  // namespace smx
