// Dense (MLP) GEMMs on the warp-specialised tcgen05 kernel of conv_ws.cuh.
//
//   C_g[m][n] = epi( sum_k A_g(m,k) * B_g(n,k) ),  groups = active slots (GemmArgs, gemm_simt.cuh)
//
// AM / BMODE: 0 -> K-contiguous rows (X[m*ld + k]), 1 -> MN-contiguous (X[k*ld + m]).  M or K may
// be the slot's batch size; one N tile of up to 128 columns per blockIdx.x.  A_EXACT / B_EXACT
// mark an operand that is exact in tf32 (the synthetic data, k/128) so its lo MMA is skipped.
// Epilogues: bias(+ReLU), plain, ReLU mask (dH = (H > 0) ? . : 0), transposed store; SGD = a
// plain-store weight gradient whose tile is applied to the slot's w | m in place (K3+K5 fusion,
// the sgd_update_kernel rule element by element).
#pragma once

#include "conv_ws.cuh"

namespace smx {
namespace dws {

using cnn::ctc::kEpiBias;
using cnn::ctc::kEpiBiasRelu;
using cnn::ctc::kEpiMask;
using cnn::ctc::kEpiPartT;
using cnn::ctc::kEpiStore;

template <int AM_, int BM_, int EPI_, bool AX, bool BX, bool SGD = false>
struct DenseOp {
    using Args = GemmArgs;
    static constexpr int AM = AM_, BMODE = BM_, EPI = EPI_, kMaxN = 128;
    static constexpr bool A_EXACT = AX, B_EXACT = BX, B_IMAGE = false, A_TMA = false, B_TMA = false;
    const CUtensorMap* btmap = nullptr;
    static constexpr int kBoxes = 1, kTmaCi = 1;
    static constexpr bool kInMaskBits = false, kMaskFromBits = false, kSgd = SGD;
    static constexpr int kOnesRow = -1, kPartLd = 0, kSegChunks = SMX_SEG_CHUNKS, kEpiWarps = 4;
    const float* A;
    const float* B;
    float* C;
    const float* bias;
    const float* mask;
    int lda, ldb, ldc, ldmask;
    int M, N, K, kbeg, m0, split, n0;
    long long m_off;
    SgdRow h;

    __device__ void setup(const GemmArgs& p, int z, int x) {
        const int slot = p.slots[z];
        const int bs = (p.m_is_bs || p.k_is_bs) ? slot_bs(p, slot) : 0;
        M = p.m_is_bs ? bs : p.M;
        K = p.k_is_bs ? bs : p.K;
        n0 = x * 128;
        N = max(0, min(128, p.N - n0));
        if (N == 0) K = 0;  // no work for this N tile
        kbeg = 0;
        split = 0;
        m0 = 0;
        A = opnd_ptr(p.a, slot, p.st, p.n_train_mask);
        B = opnd_ptr(p.b, slot, p.st, p.n_train_mask);
        lda = p.a.ld;
        ldb = p.b.ld;
        C = p.c + p.c_stride * slot;
        ldc = p.ldc;
        bias = (EPI == kEpiBias || EPI == kEpiBiasRelu) ? p.bias + p.bias_stride * slot : nullptr;
        mask = EPI == kEpiMask ? p.mask + p.mask_stride * slot : nullptr;
        ldmask = p.ldmask;
        m_off = p.m_off;
        if (SGD) h = sgd_row(p.hp, p.hp_cap, p.st, slot);
    }

    // ---- A, K-contiguous: row pointer once per tile, k per chunk
    struct RowInfo {
        const float* ptr;  // A row (nullptr: row >= M); MN mode: first row of the quad
        int row;
    };
    struct TapInfo {
        int k;
    };
    __device__ __forceinline__ RowInfo row_info(int m) const {
        if (AM == 0) return RowInfo{m < M ? A + (long long)m * lda : nullptr, m};
        return RowInfo{m < M ? A + m : nullptr, m};
    }
    __device__ __forceinline__ TapInfo tap_info(int k) const { return TapInfo{k < K ? k : -1}; }
    __device__ __forceinline__ const float* a_ptr_tap(const RowInfo& r, const TapInfo& t) const {
        return (r.ptr && t.k >= 0) ? r.ptr + t.k : nullptr;
    }
    // ---- A, MN-contiguous: 4 consecutive rows at reduction index k
    struct RedInfo {
        int k;
    };
    __device__ __forceinline__ RedInfo red_info(int k) const { return RedInfo{k}; }
    __device__ __forceinline__ const float* a_ptr_red(const RowInfo& r, const RedInfo& d) const {
        return a_ptr_red_step(r, d, 0);
    }
    __device__ __forceinline__ const float* a_ptr_red_step(const RowInfo& r, const RedInfo& d, int j) const {
        return (r.ptr && d.k + j < K) ? r.ptr + (long long)(d.k + j) * lda : nullptr;
    }
    // ---- B (register path): BMODE 0 -> 4 consecutive k of row n; BMODE 1 -> rows n..n+3 at k
    __device__ __forceinline__ const float* b_ptr(int n, int k) const {
        if (BMODE == 0) return B + (long long)(n0 + n) * ldb + k;
        return B + (long long)k * ldb + n0 + n;
    }
    __device__ __forceinline__ const float* b_image(int) const { return nullptr; }

    // ---- epilogue targets
    __device__ __forceinline__ float4 bias4(int col) const {
        return __ldg(reinterpret_cast<const float4*>(bias + n0 + col));
    }
    __device__ __forceinline__ void store4(int m, int col, float4 x) const {
        float* c = C + (long long)m * ldc + n0 + col;
        if constexpr (SGD) {
            static_assert(EPI == kEpiStore, "the SGD epilogue consumes a plain gradient tile");
            const float v[4] = {x.x, x.y, x.z, x.w};
            if ((ldc & 3) == 0 && col + 4 <= N) {
                float4 wv = *reinterpret_cast<float4*>(c), mv = *reinterpret_cast<float4*>(c + m_off);
                float* wp = &wv.x;
                float* mp = &mv.x;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    mp[j] = __fmaf_rn(h.mu, mp[j], __fmaf_rn(h.wd, wp[j], v[j]));
                    wp[j] = __fmaf_rn(h.nlr, mp[j], wp[j]);
                }
                *reinterpret_cast<float4*>(c) = wv;
                *reinterpret_cast<float4*>(c + m_off) = mv;
            } else {
                for (int j = 0; j < 4 && col + j < N; ++j) sgd_apply(c, c + m_off, j, v[j], h);
            }
            return;
        }
        if ((ldc & 3) == 0 && n0 + col + 4 <= n0 + N) {
            *reinterpret_cast<float4*>(c) = x;
        } else {
            const float v[4] = {x.x, x.y, x.z, x.w};
            for (int j = 0; j < 4 && col + j < N; ++j) c[j] = v[j];
        }
    }
    __device__ __forceinline__ const void* mask_at(int m, int col) const { return mask + (long long)m * ldmask + n0 + col; }
    // SGD epilogue: the parameter at (m, col) of the tile (w; its momentum at + m_off)
    __device__ __forceinline__ float* w_at(int m, int col) const { return C + (long long)m * ldc + n0 + col; }
    __device__ __forceinline__ void sgd4(float4& w, float4& m, float4 g) const {
        m.x = __fmaf_rn(h.mu, m.x, __fmaf_rn(h.wd, w.x, g.x));
        m.y = __fmaf_rn(h.mu, m.y, __fmaf_rn(h.wd, w.y, g.y));
        m.z = __fmaf_rn(h.mu, m.z, __fmaf_rn(h.wd, w.z, g.z));
        m.w = __fmaf_rn(h.mu, m.w, __fmaf_rn(h.wd, w.w, g.w));
        w.x = __fmaf_rn(h.nlr, m.x, w.x);
        w.y = __fmaf_rn(h.nlr, m.y, w.y);
        w.z = __fmaf_rn(h.nlr, m.z, w.z);
        w.w = __fmaf_rn(h.nlr, m.w, w.w);
    }
    __device__ __forceinline__ long long mask_off(int m, int col) const {
        return (long long)m * ldmask + n0 + col;
    }
    __device__ __forceinline__ float4 mask4(long long off) const {
        return __ldg(reinterpret_cast<const float4*>(mask + off));
    }
    __device__ __forceinline__ void store_masked(int m, int col, long long, float4 x) const { store4(m, col, x); }
    __device__ __forceinline__ float* ct_at(int col, int m) const { return C + (long long)(n0 + col) * ldc + m; }
};

}  // namespace dws
}  // namespace smx
