// smx.cu — the B200 stage executor behind include/smx.h.
//
// One smx_ctx owns one GPU: the slot slab (w | m per slot), the gradient slab, the checkpoint
// pool (w | m per entry), the per-slot hp table and loss history, the synthetic dataset and
// the activation scratch.  A lockstep trains every active slot by one step with one launch
// per kernel class (grouped over slots); smx_train replays the lockstep sequence through a
// CUDA graph keyed by the active slot set.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (through cudaGetDriverEntryPoint: no -lcuda)

#include <algorithm>
#include <cmath>
#include <functional>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/smx.h"
#include "kernels/common.cuh"
#include "kernels/gemm_simt.cuh"
#include "kernels/gemm_tc.cuh"
#include "kernels/step_kernels.cuh"
#include "kernels/cnn.cuh"
#include "kernels/conv_ws.cuh"
#include "kernels/dense_ws.cuh"
#include "kernels/wgrad2_at.cuh"
#include "kernels/conv1_tc.cuh"

using namespace smx;

namespace {

thread_local std::string g_err;

struct SmxError {
    int code;
    std::string what;
};

[[noreturn]] void fail(int code, const std::string& what) { throw SmxError{code, what}; }

void ck(cudaError_t e, const char* where) {
    if (e != cudaSuccess) fail(SMX_EDEVICE, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr int kEvalChunk = 16;  // slots evaluated per eval launch group

}  // namespace

struct smx_ctx {
    smx_model_desc d{};
    int device = 0;
    int num_sms = 148;  // SMs of the device (persistent kernels)
    int S = 0, C = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // second branch of the lockstep (weight gradients)
    cudaStream_t cur = nullptr;   // stream the GEMM / reduction helpers enqueue on
    cudaEvent_t fj[4] = {};       // fork / join events of the lockstep branches
    cudaEvent_t xev = nullptr;    // cross-context ordering of peer copies (K7)

    float* slab = nullptr;      // S x 2 x PAlloc  (w | m)
    float* grad = nullptr;      // S x PAlloc
    float* pool = nullptr;      // C x 2 x PAlloc  (w | m)
    SlotState* st = nullptr;    // S
    SlotState* ck_st = nullptr; // C
    float* hp = nullptr;        // S x cap x 4
    float* loss = nullptr;      // S x cap
    float* act = nullptr;       // S x act_stride
    float* xtrain = nullptr;    // (n_train + max_batch) x 784
    int* ytrain = nullptr;
    float* xval = nullptr;      // n_val x 784
    int* yval = nullptr;
    float* eval_act = nullptr;  // kEvalChunk x n_val x (256 + 256 + 16)
    float* eval_scratch = nullptr;
    double* eval_out = nullptr;
    int* eval_slots = nullptr;
    std::vector<char> ck_valid;
    std::vector<char> slot_live;  // slot holds a state (init / load / write since open or release)
    // every training / validation input value is exact in tf32 (true for the synthetic k/128
    // data; re-checked on every smx_dataset_upload): only then may the tensor-core GEMMs skip
    // the data operand's lo MMA
    bool data_tf32_exact = true;
    int* flag = nullptr;  // device scratch int

    struct Graph {
        int* d_slots = nullptr;
        cudaGraphExec_t exec = nullptr;
        long long launches = 0;  // kernels in the captured lockstep
    };
    std::map<std::vector<int>, Graph> graphs;
    int* scratch_slots = nullptr;  // for non-graph launches
    bool use_graphs = true;
    bool timing = false;
    smx_stats stats{};
    cudaEvent_t ev[8] = {};

    // model geometry (MLP: common.cuh constants; CNN: cnn.cuh)
    bool cnn = false;
    long long palloc = kPAlloc;      // floats per parameter vector
    long long act_stride = kActStride;
    long long d_in = kD0;            // floats per input sample
    cnn::ActLayout al{};
    float* zval = nullptr;           // CNN eval logits [kEvalChunk][n_val][16]
    CUtensorMap* tmaps = nullptr;    // CNN: [S][cnn::kTmapKinds] TMA maps of the conv A operands

    long long slab_stride() const { return 2 * palloc; }
};

namespace {

void launch_check(smx_ctx* c, const char* what) {
    c->stats.launches += 1;
    ck(cudaGetLastError(), what);
}

StepCtx step_ctx(smx_ctx* c, const int* d_slots) {
    return StepCtx{d_slots, c->st, c->hp, c->d.max_steps};
}

GemmArgs base_args(smx_ctx* c, const int* d_slots) {
    GemmArgs a{};
    a.slots = d_slots;
    a.st = c->st;
    a.hp = c->hp;
    a.hp_cap = c->d.max_steps;
    a.n_train_mask = c->d.n_train - 1;
    return a;
}

// Tensor-core GEMMs of the MLP: the warp-specialised tcgen05 kernel (conv_ws.cuh) with the dense
// Op policy (dense_ws.cuh); a data operand skips its lo MMA only while the context's dataset is
// verified tf32-exact (smx_ctx::data_tf32_exact).
// cudaFuncSetAttribute is per device: one bit per device that has the kernel configured
template <class Op>
void configure_ws(smx_ctx* c) {
    static unsigned long long configured = 0;  // calls on one context come from one thread (smx.h)
    const unsigned long long bit = 1ull << (c->device & 63);
    if (configured & bit) return;
    ck(cudaFuncSetAttribute(cnn::ws::conv_ws_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            cnn::ws::ws_smem<Op>()),
       "conv_ws smem attribute");
    configured |= bit;
}

template <class Op>
void dense_ws_launch(smx_ctx* c, const GemmArgs& a, int groups, int m_max) {
    configure_ws<Op>(c);
    const int mtiles = (m_max + tc3::kBM - 1) / tc3::kBM;
    dim3 grid((a.N + 127) / 128, mtiles, groups);
    cnn::ws::conv_ws_kernel<Op><<<grid, cnn::ws::WsPlan<Op>::Threads, cnn::ws::ws_smem<Op>(), c->cur>>>(a, 1);
    launch_check(c, "dense_ws");
}

template <int AM, int BMODE, int EPI>
void tc_launch(smx_ctx* c, const GemmArgs& a, int groups, int m_max) {
    if ((a.a.ld & 3) || (a.b.ld & 3))
        fail(SMX_ECONFIG, "tensor-core GEMM needs 16-byte aligned operand rows (ld % 4 == 0)");
    constexpr int wepi = EPI == tc::kTcStore ? dws::kEpiStore : EPI == tc::kTcBiasRelu ? dws::kEpiBiasRelu
                         : EPI == tc::kTcBias ? dws::kEpiBias : EPI == tc::kTcMask ? dws::kEpiMask : dws::kEpiPartT;
    if constexpr (AM == 0 && BMODE == 0 && EPI == tc::kTcBiasRelu) {
        if (a.a.from_data && c->data_tf32_exact) return dense_ws_launch<dws::DenseOp<AM, BMODE, wepi, true, false>>(c, a, groups, m_max);
    }
    if constexpr (AM == 1 && BMODE == 1 && EPI == tc::kTcStore) {
        if (a.m_off) {  // layer-1 weight gradient with the K5 update fused into its epilogue
            if (a.b.from_data && c->data_tf32_exact)
                return dense_ws_launch<dws::DenseOp<AM, BMODE, wepi, false, true, true>>(c, a, groups, m_max);
            return dense_ws_launch<dws::DenseOp<AM, BMODE, wepi, false, false, true>>(c, a, groups, m_max);
        }
        if (a.b.from_data && c->data_tf32_exact) return dense_ws_launch<dws::DenseOp<AM, BMODE, wepi, false, true>>(c, a, groups, m_max);
    }
    dense_ws_launch<dws::DenseOp<AM, BMODE, wepi, false, false>>(c, a, groups, m_max);
}

template <int AM, int BMODE, int EPI>
void gemm(smx_ctx* c, const GemmArgs& a, int groups, int m_max) {
    if (c->d.gemm_mode == SMX_GEMM_TC) {
        constexpr int tepi = EPI == kEpiStore ? tc::kTcStore : EPI == kEpiBiasRelu ? tc::kTcBiasRelu
                             : EPI == kEpiBias ? tc::kTcBias : tc::kTcMask;
        tc_launch<AM, BMODE, tepi>(c, a, groups, m_max);
        return;
    }
    dim3 grid((a.N + kTN - 1) / kTN, (m_max + kTM - 1) / kTM, groups);
    gemm_simt_kernel<AM, BMODE, EPI><<<grid, 256, 0, c->cur>>>(a);
    launch_check(c, "gemm_simt");
}

// Bias gradient of one layer: db[n] = sum over the batch of dY[r][n].
void colsum(smx_ctx* c, const StepCtx& sc, int groups, long long dy_off, int ld, int N, long long db_off) {
    if (c->d.gemm_mode == SMX_GEMM_TC)
        colsum_fast_kernel<<<dim3((N + 31) / 32, groups), 256, 0, c->cur>>>(sc, c->act, kActStride, dy_off, ld, N,
                                                                             c->grad, kPAlloc, db_off);
    else
        colsum_kernel<<<dim3((N + 127) / 128, groups), 128, 0, c->cur>>>(sc, c->act, kActStride, dy_off, ld, N,
                                                                             c->grad, kPAlloc, db_off);
    launch_check(c, "colsum");
}

// ---- CNN (SMX_MODEL_CNN) -------------------------------------------------------------
// TMA maps of the tensor-core convolutions' A operands (cnn.cuh kTm*), one set per slot: NHWC
// fp32 tensors of max_batch samples, dims innermost first (channel, column, row, sample), boxes of
// 4096 floats (16 KB = one raw A tile), 128-byte swizzle, zero fill out of bounds.
void make_conv_tmaps(smx_ctx* c) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q{};
    ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q),
       "cuTensorMapEncodeTiled entry point");
    if (!enc || q != cudaDriverEntryPointSuccess) fail(SMX_EDEVICE, "cuTensorMapEncodeTiled unavailable");
    struct Spec {
        long long off;
        int C, W, H, n_box, w_box, h_box, stride;  // box: 32 (conv2 / conv3 A tiles) or C channels x w_box x h_box x n_box
    };
    const long long mb = c->d.max_batch;
    const Spec specs[cnn::kTmWgB2] = {
        {c->al.a1, 32, 32, 32, 1, 16, 8, 2},   // conv2 forward: a1, output tile = 8 rows x 16 columns
        {c->al.a2, 64, 16, 16, 2, 8, 8, 2},    // conv3 forward: a2, 2 samples x 8 x 8
        {c->al.d2, 64, 16, 16, 1, 17, 9, 1},   // conv2 input gradient: d2, 8 x 16 blocks + their (1, 1) neighbours
        {c->al.d3, 128, 8, 8, 2, 8, 8, 1},     // conv3 input gradient: d3, 2 samples x 8 x 8 blocks
        {c->al.a1, 32, 32, 32, 1, 33, 5, 1},   // conv2 weight gradient: a1 window of 32 output pixels (2 x 16), all taps
        {c->al.a2, 64, 16, 16, 1, 8, 4, 2},    // conv3 weight gradient: a2, 32 output pixels (4 x 8) per tap
    };
    std::vector<CUtensorMap> h((size_t)c->S * cnn::kTmapKinds);
    for (int s = 0; s < c->S; ++s)
        for (int k = 0; k < cnn::kTmWgB2; ++k) {
            const Spec& sp = specs[k];
            float* base = c->act + c->act_stride * s + sp.off;
            const cuuint64_t dims[4] = {(cuuint64_t)sp.C, (cuuint64_t)sp.W, (cuuint64_t)sp.H, (cuuint64_t)mb};
            const cuuint64_t strides[3] = {(cuuint64_t)sp.C * 4, (cuuint64_t)sp.W * sp.C * 4,
                                           (cuuint64_t)sp.H * sp.W * sp.C * 4};
            const bool wg = k >= cnn::kTmWg2;  // weight-gradient boxes take every channel of a tap
            const cuuint32_t box[4] = {(cuuint32_t)(wg ? sp.C : 32), (cuuint32_t)(sp.w_box * sp.stride),
                                       (cuuint32_t)(sp.h_box * sp.stride), (cuuint32_t)sp.n_box};
            const cuuint32_t es[4] = {1, (cuuint32_t)sp.stride, (cuuint32_t)sp.stride, 1};
            const CUresult r = enc(&h[(size_t)s * cnn::kTmapKinds + k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims,
                                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   wg ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) fail(SMX_EDEVICE, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        }
    // the weight gradients' B operands: d2 / d3 as 2-D [max_batch x pixels][Co] tensors, boxes of
    // 32 channels (128 bytes) x 32 reduction rows with the 128-byte / 32-byte-atom swizzle (the
    // UMMA MN-major tf32 layout SWIZZLE_128B_BASE32B)
    for (int s = 0; s < c->S; ++s)
        for (int L = 2; L <= 3; ++L) {
            const int C = L == 2 ? 64 : 128, pix = L == 2 ? 256 : 64;
            float* base = c->act + c->act_stride * s + (L == 2 ? c->al.d2 : c->al.d3);
            const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)(mb * pix)};
            const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
            const cuuint32_t box[2] = {32, 32};
            const cuuint32_t es[2] = {1, 1};
            const int k = L == 2 ? cnn::kTmWgB2 : cnn::kTmWgB3;
            const CUresult r = enc(&h[(size_t)s * cnn::kTmapKinds + k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims,
                                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) fail(SMX_EDEVICE, "cuTensorMapEncodeTiled (B) failed (" + std::to_string((int)r) + ")");
        }
    // the conv1 forward's output a1 as [max_batch x 1024 pixels][32], one image row per box
    for (int s = 0; s < c->S; ++s) {
        float* base = c->act + c->act_stride * s + c->al.a1;
        const cuuint64_t dims[2] = {32, (cuuint64_t)(mb * 1024)};
        const cuuint64_t strides[1] = {32 * 4};
        const cuuint32_t box[2] = {32, 32};
        const cuuint32_t es[2] = {1, 1};
        const CUresult r = enc(&h[(size_t)s * cnn::kTmapKinds + cnn::kTmA1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base,
                               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(SMX_EDEVICE, "cuTensorMapEncodeTiled (a1) failed (" + std::to_string((int)r) + ")");
    }
    // the conv2 input gradient's output d1 as {32 channels, 32 columns, max_batch x 32 rows}: one
    // box = the 16 input rows of one M tile (64 KB)
    for (int s = 0; s < c->S; ++s) {
        float* base = c->act + c->act_stride * s + c->al.d1;
        const cuuint64_t dims[3] = {32, 32, (cuuint64_t)(mb * 32)};
        const cuuint64_t strides[2] = {32 * 4, 32 * 32 * 4};
        const cuuint32_t box[3] = {32, 32, 16};
        const cuuint32_t es[3] = {1, 1, 1};
        const CUresult r = enc(&h[(size_t)s * cnn::kTmapKinds + cnn::kTmD1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base,
                               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(SMX_EDEVICE, "cuTensorMapEncodeTiled (d1) failed (" + std::to_string((int)r) + ")");
    }
    // the conv3 input gradient's output d2 as {64 channels, 16 columns, 2 row parities, 8 row
    // pairs, max_batch}: one box = 32 channels of one parity row set of two samples (32 KB)
    for (int s = 0; s < c->S; ++s) {
        float* base = c->act + c->act_stride * s + c->al.d2;
        const cuuint64_t dims[5] = {64, 16, 2, 8, (cuuint64_t)mb};
        const cuuint64_t strides[4] = {64 * 4, 16 * 64 * 4, 2 * 16 * 64 * 4, 16 * 16 * 64 * 4};
        const cuuint32_t box[5] = {32, 16, 1, 8, 2};
        const cuuint32_t es[5] = {1, 1, 1, 1, 1};
        const CUresult r = enc(&h[(size_t)s * cnn::kTmapKinds + cnn::kTmD2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, base,
                               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(SMX_EDEVICE, "cuTensorMapEncodeTiled (d2) failed (" + std::to_string((int)r) + ")");
    }
    ck(cudaMalloc(&c->tmaps, sizeof(CUtensorMap) * h.size()), "tensor maps");
    ck(cudaMemcpy(c->tmaps, h.data(), sizeof(CUtensorMap) * h.size(), cudaMemcpyHostToDevice), "tensor maps H2D");
}

cnn::ConvArgs cnn_args(smx_ctx* c, const int* d_slots) {
    cnn::ConvArgs a{};
    a.slots = d_slots;
    a.st = c->st;
    a.hp = c->hp;
    a.hp_cap = c->d.max_steps;
    a.n_train_mask = c->d.n_train - 1;
    a.x = c->xtrain;
    a.x_from_slot = 1;
    a.slab = c->slab;
    a.slab_stride = c->slab_stride();
    a.act = c->act;
    a.al = c->al;
    a.grad = c->grad;
    a.grad_stride = c->palloc;
    a.labels = c->ytrain;
    a.loss_hist = c->loss;
    a.tmaps = c->tmaps;
    a.fuse_update = c->d.gemm_mode == SMX_GEMM_TC ? 1 : 0;
    a.pooled = c->d.gemm_mode == SMX_GEMM_TC ? 1 : 0;
    return a;
}

#ifndef SMX_TPC_FILL
#define SMX_TPC_FILL 1.5  // per-CTA pipeline fill / drain in tiles (conv_tc grid choice; profiles/debug/r2s3_tpc.sh)
#endif
#ifndef SMX_TPC_FWD3
#define SMX_TPC_FWD3 16
#endif
#ifndef SMX_TPC_DGR3
#define SMX_TPC_DGR3 16
#endif
// tiles per CTA of each tensor-core conv (amortises the CTA prologue over several M tiles)
template <class Op>
constexpr int conv_tpc() {
    return 1;
}
template <>
constexpr int conv_tpc<cnn::ctc::Fwd<1>>() { return 8; }
template <>
constexpr int conv_tpc<cnn::ctc::Fwd<2>>() { return 16; }
template <>
constexpr int conv_tpc<cnn::ctc::Fwd<3>>() { return SMX_TPC_FWD3; }
template <>
constexpr int conv_tpc<cnn::ctc::Dgrad<2>>() { return 16; }
template <>
constexpr int conv_tpc<cnn::ctc::Dgrad<3>>() { return SMX_TPC_DGR3; }

template <class Op>
void conv_tc(smx_ctx* c, const cnn::ConvArgs& a, int gx, int m_max, int groups) {
    configure_ws<Op>(c);
    // tiles per CTA (one CTA per SM at a time): the count <= the Op's maximum that minimises
    // waves x (tiles + per-CTA fill / drain ~1.5 tiles), so that the last wave is not a short one
    // at any slot count (e.g. 10 slots of the conv2 input gradient: 8 tiles per CTA = 2.2 waves,
    // 6 = 2.9).  It changes only the work split, never the arithmetic.
    const int mtiles = (m_max + tc3::kBM - 1) / tc3::kBM;
    int tpc = 1;
    double best = 1e30;
    for (int t = conv_tpc<Op>(); t >= 1; --t) {
        const long long ctas = (long long)gx * ((mtiles + t - 1) / t) * groups;
        const double cost = (double)((ctas + c->num_sms - 1) / c->num_sms) * (t + SMX_TPC_FILL);
        if (cost < best - 1e-9) {
            best = cost;
            tpc = t;
        }
    }
    dim3 grid(gx, (mtiles + tpc - 1) / tpc, groups);
    cnn::ws::conv_ws_kernel<Op><<<grid, cnn::ws::WsPlan<Op>::Threads, cnn::ws::ws_smem<Op>(), c->cur>>>(a, tpc);
    launch_check(c, "conv_ws");
}

// conv2 weight gradient, all taps per CTA (kernels/wgrad2_at.cuh): one CTA per (2048-pixel split, slot)
void wgrad2_at(smx_ctx* c, const cnn::ConvArgs& a, int splits, int groups) {
    static unsigned long long configured = 0;
    const unsigned long long bit = 1ull << (c->device & 63);
    if (!(configured & bit)) {
        ck(cudaFuncSetAttribute(cnn::wg2::wgrad2_at_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cnn::wg2::kSmem),
           "wgrad2_at smem attribute");
        configured |= bit;
    }
    const int items = splits * groups;
    cnn::wg2::wgrad2_at_kernel<<<std::min(items, c->num_sms), cnn::wg2::kThreads, cnn::wg2::kSmem, c->cur>>>(
        a, splits, items);
    launch_check(c, "wgrad2_at");
}

// conv1 weight gradient on the tensor cores (kernels/conv1_tc.cuh): persistent grid, one CTA per
// SM, one work item per (slot, group of kImgs samples) -> one partial row each
void conv1_wgrad_tc(smx_ctx* c, const cnn::ConvArgs& a, int mb, int groups) {
    namespace c1 = cnn::c1;
    static unsigned long long configured = 0;
    const unsigned long long bit = 1ull << (c->device & 63);
    if (!(configured & bit)) {
        ck(cudaFuncSetAttribute(c1::conv1_wgrad_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1::kSmem),
           "conv1_wgrad_tc smem attribute");
        ck(cudaFuncSetAttribute(c1::conv1_wgrad_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1::kSmem),
           "conv1_wgrad_tc smem attribute");
        configured |= bit;
    }
    const int parts = (mb + c1::kImgs - 1) / c1::kImgs, items = parts * groups;
    const int grid = std::min(items, c->num_sms);  // one CTA per SM (all 512 TMEM columns)
    if (c->data_tf32_exact)
        c1::conv1_wgrad_tc_kernel<true><<<grid, c1::kThreads, c1::kSmem, c->cur>>>(a, parts, items);
    else
        c1::conv1_wgrad_tc_kernel<false><<<grid, c1::kThreads, c1::kSmem, c->cur>>>(a, parts, items);
    launch_check(c, "conv1_wgrad_tc");
}

// conv1 forward on the tensor cores (kernels/conv1_tc.cuh, namespace f1): 2 CTAs per SM, items
// (slot, sample) in contiguous per-CTA ranges
void conv1_fwd_tc(smx_ctx* c, const cnn::ConvArgs& a, int mb, int groups) {
    namespace f1 = cnn::c1::f1;
    static unsigned long long configured = 0;
    const unsigned long long bit = 1ull << (c->device & 63);
    if (!(configured & bit)) {
        ck(cudaFuncSetAttribute(f1::conv1_fwd_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, f1::kSmem),
           "conv1_fwd_tc smem attribute");
        ck(cudaFuncSetAttribute(f1::conv1_fwd_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, f1::kSmem),
           "conv1_fwd_tc smem attribute");
        configured |= bit;
    }
    const int items = mb * groups;
    const int grid = std::min(items, 2 * c->num_sms);
    if (c->data_tf32_exact)
        f1::conv1_fwd_tc_kernel<true><<<grid, f1::kThreads, f1::kSmem, c->cur>>>(a, mb, items);
    else
        f1::conv1_fwd_tc_kernel<false><<<grid, f1::kThreads, f1::kSmem, c->cur>>>(a, mb, items);
    launch_check(c, "conv1_fwd_tc");
}

template <int L>
void conv_forward(smx_ctx* c, const cnn::ConvArgs& a, int n, int mb) {
    using G = cnn::Geo<L>;
    if (c->d.gemm_mode == SMX_GEMM_TC && L == 1) {
        conv1_fwd_tc(c, a, mb, n);
        return;
    }
    if (c->d.gemm_mode == SMX_GEMM_TC) {
        conv_tc<cnn::ctc::Fwd<L>>(c, a, 1, mb * G::OH * G::OH, n);
        return;
    }
    const long long total = (long long)mb * G::OH * G::OH * G::Co;
    cnn::conv_fwd_simt<L><<<dim3((unsigned)std::min<long long>((total + 255) / 256, 1024), n), 256, 0, c->cur>>>(a);
    launch_check(c, "conv_fwd_simt");
}

template <int L>
void conv_wgrad(smx_ctx* c, const cnn::ConvArgs& a, int n, int mb) {
    using G = cnn::Geo<L>;
    if (c->d.gemm_mode == SMX_GEMM_TC && L == 1) {
        conv1_wgrad_tc(c, a, mb, n);
        cnn::conv1_wgrad_reduce<<<dim3((cnn::kL1Outs + 127) / 128, n), 128, 0, c->cur>>>(a, cnn::c1::kImgs);
        launch_check(c, "conv1_wgrad_reduce");
        return;
    }
    if (c->d.gemm_mode == SMX_GEMM_TC) {
        const int splits = (mb * G::OH * G::OH + cnn::kSplitRows - 1) / cnn::kSplitRows;
        if constexpr (L == 2)
            wgrad2_at(c, a, splits, n);
        else
            conv_tc<cnn::ctc::Wgrad<L>>(c, a, splits, cnn::Part<L>::Rows, n);
        const int fc = (L == 3 && a.fuse_update) ? cnn::kFcBlocks : 0;  // + the FC layer's update
        cnn::wgrad_reduce_kernel<L><<<dim3(G::Co + fc, n), 128, 0, c->cur>>>(a);
        launch_check(c, "wgrad_reduce");
        return;
    }
    cnn::conv_wgrad_simt<L><<<dim3((G::Co * 9 * G::Ci + G::Co + 127) / 128, n), 128, 0, c->cur>>>(a);
    launch_check(c, "conv_wgrad_simt");
}

template <int L>
void conv_dgrad(smx_ctx* c, const cnn::ConvArgs& a, int n, int mb) {
    using G = cnn::Geo<L>;
    if (c->d.gemm_mode == SMX_GEMM_TC) {
        conv_tc<cnn::ctc::Dgrad<L>>(c, a, cnn::WImg<L>::DgrN / cnn::WImg<L>::DgrNTile, mb * (G::H / 2) * (G::H / 2), n);
        return;
    }
    const long long total = (long long)mb * G::H * G::H * G::Ci;
    cnn::conv_dgrad_simt<L><<<dim3((unsigned)std::min<long long>((total + 255) / 256, 1024), n), 256, 0, c->cur>>>(a);
    launch_check(c, "conv_dgrad_simt");
}

// Pre-split tf32 hi/lo weight images of the three convs (tensor-core mode), see cnn::WImg.
void weight_images(smx_ctx* c, const cnn::ConvArgs& a, int n) {
    if (c->d.gemm_mode != SMX_GEMM_TC) return;
    cnn::weight_image_kernel<<<dim3(cnn::kWImgBlocks1 + cnn::kWImgBlocks2 + cnn::kWImgBlocks3, n), 256, 0, c->cur>>>(a);
    launch_check(c, "weight_image");
}

// One lockstep of the CNN over `n` slots: forward, head, backward as two branches (input
// gradients on the main stream, weight gradients on the side stream), K5 update, advance.
void enqueue_lockstep_cnn(smx_ctx* c, const int* d_slots, int n) {
    const int mb = c->d.max_batch;
    const cnn::ConvArgs a = cnn_args(c, d_slots);
    StepCtx sc = step_ctx(c, d_slots);
    c->cur = c->stream;
    weight_images(c, a, n);
    conv_forward<1>(c, a, n, mb);
    conv_forward<2>(c, a, n, mb);
    conv_forward<3>(c, a, n, mb);
    cnn::head_fwd_kernel<<<dim3(mb, n), 128, 0, c->stream>>>(a);  // + dA3 (the pool / ReLU backward)
    launch_check(c, "head_fwd");
    auto fork = [&](int i) {
        ck(cudaEventRecord(c->fj[i], c->stream), "fork record");
        ck(cudaStreamWaitEvent(c->side, c->fj[i], 0), "fork wait");
    };
    fork(0);
    c->cur = c->side;
    // FC gradients + the step's loss: only the conv3 weight-gradient reduction (the FC update) reads them
    cnn::head_grad_kernel<<<dim3((cnn::kNCP * cnn::kFeat + cnn::kNCP + 127) / 128, n), 128, 0, c->side>>>(a);
    launch_check(c, "head_grad");
    conv_wgrad<3>(c, a, n, mb);
    c->cur = c->stream;
    conv_dgrad<3>(c, a, n, mb);
    fork(1);
    c->cur = c->side;
    conv_wgrad<2>(c, a, n, mb);
    c->cur = c->stream;
    conv_dgrad<2>(c, a, n, mb);
    fork(2);
    c->cur = c->side;
    conv_wgrad<1>(c, a, n, mb);
    ck(cudaEventRecord(c->fj[3], c->side), "join record");
    ck(cudaStreamWaitEvent(c->stream, c->fj[3], 0), "join wait");
    c->cur = c->stream;
    if (c->d.gemm_mode == SMX_GEMM_TC && c->timing) {  // fused: no separate update interval
        cudaEventRecord(c->ev[2], c->stream);
        cudaEventRecord(c->ev[3], c->stream);
    }
    if (c->d.gemm_mode != SMX_GEMM_TC) {  // tensor-core mode: K5 fused into the reductions
        if (c->timing) cudaEventRecord(c->ev[2], c->stream);
        const long long n4 = c->palloc / 4;
        const int bx = (int)((n4 + 256 * 4 - 1) / (256 * 4));
        sgd_update_kernel<<<dim3(bx, n), 256, 0, c->stream>>>(sc, c->slab, c->slab_stride(), c->grad, c->palloc, n4);
        launch_check(c, "sgd_update");
        if (c->timing) cudaEventRecord(c->ev[3], c->stream);
    }
    advance_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(sc, n);
    launch_check(c, "advance");
}

// Validation metrics of k slots (device list eval_slots): forward in chunks of max_batch
// samples through the slots' own activation buffers, logits to zval, then the shared
// fixed-order reduction (eval_reduce_kernel).
void eval_cnn(smx_ctx* c, int k) {
    const int mb = c->d.max_batch, nv = c->d.n_val;
    cnn::ConvArgs a = cnn_args(c, c->eval_slots);
    a.x = c->xval;
    a.x_from_slot = 0;
    a.fixed_bs = mb;
    a.labels = c->yval;
    a.zout = c->zval;
    a.z_stride = (long long)nv * cnn::kNCP;
    c->cur = c->stream;
    weight_images(c, a, k);
    for (int r0 = 0; r0 < nv; r0 += mb) {
        a.x_row0 = r0;
        conv_forward<1>(c, a, k, mb);
        conv_forward<2>(c, a, k, mb);
        conv_forward<3>(c, a, k, mb);
        cnn::head_fwd_kernel<<<dim3(mb, k), 128, 0, c->stream>>>(a);
        launch_check(c, "head_fwd eval");
    }
    eval_reduce_kernel<<<k, 256, 0, c->stream>>>(c->eval_slots, c->zval, a.z_stride, c->yval, nv, c->eval_scratch,
                                                 c->eval_out);
    launch_check(c, "eval_reduce");
}

// One lockstep of the MLP over `n` slots listed in device array d_slots.
void enqueue_lockstep(smx_ctx* c, const int* d_slots, int n) {
    if (c->cnn) {
        enqueue_lockstep_cnn(c, d_slots, n);
        return;
    }
    const int mb = c->d.max_batch;
    const long long SW = c->slab_stride(), AS = kActStride;
    float* W = c->slab;
    float* G = c->grad;
    float* A = c->act;
    StepCtx sc = step_ctx(c, d_slots);

    {
        // ---- forward
        {
            GemmArgs g = base_args(c, d_slots);
            g.a = Opnd{c->xtrain, 0, kD0, 1};
            g.b = Opnd{W + kOffW1, SW, kD0, 0};
            g.c = A + kActH1; g.c_stride = AS; g.ldc = kH;
            g.bias = W + kOffB1; g.bias_stride = SW;
            g.M = mb; g.m_is_bs = 1; g.N = kH; g.K = kD0;
            gemm<0, 0, kEpiBiasRelu>(c, g, n, mb);
        }
        {
            GemmArgs g = base_args(c, d_slots);
            g.a = Opnd{A + kActH1, AS, kH, 0};
            g.b = Opnd{W + kOffW2, SW, kH, 0};
            g.c = A + kActH2; g.c_stride = AS; g.ldc = kH;
            g.bias = W + kOffB2; g.bias_stride = SW;
            g.M = mb; g.m_is_bs = 1; g.N = kH; g.K = kH;
            gemm<0, 0, kEpiBiasRelu>(c, g, n, mb);
        }
        {
            GemmArgs g = base_args(c, d_slots);
            g.a = Opnd{A + kActH2, AS, kH, 0};
            g.b = Opnd{W + kOffW3, SW, kH, 0};
            g.c = A + kActZ; g.c_stride = AS; g.ldc = kCP;
            g.bias = W + kOffB3; g.bias_stride = SW;
            g.M = mb; g.m_is_bs = 1; g.N = kCP; g.K = kH;
            gemm<0, 0, kEpiBias>(c, g, n, mb);
        }
        // ---- loss
        loss_train_kernel<<<n, kMaxBatch, 0, c->stream>>>(sc, c->ytrain, c->d.n_train - 1, A, AS, c->loss);
        launch_check(c, "loss_train");
        // The backward pass runs as two branches: input gradients (dgrad) on the main stream,
        // weight / bias gradients on the side stream as soon as their inputs exist.
        auto fork = [&](int i) {
            ck(cudaEventRecord(c->fj[i], c->stream), "fork record");
            ck(cudaStreamWaitEvent(c->side, c->fj[i], 0), "fork wait");
        };
        // ---- layer 3 grads
        fork(0);
        c->cur = c->side;
        if (c->d.gemm_mode == SMX_GEMM_TC) {
            GemmArgs g = base_args(c, d_slots);  // gW3^T[k][c] = sum_r H2[r][k] dZ[r][c], stored transposed
            g.a = Opnd{A + kActH2, AS, kH, 0};
            g.b = Opnd{A + kActDZ, AS, kCP, 0};
            g.c = G + kOffW3; g.c_stride = kPAlloc; g.ldc = kH;
            g.M = kH; g.N = kCP; g.K = mb; g.k_is_bs = 1;
            tc_launch<1, 1, tc::kTcStoreT>(c, g, n, kH);
        } else {
            GemmArgs g = base_args(c, d_slots);  // gW3[c][k] = sum_r dZ[r][c] H2[r][k]
            g.a = Opnd{A + kActDZ, AS, kCP, 0};
            g.b = Opnd{A + kActH2, AS, kH, 0};
            g.c = G + kOffW3; g.c_stride = kPAlloc; g.ldc = kH;
            g.M = kCP; g.N = kH; g.K = mb; g.k_is_bs = 1;
            gemm<1, 1, kEpiStore>(c, g, n, kCP);
        }
        colsum(c, sc, n, kActDZ, kCP, kCP, kOffB3);
        c->cur = c->stream;
        {
            GemmArgs g = base_args(c, d_slots);  // dH2[r][k] = (H2>0) sum_c dZ[r][c] W3[c][k]
            g.a = Opnd{A + kActDZ, AS, kCP, 0};
            g.b = Opnd{W + kOffW3, SW, kH, 0};
            g.c = A + kActDH2; g.c_stride = AS; g.ldc = kH;
            g.mask = A + kActH2; g.mask_stride = AS; g.ldmask = kH;
            g.M = mb; g.m_is_bs = 1; g.N = kH; g.K = kCP;
            gemm<0, 1, kEpiMask>(c, g, n, mb);
        }
        // ---- layer 2 grads
        fork(1);
        c->cur = c->side;
        {
            GemmArgs g = base_args(c, d_slots);
            g.a = Opnd{A + kActDH2, AS, kH, 0};
            g.b = Opnd{A + kActH1, AS, kH, 0};
            g.c = G + kOffW2; g.c_stride = kPAlloc; g.ldc = kH;
            g.M = kH; g.N = kH; g.K = mb; g.k_is_bs = 1;
            gemm<1, 1, kEpiStore>(c, g, n, kH);
        }
        colsum(c, sc, n, kActDH2, kH, kH, kOffB2);
        c->cur = c->stream;
        {
            GemmArgs g = base_args(c, d_slots);
            g.a = Opnd{A + kActDH2, AS, kH, 0};
            g.b = Opnd{W + kOffW2, SW, kH, 0};
            g.c = A + kActDH1; g.c_stride = AS; g.ldc = kH;
            g.mask = A + kActH1; g.mask_stride = AS; g.ldmask = kH;
            g.M = mb; g.m_is_bs = 1; g.N = kH; g.K = kH;
            gemm<0, 1, kEpiMask>(c, g, n, mb);
        }
        // ---- layer 1 grads
        fork(2);
        c->cur = c->side;
        const bool fused = c->d.gemm_mode == SMX_GEMM_TC;
        {
            GemmArgs g = base_args(c, d_slots);
            g.a = Opnd{A + kActDH1, AS, kH, 0};
            g.b = Opnd{c->xtrain, 0, kD0, 1};
            g.M = kH; g.N = kD0; g.K = mb; g.k_is_bs = 1;
            if (fused) {  // K3+K5: the epilogue updates W1 in place (tensor-core mode)
                g.c = W + kOffW1; g.c_stride = SW; g.ldc = kD0; g.m_off = kPAlloc;
            } else {
                g.c = G + kOffW1; g.c_stride = kPAlloc; g.ldc = kD0;
            }
            gemm<1, 1, kEpiStore>(c, g, n, kH);
        }
        if (c->timing) cudaEventRecord(c->ev[2], c->cur);
        if (fused) {
            // b1 with its update fused, then W2 b2 W3 b3 from the gradient slab: the input-gradient
            // GEMMs (their only readers after the forward) finished before fork(2)
            const int nb = (kH + 31) / 32;
            colsum_sgd_kernel<<<dim3(nb + 64, n), 256, 0, c->side>>>(sc, c->act, kActStride, kActDH1, kH, kH, W, SW, G,
                                                                     kPAlloc, kOffB1, nb, kOffW2, kPEnd);
            launch_check(c, "colsum_sgd");
        } else {
            colsum(c, sc, n, kActDH1, kH, kH, kOffB1);
        }
        if (c->timing) cudaEventRecord(c->ev[3], c->cur);
        ck(cudaEventRecord(c->fj[3], c->side), "join record");
        ck(cudaStreamWaitEvent(c->stream, c->fj[3], 0), "join wait");
        c->cur = c->stream;
    }
    // ---- K5 update (exact mode; tensor-core mode fused it above) + advance
    if (c->d.gemm_mode != SMX_GEMM_TC) {
        if (c->timing) cudaEventRecord(c->ev[2], c->stream);
        const long long n4 = kPAlloc / 4;
        const int bx = (int)((n4 + 256 * 4 - 1) / (256 * 4));
        sgd_update_kernel<<<dim3(bx, n), 256, 0, c->stream>>>(sc, W, SW, G, kPAlloc, n4);
        launch_check(c, "sgd_update");
        if (c->timing) cudaEventRecord(c->ev[3], c->stream);
    }
    advance_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(sc, n);
    launch_check(c, "advance");
}

void free_graphs(smx_ctx* c) {
    for (auto& [k, g] : c->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.d_slots) cudaFree(g.d_slots);
    }
    c->graphs.clear();
}

smx_ctx::Graph& graph_for(smx_ctx* c, const std::vector<int>& slots) {
    auto it = c->graphs.find(slots);
    if (it != c->graphs.end()) return it->second;
    if (c->graphs.size() >= 256) free_graphs(c);
    smx_ctx::Graph g;
    const int n = (int)slots.size();
    ck(cudaMalloc(&g.d_slots, sizeof(int) * n), "cudaMalloc graph slots");
    ck(cudaMemcpyAsync(g.d_slots, slots.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream),
       "slots H2D");
    cudaGraph_t graph;
    ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    const long long launches = c->stats.launches;
    try {
        enqueue_lockstep(c, g.d_slots, n);
    } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        throw;
    }
    g.launches = c->stats.launches - launches;
    c->stats.launches = launches;
    ck(cudaStreamEndCapture(c->stream, &graph), "end capture");
    ck(cudaGraphInstantiate(&g.exec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    return c->graphs.emplace(slots, g).first->second;
}

void gen_dataset(smx_ctx* c) {
    const long long rows = (long long)c->d.n_train + c->d.max_batch;
    if (c->cnn) {
        cnn::gen_img_kernel<<<1184, 256, 0, c->stream>>>(c->xtrain, rows, c->d.n_train, c->d.seed, 5);
        launch_check(c, "gen_img train");
        cnn::gen_img_labels_kernel<<<296, 128, 0, c->stream>>>(c->xtrain, c->ytrain, rows, c->d.seed);
        launch_check(c, "gen_img_labels train");
        cnn::gen_img_kernel<<<1184, 256, 0, c->stream>>>(c->xval, c->d.n_val, c->d.n_val, c->d.seed, 6);
        launch_check(c, "gen_img val");
        cnn::gen_img_labels_kernel<<<296, 128, 0, c->stream>>>(c->xval, c->yval, c->d.n_val, c->d.seed);
        launch_check(c, "gen_img_labels val");
        return;
    }
    gen_x_kernel<<<1184, 256, 0, c->stream>>>(c->xtrain, rows, c->d.n_train, c->d.seed, kStreamTrain);
    launch_check(c, "gen_x train");
    gen_labels_kernel<<<296, 128, 0, c->stream>>>(c->xtrain, c->ytrain, rows, c->d.seed);
    launch_check(c, "gen_labels train");
    gen_x_kernel<<<1184, 256, 0, c->stream>>>(c->xval, c->d.n_val, c->d.n_val, c->d.seed, kStreamVal);
    launch_check(c, "gen_x val");
    gen_labels_kernel<<<296, 128, 0, c->stream>>>(c->xval, c->yval, c->d.n_val, c->d.seed);
    launch_check(c, "gen_labels val");
}

float init_scale(int fan_in) {
    // bound = sqrt(6 / fan_in) rounded to fp32, then scaled by 2^-23 (exact)
    return (float)std::sqrt(6.0 / (double)fan_in) * (1.0f / 8388608.0f);
}

void check_slot(smx_ctx* c, int slot) {
    if (slot < 0 || slot >= c->S) fail(SMX_ECONFIG, "slot " + std::to_string(slot) + " out of range");
}
void check_ckpt(smx_ctx* c, int ck_) {
    if (ck_ < 0 || ck_ >= c->C) fail(SMX_ECONFIG, "checkpoint " + std::to_string(ck_) + " out of range");
}

// blocks per fork job: every thread moves 4 x 16 B per pass (the kernel's unrolled loop)
unsigned fork_blocks(long long n4) { return (unsigned)std::max<long long>(1, std::min<long long>(148, (n4 + 1023) / 1024)); }

void run_copy(smx_ctx* c, const std::vector<CopyJob>& jobs) {
    if (jobs.empty()) return;
    constexpr int kB = 16;
    const long long n4 = 2 * c->palloc / 4;
    if (c->timing) cudaEventRecord(c->ev[4], c->stream);
    for (std::size_t i0 = 0; i0 < jobs.size(); i0 += kB) {
        const int nj = (int)std::min<std::size_t>(kB, jobs.size() - i0);
        CopyBatch<kB> b{};
        for (int i = 0; i < nj; ++i) b.j[i] = jobs[i0 + i];
        fork_copy_kernel<kB><<<dim3(fork_blocks(n4), (unsigned)nj), 256, 0, c->stream>>>(b, n4);
        launch_check(c, "fork_copy");
    }
    if (c->timing) {
        cudaEventRecord(c->ev[5], c->stream);
        cudaEventSynchronize(c->ev[5]);
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
        c->stats.fork_ms += ms;
        c->stats.fork_launches += 1;
    }
    // no host sync: the jobs are kernel parameters and every later reader of the slot / entry is
    // ordered behind the copy on the same stream
    c->stats.forks += (long long)jobs.size();
}

int guard(const std::function<void()>& f) {
    try {
        f();
        return SMX_OK;
    } catch (const SmxError& e) {
        g_err = e.what;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SMX_EDEVICE;
    }
}
}  // namespace

extern "C" {

const char* smx_last_error(void) { return g_err.c_str(); }
const char* smx_version(void) { return "smx 0.1 (sm_100a; exact SIMT + tcgen05 3xTF32)"; }

int smx_open(const smx_model_desc* desc, int device, int n_slots, int n_ckpts, smx_ctx** out) {
    return guard([&] {
        if (!desc || !out) fail(SMX_ECONFIG, "null argument");
        const smx_model_desc& d = *desc;
        if (d.model != SMX_MODEL_MLP && d.model != SMX_MODEL_CNN)
            fail(SMX_ECONFIG, "unsupported model id " + std::to_string(d.model));
        if (d.max_batch < 1 || d.max_batch > kMaxBatch) fail(SMX_ECONFIG, "max_batch must be in [1, 256]");
        if (d.n_train < 256 || (d.n_train & (d.n_train - 1))) fail(SMX_ECONFIG, "n_train must be a power of two >= 256");
        if (d.n_val < 128 || d.n_val % 128) fail(SMX_ECONFIG, "n_val must be a positive multiple of 128");
        if (d.max_steps < 1) fail(SMX_ECONFIG, "max_steps must be >= 1");
        if (d.gemm_mode != SMX_GEMM_EXACT && d.gemm_mode != SMX_GEMM_TC) fail(SMX_ECONFIG, "bad gemm_mode");
        if (n_slots < 1 || n_ckpts < 0) fail(SMX_ECONFIG, "bad slot/checkpoint counts");
        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) fail(SMX_ECONFIG, "device out of range");
        ck(cudaSetDevice(device), "cudaSetDevice");
        auto* c = new smx_ctx();
        c->d = d;
        c->device = device;
        ck(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device), "SM count");
        c->S = n_slots;
        c->C = n_ckpts;
        if (d.model == SMX_MODEL_CNN) {
            if (d.n_val % d.max_batch) fail(SMX_ECONFIG, "CNN: n_val must be a multiple of max_batch");
            c->cnn = true;
            c->palloc = cnn::kPAlloc;
            c->al = cnn::act_layout(d.max_batch);
            c->act_stride = c->al.stride;
            c->d_in = cnn::kSample;
        }
        try {
            ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
            c->cur = c->stream;
            for (auto& e : c->fj) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "fork event");
            ck(cudaEventCreateWithFlags(&c->xev, cudaEventDisableTiming), "peer event");
            const long long P2 = 2 * c->palloc;
            ck(cudaMalloc(&c->slab, sizeof(float) * P2 * n_slots), "slab");
            ck(cudaMalloc(&c->grad, sizeof(float) * c->palloc * n_slots), "grad");
            if (n_ckpts) ck(cudaMalloc(&c->pool, sizeof(float) * P2 * n_ckpts), "pool");
            ck(cudaMalloc(&c->st, sizeof(SlotState) * n_slots), "state");
            ck(cudaMalloc(&c->ck_st, sizeof(SlotState) * (n_ckpts ? n_ckpts : 1)), "ck state");
            ck(cudaMalloc(&c->hp, sizeof(float) * 4 * (long long)d.max_steps * n_slots), "hp");
            ck(cudaMalloc(&c->loss, sizeof(float) * (long long)d.max_steps * n_slots), "loss");
            ck(cudaMalloc(&c->act, sizeof(float) * c->act_stride * n_slots), "act");
            const long long rows = (long long)d.n_train + d.max_batch;
            ck(cudaMalloc(&c->xtrain, sizeof(float) * rows * c->d_in), "xtrain");
            ck(cudaMalloc(&c->ytrain, sizeof(int) * rows), "ytrain");
            ck(cudaMalloc(&c->xval, sizeof(float) * (long long)d.n_val * c->d_in), "xval");
            ck(cudaMalloc(&c->yval, sizeof(int) * d.n_val), "yval");
            if (c->cnn)
                ck(cudaMalloc(&c->zval, sizeof(float) * kEvalChunk * (long long)d.n_val * cnn::kNCP), "eval logits");
            else
                ck(cudaMalloc(&c->eval_act, sizeof(float) * kEvalChunk * (long long)d.n_val * (2 * kH + kCP)),
                   "eval act");
            ck(cudaMalloc(&c->eval_scratch, sizeof(float) * kEvalChunk * (long long)d.n_val), "eval scratch");
            ck(cudaMalloc(&c->eval_out, sizeof(double) * 2 * kEvalChunk), "eval out");
            ck(cudaMalloc(&c->eval_slots, sizeof(int) * kEvalChunk), "eval slots");
            ck(cudaMalloc(&c->scratch_slots, sizeof(int) * n_slots), "scratch slots");
            ck(cudaMalloc(&c->flag, sizeof(int)), "flag");
            ck(cudaMemsetAsync(c->grad, 0, sizeof(float) * c->palloc * n_slots, c->stream), "grad zero");
            ck(cudaMemsetAsync(c->hp, 0, sizeof(float) * 4 * (long long)d.max_steps * n_slots, c->stream), "hp zero");
            ck(cudaMemsetAsync(c->loss, 0, sizeof(float) * (long long)d.max_steps * n_slots, c->stream), "loss zero");
            ck(cudaMemsetAsync(c->act, 0, sizeof(float) * c->act_stride * n_slots, c->stream), "act zero");
            ck(cudaMemsetAsync(c->st, 0, sizeof(SlotState) * n_slots, c->stream), "state zero");
            for (auto& e : c->ev) ck(cudaEventCreate(&e), "event");
            c->ck_valid.assign(n_ckpts, 0);
            c->slot_live.assign(n_slots, 0);
            if (c->cnn) make_conv_tmaps(c);
            gen_dataset(c);
            ck(cudaStreamSynchronize(c->stream), "open sync");
        } catch (...) {
            smx_close(c);
            throw;
        }
        *out = c;
    });
}

int smx_close(smx_ctx* c) {
    if (!c) return SMX_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_graphs(c);
    void* bufs[] = {c->slab, c->grad, c->pool, c->st, c->ck_st, c->hp, c->loss, c->act, c->xtrain, c->ytrain,
                    c->xval, c->yval, c->eval_act, c->zval, c->eval_scratch, c->eval_out, c->eval_slots,
                    c->scratch_slots, c->tmaps, c->flag};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->xev) cudaEventDestroy(c->xev);
    for (auto& e : c->fj)
        if (e) cudaEventDestroy(e);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return SMX_OK;
}

int smx_param_count(const smx_ctx* c, int64_t* p, int64_t* p_alloc) {
    // without a context: the MLP (the default model)
    const bool cnn_model = c && c->cnn;
    if (p) *p = cnn_model ? cnn::kPAlgo : kPAlgo;
    if (p_alloc) *p_alloc = cnn_model ? cnn::kPAlloc : kPAlloc;
    return SMX_OK;
}

int smx_dataset_digest(smx_ctx* c, uint64_t* out) {
    return guard([&] {
        cudaSetDevice(c->device);
        const long long rows = (long long)c->d.n_train + c->d.max_batch;
        std::vector<float> x(rows * c->d_in);
        std::vector<int> y(rows);
        std::vector<float> vx((long long)c->d.n_val * c->d_in);
        std::vector<int> vy(c->d.n_val);
        ck(cudaMemcpyAsync(x.data(), c->xtrain, sizeof(float) * x.size(), cudaMemcpyDeviceToHost, c->stream), "x D2H");
        ck(cudaMemcpyAsync(y.data(), c->ytrain, sizeof(int) * y.size(), cudaMemcpyDeviceToHost, c->stream), "y D2H");
        ck(cudaMemcpyAsync(vx.data(), c->xval, sizeof(float) * vx.size(), cudaMemcpyDeviceToHost, c->stream), "vx D2H");
        ck(cudaMemcpyAsync(vy.data(), c->yval, sizeof(int) * vy.size(), cudaMemcpyDeviceToHost, c->stream), "vy D2H");
        ck(cudaStreamSynchronize(c->stream), "digest sync");
        uint64_t h = 0xcbf29ce484222325ull;
        auto eat = [&](const void* p, size_t n) {
            const unsigned char* b = static_cast<const unsigned char*>(p);
            for (size_t i = 0; i < n; ++i) {
                h ^= b[i];
                h *= 0x100000001b3ull;
            }
        };
        eat(x.data(), x.size() * 4);
        eat(y.data(), y.size() * 4);
        eat(vx.data(), vx.size() * 4);
        eat(vy.data(), vy.size() * 4);
        *out = h;
    });
}

int smx_dataset_upload(smx_ctx* c, const float* x, const int32_t* y, const float* vx, const int32_t* vy) {
    return guard([&] {
        if (!x || !y || !vx || !vy) fail(SMX_ECONFIG, "null dataset buffer");
        cudaSetDevice(c->device);
        const long long rows = (long long)c->d.n_train + c->d.max_batch;
        ck(cudaMemcpyAsync(c->xtrain, x, sizeof(float) * rows * c->d_in, cudaMemcpyHostToDevice, c->stream), "x H2D");
        ck(cudaMemcpyAsync(c->ytrain, y, sizeof(int) * rows, cudaMemcpyHostToDevice, c->stream), "y H2D");
        ck(cudaMemcpyAsync(c->xval, vx, sizeof(float) * (long long)c->d.n_val * c->d_in, cudaMemcpyHostToDevice, c->stream),
           "vx H2D");
        ck(cudaMemcpyAsync(c->yval, vy, sizeof(int) * c->d.n_val, cudaMemcpyHostToDevice, c->stream), "vy H2D");
        // tf32-exactness of the new inputs decides the GEMM path; captured graphs embed it
        ck(cudaMemsetAsync(c->flag, 0, sizeof(int), c->stream), "flag zero");
        tf32_inexact_kernel<<<592, 256, 0, c->stream>>>(reinterpret_cast<const uint32_t*>(c->xtrain), rows * c->d_in,
                                                        c->flag);
        launch_check(c, "tf32 check train");
        tf32_inexact_kernel<<<148, 256, 0, c->stream>>>(reinterpret_cast<const uint32_t*>(c->xval),
                                                        (long long)c->d.n_val * c->d_in, c->flag);
        launch_check(c, "tf32 check val");
        int inexact = 0;
        ck(cudaMemcpyAsync(&inexact, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "flag D2H");
        ck(cudaStreamSynchronize(c->stream), "dataset sync");
        const bool exact = inexact == 0;
        if (exact != c->data_tf32_exact) free_graphs(c);
        c->data_tf32_exact = exact;
    });
}

int smx_dataset_read(smx_ctx* c, float* x, int32_t* y, float* vx, int32_t* vy) {
    return guard([&] {
        if (!x || !y || !vx || !vy) fail(SMX_ECONFIG, "null dataset buffer");
        cudaSetDevice(c->device);
        const long long rows = (long long)c->d.n_train + c->d.max_batch;
        ck(cudaMemcpyAsync(x, c->xtrain, sizeof(float) * rows * c->d_in, cudaMemcpyDeviceToHost, c->stream), "x D2H");
        ck(cudaMemcpyAsync(y, c->ytrain, sizeof(int) * rows, cudaMemcpyDeviceToHost, c->stream), "y D2H");
        ck(cudaMemcpyAsync(vx, c->xval, sizeof(float) * (long long)c->d.n_val * c->d_in, cudaMemcpyDeviceToHost, c->stream),
           "vx D2H");
        ck(cudaMemcpyAsync(vy, c->yval, sizeof(int) * c->d.n_val, cudaMemcpyDeviceToHost, c->stream), "vy D2H");
        ck(cudaStreamSynchronize(c->stream), "dataset read sync");
    });
}

int smx_host_alloc(uint64_t bytes, void** out) {
    return guard([&] { ck(cudaMallocHost(out, bytes), "cudaMallocHost"); });
}

int smx_host_free(void* p) {
    return guard([&] { ck(cudaFreeHost(p), "cudaFreeHost"); });
}

int smx_hp_upload(smx_ctx* c, int slot, int64_t step0, int64_t n, const float* hp) {
    return guard([&] {
        check_slot(c, slot);
        if (step0 < 0 || n < 0 || step0 + n > c->d.max_steps)
            fail(SMX_ECONFIG, "hp rows [" + std::to_string(step0) + ", " + std::to_string(step0 + n) +
                                  ") exceed max_steps " + std::to_string(c->d.max_steps));
        for (int64_t i = 0; i < n; ++i) {
            const float bs = hp[i * 4 + 3];
            if (!(bs >= 1.0f) || bs > (float)c->d.max_batch || bs != std::floor(bs))
                fail(SMX_ECONFIG, "batch size " + std::to_string(bs) + " at step " + std::to_string(step0 + i) +
                                      " outside [1, max_batch]");
        }
        if (n == 0) return;
        cudaSetDevice(c->device);
        // pageable source: cudaMemcpyAsync stages it, so the caller's buffer is free on return
        ck(cudaMemcpyAsync(c->hp + ((long long)slot * c->d.max_steps + step0) * 4, hp, sizeof(float) * 4 * n,
                           cudaMemcpyHostToDevice, c->stream),
           "hp H2D");
    });
}

int smx_slot_init(smx_ctx* c, int slot) {
    return guard([&] {
        check_slot(c, slot);
        cudaSetDevice(c->device);
        float* w = c->slab + c->slab_stride() * slot;
        if (c->cnn)
            cnn::cnn_init_kernel<<<296, 256, 0, c->stream>>>(w, w + c->palloc, c->d.seed, init_scale(27), init_scale(288),
                                                             init_scale(576), init_scale(128));
        else
            init_kernel<<<296, 256, 0, c->stream>>>(w, w + kPAlloc, c->d.seed, init_scale(kD0), init_scale(kH),
                                                    init_scale(kH));
        launch_check(c, "init");
        ck(cudaMemsetAsync(c->st + slot, 0, sizeof(SlotState), c->stream), "state reset");
        c->slot_live[slot] = 1;
    });
}

int smx_slot_load(smx_ctx* c, int slot, int ckpt) {
    return guard([&] {
        check_slot(c, slot);
        check_ckpt(c, ckpt);
        if (!c->ck_valid[ckpt]) fail(SMX_EINTEGRITY, "load from empty checkpoint entry " + std::to_string(ckpt));
        cudaSetDevice(c->device);
        CopyJob j{reinterpret_cast<const float4*>(c->pool + c->slab_stride() * ckpt),
                  reinterpret_cast<float4*>(c->slab + c->slab_stride() * slot), c->ck_st + ckpt, c->st + slot};
        run_copy(c, {j});
        c->slot_live[slot] = 1;
    });
}

int smx_slot_save(smx_ctx* c, int slot, int ckpt) {
    return guard([&] {
        check_slot(c, slot);
        check_ckpt(c, ckpt);
        cudaSetDevice(c->device);
        CopyJob j{reinterpret_cast<const float4*>(c->slab + c->slab_stride() * slot),
                  reinterpret_cast<float4*>(c->pool + c->slab_stride() * ckpt), c->st + slot, c->ck_st + ckpt};
        run_copy(c, {j});
        c->ck_valid[ckpt] = 1;
    });
}

int smx_release_slot(smx_ctx* c, int slot) {
    return guard([&] {
        check_slot(c, slot);
        c->slot_live[slot] = 0;
    });
}

int smx_ckpt_free(smx_ctx* c, int ckpt) {
    return guard([&] {
        check_ckpt(c, ckpt);
        c->ck_valid[ckpt] = 0;
    });
}

int smx_ckpt_peer_copy(smx_ctx* dst, int dst_ckpt, smx_ctx* src, int src_ckpt) {
    return guard([&] {
        check_ckpt(dst, dst_ckpt);
        check_ckpt(src, src_ckpt);
        if (!src->ck_valid[src_ckpt]) fail(SMX_EINTEGRITY, "peer copy from empty checkpoint entry");
        if (dst->palloc != src->palloc) fail(SMX_ECONFIG, "peer copy between different models");
        // the copy runs on the destination stream behind everything the source stream has queued
        // (the SAVE that filled the entry), and the source stream waits for the copy before it
        // can overwrite the entry: device-side ordering, no host sync
        cudaSetDevice(src->device);
        ck(cudaEventRecord(src->xev, src->stream), "src record");
        cudaSetDevice(dst->device);
        ck(cudaStreamWaitEvent(dst->stream, src->xev, 0), "dst wait");
        bool direct = dst->device == src->device;
        if (!direct) {
            int can = 0;
            ck(cudaDeviceCanAccessPeer(&can, dst->device, src->device), "can access peer");
            if (can) {
                cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "enable peer");
                cudaGetLastError();
                direct = true;
            }
        }
        if (direct) {
            // K7 = the K6 fork kernel on the destination GPU reading the source pool through
            // NVLink peer loads (unified addressing): one launch, w | m and the slot state
            CopyJob j{reinterpret_cast<const float4*>(src->pool + src->slab_stride() * src_ckpt),
                      reinterpret_cast<float4*>(dst->pool + dst->slab_stride() * dst_ckpt), src->ck_st + src_ckpt,
                      dst->ck_st + dst_ckpt};
            CopyBatch<1> b{{j}};
            const long long n4 = 2 * dst->palloc / 4;
            if (dst->timing) cudaEventRecord(dst->ev[4], dst->stream);
            fork_copy_kernel<1><<<dim3(fork_blocks(n4), 1), 256, 0, dst->stream>>>(b, n4);
            launch_check(dst, "peer fork_copy");
        } else {  // no peer access between these GPUs: the runtime's staged peer copy
            if (dst->timing) cudaEventRecord(dst->ev[4], dst->stream);
            const size_t bytes = sizeof(float) * dst->slab_stride();
            ck(cudaMemcpyPeerAsync(dst->pool + dst->slab_stride() * dst_ckpt, dst->device,
                                   src->pool + src->slab_stride() * src_ckpt, src->device, bytes, dst->stream),
               "peer copy");
            ck(cudaMemcpyPeerAsync(dst->ck_st + dst_ckpt, dst->device, src->ck_st + src_ckpt, src->device,
                                   sizeof(SlotState), dst->stream),
               "peer state copy");
        }
        if (dst->timing) {
            cudaEventRecord(dst->ev[5], dst->stream);
            cudaEventSynchronize(dst->ev[5]);
            float ms = 0;
            cudaEventElapsedTime(&ms, dst->ev[4], dst->ev[5]);
            dst->stats.fork_ms += ms;
            dst->stats.fork_launches += 1;
        }
        ck(cudaEventRecord(dst->xev, dst->stream), "dst record");
        cudaSetDevice(src->device);
        ck(cudaStreamWaitEvent(src->stream, dst->xev, 0), "src wait");
        cudaSetDevice(dst->device);
        dst->ck_valid[dst_ckpt] = 1;
        dst->stats.forks += 1;
    });
}

int smx_bench_peer_copy(smx_ctx* dst, smx_ctx* src, int n, int reps, double* ms_per_copy) {
    return guard([&] {
        if (n < 1 || n > 16 || n > dst->C || n > src->C || reps < 1) fail(SMX_ECONFIG, "bench_peer_copy: 1 <= n <= 16");
        if (dst->palloc != src->palloc) fail(SMX_ECONFIG, "peer copy between different models");
        for (int i = 0; i < n; ++i)
            if (!src->ck_valid[i]) fail(SMX_EINTEGRITY, "peer copy from empty checkpoint entry");
        cudaSetDevice(src->device);
        ck(cudaStreamSynchronize(src->stream), "src sync");
        cudaSetDevice(dst->device);
        bool direct = dst->device == src->device;
        if (!direct) {
            int can = 0;
            ck(cudaDeviceCanAccessPeer(&can, dst->device, src->device), "can access peer");
            if (can) {
                cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "enable peer");
                cudaGetLastError();
                direct = true;
            }
        }
        // K7 as the engine issues it, n entries per launch (the fork kernel reading the source
        // pool through peer loads), reps launches between events on the destination stream
        CopyBatch<16> b{};
        for (int i = 0; i < n; ++i)
            b.j[i] = CopyJob{reinterpret_cast<const float4*>(src->pool + src->slab_stride() * i),
                             reinterpret_cast<float4*>(dst->pool + dst->slab_stride() * i), src->ck_st + i, dst->ck_st + i};
        const long long n4 = 2 * dst->palloc / 4;
        const size_t bytes = sizeof(float) * dst->slab_stride();
        auto once = [&] {
            if (direct) {
                fork_copy_kernel<16><<<dim3(fork_blocks(n4), n), 256, 0, dst->stream>>>(b, n4);
                launch_check(dst, "bench peer fork_copy");
            } else {
                for (int i = 0; i < n; ++i)
                    ck(cudaMemcpyPeerAsync(dst->pool + dst->slab_stride() * i, dst->device, src->pool + src->slab_stride() * i,
                                           src->device, bytes, dst->stream),
                       "peer copy");
            }
        };
        once();
        cudaEventRecord(dst->ev[6], dst->stream);
        for (int r = 0; r < reps; ++r) once();
        cudaEventRecord(dst->ev[7], dst->stream);
        ck(cudaEventSynchronize(dst->ev[7]), "bench sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, dst->ev[6], dst->ev[7]);
        *ms_per_copy = (double)ms / ((double)reps * n);
        for (int i = 0; i < n; ++i) dst->ck_valid[i] = 1;
    });
}

int smx_slot_state(smx_ctx* c, int slot, int64_t* step, int64_t* offset) {
    return guard([&] {
        check_slot(c, slot);
        cudaSetDevice(c->device);
        SlotState s;
        ck(cudaMemcpyAsync(&s, c->st + slot, sizeof s, cudaMemcpyDeviceToHost, c->stream), "state D2H");
        ck(cudaStreamSynchronize(c->stream), "state sync");
        if (step) *step = s.step;
        if (offset) *offset = s.offset;
    });
}

int smx_slot_read(smx_ctx* c, int slot, float* w, float* m) {
    return guard([&] {
        check_slot(c, slot);
        cudaSetDevice(c->device);
        const float* base = c->slab + c->slab_stride() * slot;
        if (w) ck(cudaMemcpyAsync(w, base, sizeof(float) * c->palloc, cudaMemcpyDeviceToHost, c->stream), "w D2H");
        if (m) ck(cudaMemcpyAsync(m, base + c->palloc, sizeof(float) * c->palloc, cudaMemcpyDeviceToHost, c->stream), "m D2H");
        ck(cudaStreamSynchronize(c->stream), "read sync");
    });
}

int smx_slot_write(smx_ctx* c, int slot, const float* w, const float* m, int64_t step, int64_t offset) {
    return guard([&] {
        check_slot(c, slot);
        cudaSetDevice(c->device);
        float* base = c->slab + c->slab_stride() * slot;
        ck(cudaMemcpyAsync(base, w, sizeof(float) * c->palloc, cudaMemcpyHostToDevice, c->stream), "w H2D");
        ck(cudaMemcpyAsync(base + c->palloc, m, sizeof(float) * c->palloc, cudaMemcpyHostToDevice, c->stream), "m H2D");
        SlotState s{step, offset};
        ck(cudaMemcpyAsync(c->st + slot, &s, sizeof s, cudaMemcpyHostToDevice, c->stream), "state H2D");
        ck(cudaStreamSynchronize(c->stream), "write sync");
        c->slot_live[slot] = 1;
    });
}

int smx_ckpt_read(smx_ctx* c, int ckpt, float* w, float* m, int64_t* step, int64_t* offset) {
    return guard([&] {
        check_ckpt(c, ckpt);
        if (!c->ck_valid[ckpt]) fail(SMX_EINTEGRITY, "read of empty checkpoint entry");
        cudaSetDevice(c->device);
        const float* base = c->pool + c->slab_stride() * ckpt;
        SlotState s;
        if (w) ck(cudaMemcpyAsync(w, base, sizeof(float) * c->palloc, cudaMemcpyDeviceToHost, c->stream), "w D2H");
        if (m) ck(cudaMemcpyAsync(m, base + c->palloc, sizeof(float) * c->palloc, cudaMemcpyDeviceToHost, c->stream), "m D2H");
        ck(cudaMemcpyAsync(&s, c->ck_st + ckpt, sizeof s, cudaMemcpyDeviceToHost, c->stream), "state D2H");
        ck(cudaStreamSynchronize(c->stream), "ckpt read sync");
        if (step) *step = s.step;
        if (offset) *offset = s.offset;
    });
}

int smx_ckpt_write(smx_ctx* c, int ckpt, const float* w, const float* m, int64_t step, int64_t offset) {
    return guard([&] {
        check_ckpt(c, ckpt);
        cudaSetDevice(c->device);
        float* base = c->pool + c->slab_stride() * ckpt;
        ck(cudaMemcpyAsync(base, w, sizeof(float) * c->palloc, cudaMemcpyHostToDevice, c->stream), "w H2D");
        ck(cudaMemcpyAsync(base + c->palloc, m, sizeof(float) * c->palloc, cudaMemcpyHostToDevice, c->stream), "m H2D");
        SlotState s{step, offset};
        ck(cudaMemcpyAsync(c->ck_st + ckpt, &s, sizeof s, cudaMemcpyHostToDevice, c->stream), "state H2D");
        ck(cudaStreamSynchronize(c->stream), "ckpt write sync");
        c->ck_valid[ckpt] = 1;
    });
}

int smx_train(smx_ctx* c, int n_active, const int* slots, int n_steps) {
    return guard([&] {
        if (n_active < 0 || n_steps < 0) fail(SMX_ECONFIG, "negative counts");
        if (n_active == 0 || n_steps == 0) return;
        std::vector<int> v(slots, slots + n_active);
        std::vector<char> seen(c->S, 0);
        for (int s : v) {
            check_slot(c, s);
            if (seen[s]) fail(SMX_ECONFIG, "slot " + std::to_string(s) + " listed twice");
            if (!c->slot_live[s]) fail(SMX_ECONFIG, "slot " + std::to_string(s) + " has no state (init / load it first)");
            seen[s] = 1;
        }
        cudaSetDevice(c->device);
        if (c->timing) {
            // timing mode: plain launches bracketed by events (no graphs)
            ck(cudaMemcpyAsync(c->scratch_slots, v.data(), sizeof(int) * n_active, cudaMemcpyHostToDevice, c->stream),
               "slots H2D");
            for (int i = 0; i < n_steps; ++i) {
                cudaEventRecord(c->ev[0], c->stream);
                enqueue_lockstep(c, c->scratch_slots, n_active);
                cudaEventRecord(c->ev[1], c->stream);
                ck(cudaEventSynchronize(c->ev[1]), "timing sync");
                float ms = 0, ums = 0;
                cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
                cudaEventElapsedTime(&ums, c->ev[2], c->ev[3]);
                c->stats.lockstep_ms += ms;
                c->stats.update_ms += ums;
                c->stats.update_launches += 1;
                c->stats.gemm_ms += (ms - ums);
                c->stats.gemm_launches += 1;
            }
        } else if (c->use_graphs && n_steps >= 2) {
            smx_ctx::Graph& g = graph_for(c, v);
            for (int i = 0; i < n_steps; ++i) {
                ck(cudaGraphLaunch(g.exec, c->stream), "graph launch");
                c->stats.launches += g.launches;
            }
        } else {
            ck(cudaMemcpyAsync(c->scratch_slots, v.data(), sizeof(int) * n_active, cudaMemcpyHostToDevice, c->stream),
               "slots H2D");
            for (int i = 0; i < n_steps; ++i) enqueue_lockstep(c, c->scratch_slots, n_active);
            // scratch_slots is reused by the next call: make the H2D ordering explicit
        }
        c->stats.locksteps += n_steps;
        c->stats.stage_steps += (long long)n_steps * n_active;
    });
}

int smx_eval(smx_ctx* c, int n, const int* slots, double* out) {
    return guard([&] {
        cudaSetDevice(c->device);
        const int nv = c->d.n_val;
        const long long per = (long long)nv * (2 * kH + kCP);
        for (int base = 0; base < n; base += kEvalChunk) {
            const int k = std::min(kEvalChunk, n - base);
            for (int i = 0; i < k; ++i) {
                check_slot(c, slots[base + i]);
                if (!c->slot_live[slots[base + i]]) fail(SMX_ECONFIG, "eval of a slot with no state");
            }
            ck(cudaMemcpyAsync(c->eval_slots, slots + base, sizeof(int) * k, cudaMemcpyHostToDevice, c->stream),
               "eval slots H2D");
            if (c->cnn) {
                eval_cnn(c, k);
                ck(cudaMemcpyAsync(out + 2LL * base, c->eval_out, sizeof(double) * 2 * k, cudaMemcpyDeviceToHost,
                                   c->stream),
                   "eval D2H");
                ck(cudaStreamSynchronize(c->stream), "eval sync");
                continue;
            }
            // Activations are addressed by position in the chunk, weights by slot id: each slot
            // runs its three forward GEMMs as a one-group launch (M = n_val fills the GPU).
            float* H1 = c->eval_act;
            float* H2 = c->eval_act + (long long)nv * kH;
            float* Z = c->eval_act + 2LL * nv * kH;
            const long long SW = c->slab_stride();
            for (int i = 0; i < k; ++i) {
                int* d_one = c->eval_slots + i;
                GemmArgs g = base_args(c, d_one);
                g.a = Opnd{c->xval, 0, kD0, 0};
                g.b = Opnd{c->slab + kOffW1, SW, kD0, 0};
                g.c = H1 + per * i; g.c_stride = 0; g.ldc = kH;
                g.bias = c->slab + kOffB1; g.bias_stride = SW;
                g.M = nv; g.N = kH; g.K = kD0;
                gemm<0, 0, kEpiBiasRelu>(c, g, 1, nv);
                GemmArgs g2 = base_args(c, d_one);
                g2.a = Opnd{H1 + per * i, 0, kH, 0};
                g2.b = Opnd{c->slab + kOffW2, SW, kH, 0};
                g2.c = H2 + per * i; g2.c_stride = 0; g2.ldc = kH;
                g2.bias = c->slab + kOffB2; g2.bias_stride = SW;
                g2.M = nv; g2.N = kH; g2.K = kH;
                gemm<0, 0, kEpiBiasRelu>(c, g2, 1, nv);
                GemmArgs g3 = base_args(c, d_one);
                g3.a = Opnd{H2 + per * i, 0, kH, 0};
                g3.b = Opnd{c->slab + kOffW3, SW, kH, 0};
                g3.c = Z + per * i; g3.c_stride = 0; g3.ldc = kCP;
                g3.bias = c->slab + kOffB3; g3.bias_stride = SW;
                g3.M = nv; g3.N = kCP; g3.K = kH;
                gemm<0, 0, kEpiBias>(c, g3, 1, nv);
            }
            eval_reduce_kernel<<<k, 256, 0, c->stream>>>(c->eval_slots, Z, per, c->yval, nv, c->eval_scratch,
                                                         c->eval_out);
            launch_check(c, "eval_reduce");
            ck(cudaMemcpyAsync(out + 2LL * base, c->eval_out, sizeof(double) * 2 * k, cudaMemcpyDeviceToHost,
                               c->stream),
               "eval D2H");
            ck(cudaStreamSynchronize(c->stream), "eval sync");
        }
    });
}

int smx_losses(smx_ctx* c, int slot, int64_t step0, int64_t n, float* out) {
    return guard([&] {
        check_slot(c, slot);
        if (step0 < 0 || n < 0 || step0 + n > c->d.max_steps) fail(SMX_ECONFIG, "loss range out of bounds");
        cudaSetDevice(c->device);
        ck(cudaMemcpyAsync(out, c->loss + (long long)slot * c->d.max_steps + step0, sizeof(float) * n,
                           cudaMemcpyDeviceToHost, c->stream),
           "loss D2H");
        ck(cudaStreamSynchronize(c->stream), "loss sync");
    });
}

int smx_sync(smx_ctx* c) {
    return guard([&] {
        cudaSetDevice(c->device);
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

int smx_set_timing(smx_ctx* c, int enabled) {
    c->timing = enabled != 0;
    return SMX_OK;
}

int smx_set_graphs(smx_ctx* c, int enabled) {
    c->use_graphs = enabled != 0;
    return SMX_OK;
}

int smx_get_stats(smx_ctx* c, smx_stats* out) {
    *out = c->stats;
    return SMX_OK;
}

int smx_reset_stats(smx_ctx* c) {
    c->stats = smx_stats{};
    return SMX_OK;
}

int smx_bench_kernel(smx_ctx* c, int kind, int n, int reps, double* ms_per_launch) {
    return guard([&] {
        cudaSetDevice(c->device);
        if (n < 1 || reps < 1) fail(SMX_ECONFIG, "bad bench args");
        if (kind == 0) {
            if (n > c->S) fail(SMX_ECONFIG, "more slots than allocated");
            std::vector<int> v(n);
            for (int i = 0; i < n; ++i) v[i] = i;
            ck(cudaMemcpyAsync(c->scratch_slots, v.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream), "H2D");
            StepCtx sc = step_ctx(c, c->scratch_slots);
            const long long n4 = c->palloc / 4;
            const int bx = (int)((n4 + 256 * 4 - 1) / (256 * 4));
            for (int w = 0; w < 3; ++w)
                sgd_update_kernel<<<dim3(bx, n), 256, 0, c->stream>>>(sc, c->slab, c->slab_stride(), c->grad, c->palloc, n4);
            cudaEventRecord(c->ev[6], c->stream);
            for (int r = 0; r < reps; ++r)
                sgd_update_kernel<<<dim3(bx, n), 256, 0, c->stream>>>(sc, c->slab, c->slab_stride(), c->grad, c->palloc, n4);
            cudaEventRecord(c->ev[7], c->stream);
        } else if (kind == 1) {
            if (n > c->C || n > c->S) fail(SMX_ECONFIG, "more checkpoints than allocated");
            if (n > 256) fail(SMX_ECONFIG, "at most 256 fork jobs per measured launch");
            CopyBatch<256> jobs{};
            for (int i = 0; i < n; ++i)
                jobs.j[i] = CopyJob{reinterpret_cast<const float4*>(c->slab + c->slab_stride() * i),
                                    reinterpret_cast<float4*>(c->pool + c->slab_stride() * i), c->st + i, c->ck_st + i};
            const long long n4 = 2 * c->palloc / 4;
            for (int w = 0; w < 3; ++w) fork_copy_kernel<256><<<dim3(fork_blocks(n4), n), 256, 0, c->stream>>>(jobs, n4);
            cudaEventRecord(c->ev[6], c->stream);
            for (int r = 0; r < reps; ++r) fork_copy_kernel<256><<<dim3(fork_blocks(n4), n), 256, 0, c->stream>>>(jobs, n4);
            cudaEventRecord(c->ev[7], c->stream);
        } else if (kind >= 2 && kind <= 9 && c->cnn) {
            if (n > c->S) fail(SMX_ECONFIG, "more slots than allocated");
            std::vector<int> v(n);
            for (int i = 0; i < n; ++i) v[i] = i;
            ck(cudaMemcpyAsync(c->scratch_slots, v.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream), "H2D");
            const cnn::ConvArgs a = cnn_args(c, c->scratch_slots);
            c->cur = c->stream;
            weight_images(c, a, n);
            auto launch = [&] {
                if (kind == 2) {
                    conv_forward<2>(c, a, n, c->d.max_batch);
                } else if (kind == 4) {
                    conv_dgrad<2>(c, a, n, c->d.max_batch);
                } else if (kind == 5) {
                    conv_dgrad<3>(c, a, n, c->d.max_batch);
                } else if (kind == 6) {
                    conv_forward<3>(c, a, n, c->d.max_batch);
                } else if (kind == 7 && c->d.gemm_mode == SMX_GEMM_TC) {  // the implicit GEMM alone
                    using G = cnn::Geo<3>;
                    const int splits = (c->d.max_batch * G::OH * G::OH + cnn::kSplitRows - 1) / cnn::kSplitRows;
                    conv_tc<cnn::ctc::Wgrad<3>>(c, a, splits, cnn::Part<3>::Rows, n);
                } else if (kind == 7) {
                    conv_wgrad<3>(c, a, n, c->d.max_batch);
                } else if (kind == 8) {  // conv1 weight gradient + its reduction (fused update)
                    conv_wgrad<1>(c, a, n, c->d.max_batch);
                } else if (kind == 9) {
                    conv_forward<1>(c, a, n, c->d.max_batch);
                } else if (c->d.gemm_mode == SMX_GEMM_TC) {  // the implicit GEMM alone (no split reduction)
                    using G = cnn::Geo<2>;
                    const int splits = (c->d.max_batch * G::OH * G::OH + cnn::kSplitRows - 1) / cnn::kSplitRows;
                    wgrad2_at(c, a, splits, n);
                } else {
                    conv_wgrad<2>(c, a, n, c->d.max_batch);
                }
            };
            for (int w = 0; w < 3; ++w) launch();
            cudaEventRecord(c->ev[6], c->stream);
            for (int r = 0; r < reps; ++r) launch();
            cudaEventRecord(c->ev[7], c->stream);
        } else if (kind == 2 || kind == 3) {
            // the two largest GEMMs of a lockstep at bs = 128 over n slots: 2 = fwd1 (X W1^T),
            // 3 = wgrad1 (dH1^T X); the slots' hp rows must hold bs = 128 at their current step
            if (n > c->S) fail(SMX_ECONFIG, "more slots than allocated");
            std::vector<int> v(n);
            for (int i = 0; i < n; ++i) v[i] = i;
            ck(cudaMemcpyAsync(c->scratch_slots, v.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream), "H2D");
            GemmArgs g = base_args(c, c->scratch_slots);
            const long long SW = c->slab_stride();
            if (kind == 2) {
                g.a = Opnd{c->xtrain, 0, kD0, 1};
                g.b = Opnd{c->slab + kOffW1, SW, kD0, 0};
                g.c = c->act + kActH1; g.c_stride = kActStride; g.ldc = kH;
                g.bias = c->slab + kOffB1; g.bias_stride = SW;
                g.M = c->d.max_batch; g.m_is_bs = 1; g.N = kH; g.K = kD0;
            } else {
                g.a = Opnd{c->act + kActDH1, kActStride, kH, 0};
                g.b = Opnd{c->xtrain, 0, kD0, 1};
                g.c = c->grad + kOffW1; g.c_stride = kPAlloc; g.ldc = kD0;
                g.M = kH; g.N = kD0; g.K = c->d.max_batch; g.k_is_bs = 1;
            }
            auto launch = [&] {
                if (kind == 2)
                    gemm<0, 0, kEpiBiasRelu>(c, g, n, c->d.max_batch);
                else
                    gemm<1, 1, kEpiStore>(c, g, n, kH);
            };
            for (int w = 0; w < 3; ++w) launch();
            cudaEventRecord(c->ev[6], c->stream);
            for (int r = 0; r < reps; ++r) launch();
            cudaEventRecord(c->ev[7], c->stream);
        } else {
            fail(SMX_ECONFIG, "unknown kernel kind");
        }
        ck(cudaGetLastError(), "bench launch");
        ck(cudaEventSynchronize(c->ev[7]), "bench sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[6], c->ev[7]);
        *ms_per_launch = ms / reps;
    });
}

int smx_test_gemm(smx_ctx* c, int am, int bm, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                  float* C) {
    return guard([&] {
        if (M < 1 || N < 1 || K < 1) fail(SMX_ECONFIG, "bad GEMM shape");
        cudaSetDevice(c->device);
        const size_t na = (size_t)(am ? K : M) * lda, nb = (size_t)(bm ? K : N) * ldb, nc = (size_t)M * N;
        float *dA, *dB, *dC;
        int* dslot;
        SlotState* dst;
        ck(cudaMalloc(&dA, na * 4), "A");
        ck(cudaMalloc(&dB, nb * 4), "B");
        ck(cudaMalloc(&dC, nc * 4), "C");
        ck(cudaMalloc(&dslot, 4), "slot");
        ck(cudaMalloc(&dst, sizeof(SlotState)), "st");
        ck(cudaMemcpy(dA, A, na * 4, cudaMemcpyHostToDevice), "A H2D");
        ck(cudaMemcpy(dB, B, nb * 4, cudaMemcpyHostToDevice), "B H2D");
        ck(cudaMemset(dslot, 0, 4), "slot zero");
        ck(cudaMemset(dst, 0, sizeof(SlotState)), "st zero");
        ck(cudaMemset(dC, 0xFF, nc * 4), "C poison");
        GemmArgs g{};
        g.slots = dslot;
        g.st = dst;
        g.hp = c->hp;
        g.hp_cap = c->d.max_steps;
        g.n_train_mask = c->d.n_train - 1;
        g.a = Opnd{dA, 0, lda, 0};
        g.b = Opnd{dB, 0, ldb, 0};
        g.c = dC;
        g.ldc = N;
        g.M = M;
        g.N = N;
        g.K = K;
        const int sel = am * 2 + bm;
        if (sel == 0) gemm<0, 0, kEpiStore>(c, g, 1, M);
        if (sel == 1) gemm<0, 1, kEpiStore>(c, g, 1, M);
        if (sel == 2) gemm<1, 0, kEpiStore>(c, g, 1, M);
        if (sel == 3) gemm<1, 1, kEpiStore>(c, g, 1, M);
        ck(cudaStreamSynchronize(c->stream), "gemm sync");
        ck(cudaMemcpy(C, dC, nc * 4, cudaMemcpyDeviceToHost), "C D2H");
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dC);
        cudaFree(dslot);
        cudaFree(dst);
    });
}

}  // extern "C"

#ifdef SMX_DBG_TIMELINE
// profiling variant only: arm (arm = 1: clear and arm for the next conv_ws launch) or read the
// clock64 timeline of conv_ws.cuh (arm = 0: copy n <= 4096 entries to out)
extern "C" int smx_dbg_timeline(int arm, unsigned long long* out, int n) {
    if (arm) {
        static unsigned long long zero[4096];
        const int one = 1;
        if (cudaMemcpyToSymbol(smx::cnn::ws::smx_tl, zero, sizeof(zero)) != cudaSuccess) return -1;
        if (cudaMemcpyToSymbol(smx::cnn::ws::smx_tl_armed, &one, sizeof(int)) != cudaSuccess) return -1;
        return 0;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    return cudaMemcpyFromSymbol(out, smx::cnn::ws::smx_tl, sizeof(unsigned long long) * (n < 4096 ? n : 4096)) == cudaSuccess ? 0 : -1;
}
#endif
