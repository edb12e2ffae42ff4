// K1-K3 (exact mode): grouped fp32 SIMT GEMM, one group per active slot.
//
//   C_g[m][n] = epi( sum_{k=0..K-1} A_g(m,k) * B_g(n,k) )
//
// Every output element is one fmaf chain in ascending k starting from +0, so the result is
// bit-identical to the CPU oracle's loops (oracle/trainer.c) and independent of which other
// groups share the launch (no split-K, no atomics).  Per-group M (or K) is the slot's batch size
// at its current step, read from the device hp table, so one launch (and one CUDA graph) serves
// slots with different batch sizes.
#pragma once

#include "common.cuh"

namespace smx {

struct Opnd {
    const float* base;      // operand of slot 0 (or the shared tensor)
    long long slot_stride;  // floats between consecutive slots; 0 = shared
    int ld;                 // leading dimension in floats
    int from_data;          // 1: rows start at (slot offset mod n_train)
};

struct GemmArgs {
    Opnd a, b;
    float* c;
    long long c_stride;
    int ldc;
    const float* bias;
    long long bias_stride;
    const float* mask;
    long long mask_stride;
    int ldmask;
    int M, N, K;
    int m_is_bs, k_is_bs;  // take M (or K) from the slot's batch size
    const int* slots;
    const SlotState* st;
    const float* hp;
    int hp_cap;
    int n_train_mask;
    long long m_off;  // sgd epilogue (tensor-core weight gradient): C points at w, momentum at C + m_off
};

enum Epi { kEpiStore = 0, kEpiBiasRelu = 1, kEpiBias = 2, kEpiMask = 3 };

__device__ __forceinline__ int slot_bs(const GemmArgs& p, int slot) {
    long long step = p.st[slot].step;
    return (int)p.hp[((long long)slot * p.hp_cap + step) * 4 + 3];
}

__device__ __forceinline__ const float* opnd_ptr(const Opnd& o, int slot, const SlotState* st,
                                                 int n_train_mask) {
    const float* q = o.base + o.slot_stride * slot;
    if (o.from_data) q += (long long)(st[slot].offset & n_train_mask) * o.ld;
    return q;
}

constexpr int kTM = 64, kTN = 64, kTK = 16;

// AM: 0 -> A(m,k)=a[m*ld+k], 1 -> A(m,k)=a[k*ld+m]
// BMODE: 0 -> B(n,k)=b[n*ld+k], 1 -> B(n,k)=b[k*ld+n]
template <int AM, int BMODE, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs p) {
    const int slot = p.slots[blockIdx.z];
    const int bs = (p.m_is_bs || p.k_is_bs) ? slot_bs(p, slot) : 0;
    const int M = p.m_is_bs ? bs : p.M;
    const int K = p.k_is_bs ? bs : p.K;
    const int N = p.N;
    const int m0 = blockIdx.y * kTM, n0 = blockIdx.x * kTN;
    if (m0 >= M) return;

    const float* A = opnd_ptr(p.a, slot, p.st, p.n_train_mask);
    const float* B = opnd_ptr(p.b, slot, p.st, p.n_train_mask);
    const int lda = p.a.ld, ldb = p.b.ld;

    __shared__ __align__(16) float As[kTK][kTM + 4];
    __shared__ __align__(16) float Bs[kTK][kTN + 4];

    const int t = threadIdx.x;
    const int tx = t & 15, ty = t >> 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

    for (int k0 = 0; k0 < K; k0 += kTK) {
        // ---- stage A tile (kTM x kTK) as As[k][m]
        if (AM == 0) {
            const int r = t >> 2, kk = (t & 3) * 4;
            const int m = m0 + r;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = k0 + kk + i;
                As[kk + i][r] = (m < M && k < K) ? A[(long long)m * lda + k] : 0.0f;
            }
        } else {
            const int kk = t >> 4, r = (t & 15) * 4;
            const int k = k0 + kk;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = m0 + r + i;
                As[kk][r + i] = (m < M && k < K) ? A[(long long)k * lda + m] : 0.0f;
            }
        }
        // ---- stage B tile (kTN x kTK) as Bs[k][n]
        if (BMODE == 0) {
            const int r = t >> 2, kk = (t & 3) * 4;
            const int n = n0 + r;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = k0 + kk + i;
                Bs[kk + i][r] = (n < N && k < K) ? B[(long long)n * ldb + k] : 0.0f;
            }
        } else {
            const int kk = t >> 4, r = (t & 15) * 4;
            const int k = k0 + kk;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int n = n0 + r + i;
                Bs[kk][r + i] = (n < N && k < K) ? B[(long long)k * ldb + n] : 0.0f;
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kTK; ++kk) {
            const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
            const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
            const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }

    float* C = p.c + p.c_stride * slot;
    const float* bias = (EPI == kEpiBiasRelu || EPI == kEpiBias) ? p.bias + p.bias_stride * slot : nullptr;
    const float* mask = (EPI == kEpiMask) ? p.mask + p.mask_stride * slot : nullptr;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= N) continue;
            float v = acc[i][j];
            if (EPI == kEpiBiasRelu) {
                v = __fadd_rn(v, bias[n]);
                v = v > 0.0f ? v : 0.0f;
            } else if (EPI == kEpiBias) {
                v = __fadd_rn(v, bias[n]);
            } else if (EPI == kEpiMask) {
                v = mask[(long long)m * p.ldmask + n] > 0.0f ? v : 0.0f;
            }
            C[(long long)m * p.ldc + n] = v;
        }
    }
}

}  // namespace smx
