// Device-side helpers shared by every executor kernel.
//
// Everything here is integer arithmetic or IEEE fp32 with each rounding written out
// (__fmaf_rn / __fmul_rn / __fadd_rn / __fdiv_rn); the translation unit is also compiled with
// -fmad=false so nvcc never contracts on its own.  That is what makes a stage-step a pure,
// reproducible function of (w, m, data offset, hp row) — the property the plan's exact
// metric-equality check needs (reference plan.cpp:172-179).
#pragma once

#include <cstdint>

namespace smx {

// ---- model layout (MLP 784-256-256-10) -----------------------------------
// One parameter vector per slot, fp32, padded so every tensor starts 16-byte aligned and the
// classifier has 16 rows (rows 10..15 stay exactly zero: their gradient is always 0).
constexpr int kD0 = 784;   // input features
constexpr int kH = 256;    // hidden width
constexpr int kC = 10;     // classes
constexpr int kCP = 16;    // padded classes
constexpr int kMaxBatch = 256;

constexpr long long kOffW1 = 0;
constexpr long long kOffB1 = kOffW1 + (long long)kH * kD0;   // 200704
constexpr long long kOffW2 = kOffB1 + kH;                    // 200960
constexpr long long kOffB2 = kOffW2 + (long long)kH * kH;    // 266496
constexpr long long kOffW3 = kOffB2 + kH;                    // 266752
constexpr long long kOffB3 = kOffW3 + (long long)kCP * kH;   // 270848
constexpr long long kPEnd = kOffB3 + kCP;                    // 270864
constexpr long long kPAlloc = (kPEnd + 63) / 64 * 64;        // 270912 (256-byte multiple)
constexpr long long kPAlgo = (long long)kH * kD0 + kH + (long long)kH * kH + kH + (long long)kC * kH + kC;  // 269322

// Activation scratch per slot (rows = max batch).
constexpr long long kActH1 = 0;
constexpr long long kActH2 = kActH1 + (long long)kMaxBatch * kH;
constexpr long long kActZ = kActH2 + (long long)kMaxBatch * kH;
constexpr long long kActDZ = kActZ + (long long)kMaxBatch * kCP;
constexpr long long kActDH2 = kActDZ + (long long)kMaxBatch * kCP;
constexpr long long kActDH1 = kActDH2 + (long long)kMaxBatch * kH;
constexpr long long kActStride = kActDH1 + (long long)kMaxBatch * kH;

// ---- synthetic data / init streams ----------------------------------------------------
constexpr uint64_t kStreamTrain = 1, kStreamVal = 2, kStreamTeacher = 3, kStreamInit = 4;

struct SlotState {
    long long step;    // absolute training step the slot is at
    long long offset;  // samples consumed so far (sum of bs over the prefix)
};

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Counter-based hash of (seed, stream, i, j): i < 2^36, j < 2^20.
__host__ __device__ inline uint64_t ckey(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
    return mix64(seed ^ mix64((stream << 56) ^ (i << 20) ^ j));
}

// ---- deterministic transcendental functions -----------------------------------------
// exp for x <= 88 (softmax calls it with x <= 0); Cody-Waite reduction + degree-7 Taylor.
__device__ __forceinline__ float exp_det(float x) {
    if (x < -87.0f) return 0.0f;
    float n = rintf(__fmul_rn(x, 1.44269504f));
    float r = __fmaf_rn(-n, 0.693145751953125f, x);
    r = __fmaf_rn(-n, 1.42860682e-06f, r);
    float p = 1.98412698e-04f;
    p = __fmaf_rn(p, r, 1.38888889e-03f);
    p = __fmaf_rn(p, r, 8.33333333e-03f);
    p = __fmaf_rn(p, r, 4.16666667e-02f);
    p = __fmaf_rn(p, r, 1.66666667e-01f);
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    int e = (int)n;
    return __fmul_rn(p, __int_as_float((e + 127) << 23));
}

// natural log for normal x > 0; atanh series on the mantissa.
__device__ __forceinline__ float log_det(float x) {
    unsigned bits = __float_as_uint(x);
    int e = (int)(bits >> 23) - 127;
    float f = __uint_as_float((bits & 0x7FFFFFu) | 0x3F800000u);
    if (f > 1.41421356f) {
        f = __fmul_rn(f, 0.5f);
        e += 1;
    }
    float s = __fdiv_rn(__fsub_rn(f, 1.0f), __fadd_rn(f, 1.0f));
    float s2 = __fmul_rn(s, s);
    float q = 9.09090909e-02f;
    q = __fmaf_rn(q, s2, 1.11111111e-01f);
    q = __fmaf_rn(q, s2, 1.42857143e-01f);
    q = __fmaf_rn(q, s2, 2.00000000e-01f);
    q = __fmaf_rn(q, s2, 3.33333333e-01f);
    q = __fmaf_rn(q, s2, 1.0f);
    float lf = __fmul_rn(__fadd_rn(s, s), q);
    return __fmaf_rn((float)e, 0.693147182f, lf);
}

// Softmax cross-entropy of one row of 10 logits (the spec both the CPU oracle and the GPU
// follow): returns the row loss and writes p_c - onehot_c to `dz` unscaled.
__device__ __forceinline__ float softmax_ce_row(const float* z, int y, float* dz, int* argmax) {
    float mx = z[0];
    int best = 0;
#pragma unroll
    for (int c = 1; c < kC; ++c) {
        if (z[c] > mx) {
            mx = z[c];
            best = c;
        }
    }
    float e[kC];
    float s = 0.0f;
#pragma unroll
    for (int c = 0; c < kC; ++c) {
        e[c] = exp_det(__fsub_rn(z[c], mx));
        s = __fadd_rn(s, e[c]);
    }
    if (dz) {
#pragma unroll
        for (int c = 0; c < kC; ++c) dz[c] = __fsub_rn(__fdiv_rn(e[c], s), c == y ? 1.0f : 0.0f);
    }
    if (argmax) *argmax = best;
    return __fsub_rn(log_det(s), __fsub_rn(z[y], mx));
}

}  // namespace smx
