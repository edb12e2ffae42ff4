// Non-GEMM kernels of the stage executor: K4 loss, bias-gradient reductions, K5 fused
// SGD/momentum/wd update from the device hp table, K6 fork copy, K8 synthetic data, K9 eval
// reduction, K10 seeded init.
#pragma once

#include "common.cuh"

namespace smx {

struct StepCtx {
    const int* slots;
    SlotState* st;
    const float* hp;
    int hp_cap;
};

__device__ __forceinline__ const float* hp_row(const StepCtx& c, int slot) {
    return c.hp + ((long long)slot * c.hp_cap + c.st[slot].step) * 4;
}

// ---- K8: synthetic dataset ----------------------------------------------------------
// x[r][j] = k/128 with k = (hash & 0xFF) - 128; row r holds sample (r mod n) so any window of
// up to max_batch consecutive samples is contiguous.
__global__ void gen_x_kernel(float* x, long long rows, int n, uint64_t seed, uint64_t stream) {
    const long long total = rows * kD0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / kD0;
        const int j = (int)(i - r * kD0);
        const uint64_t h = ckey(seed, stream, (uint64_t)(r % n), (uint64_t)j);
        x[i] = (float)((int)(h & 0xFF) - 128) * 0.0078125f;
    }
}

// label = argmax_c sum_j k_j * T[j][c] (exact int32), ties -> smallest c.
__global__ void gen_labels_kernel(const float* x, int* y, long long rows, uint64_t seed) {
    __shared__ signed char T[kD0 * kC];
    for (int i = threadIdx.x; i < kD0 * kC; i += blockDim.x) {
        const int j = i / kC, c = i % kC;
        T[i] = (signed char)((int)((ckey(seed, kStreamTeacher, (uint64_t)c, (uint64_t)j) >> 8) & 7) - 4);
    }
    __syncthreads();
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
         r += (long long)gridDim.x * blockDim.x) {
        int acc[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c) acc[c] = 0;
        const float* xr = x + r * kD0;
        for (int j = 0; j < kD0; ++j) {
            const int k = (int)(xr[j] * 128.0f);
#pragma unroll
            for (int c = 0; c < kC; ++c) acc[c] += k * (int)T[j * kC + c];
        }
        int best = 0;
#pragma unroll
        for (int c = 1; c < kC; ++c)
            if (acc[c] > acc[best]) best = c;
        y[r] = best;
    }
}

// Is every value tf32-exact (low 13 mantissa bits zero)?  An uploaded dataset that is not must
// not take the tensor-core GEMMs' single-MMA data path (dense_ws.cuh A_EXACT / B_EXACT).
__global__ void tf32_inexact_kernel(const uint32_t* v, long long n, int* flag) {
    uint32_t acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc |= __ldcs(v + i) & 0x1FFFu;
    if (__any_sync(0xffffffffu, acc != 0) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ---- K10: seeded He-uniform init (identical for every root: prefix_digest(cfg,0) is
// config independent, reference hpseq.cpp:591-607) ---------------------------------------
__global__ void init_kernel(float* w, float* m, uint64_t seed, float s1, float s2, float s3) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < kPAlloc;
         i += (long long)gridDim.x * blockDim.x) {
        float v = 0.0f;
        int layer = 0;
        long long o = 0, in = 0;
        float sc = 0.0f;
        if (i < kOffB1) {
            layer = 1; o = i / kD0; in = i % kD0; sc = s1;
        } else if (i >= kOffW2 && i < kOffB2) {
            layer = 2; o = (i - kOffW2) / kH; in = (i - kOffW2) % kH; sc = s2;
        } else if (i >= kOffW3 && i < kOffW3 + (long long)kC * kH) {
            layer = 3; o = (i - kOffW3) / kH; in = (i - kOffW3) % kH; sc = s3;
        }
        if (layer) {
            const uint64_t h = ckey(seed, kStreamInit, ((uint64_t)layer << 16) | (uint64_t)o, (uint64_t)in);
            const int s = (int)((h >> 40) & 0xFFFFFF) - 8388608;
            v = __fmul_rn((float)s, sc);
        }
        w[i] = v;
        m[i] = 0.0f;
    }
}

// ---- K4: softmax cross-entropy + dlogits (train) ------------------------------------
// grid: one block per group, blockDim = max batch.  Row loss reduction is sequential in row
// order (thread 0) so it matches the oracle's loop exactly.
__global__ void loss_train_kernel(StepCtx c, const int* labels, int n_train_mask, float* act,
                                  long long act_stride, float* loss_hist) {
    const int slot = c.slots[blockIdx.x];
    const float* hp = hp_row(c, slot);
    const int B = (int)hp[3];
    const long long step = c.st[slot].step;
    const long long off = c.st[slot].offset & n_train_mask;
    const float* Z = act + act_stride * slot + kActZ;
    float* dZ = act + act_stride * slot + kActDZ;
    __shared__ float row_loss[kMaxBatch];
    const int r = threadIdx.x;
    if (r < B) {
        float dz[kC];
        const int y = labels[off + r];
        row_loss[r] = softmax_ce_row(Z + (long long)r * kCP, y, dz, nullptr);
        const float fb = (float)B;
#pragma unroll
        for (int k = 0; k < kC; ++k) dZ[(long long)r * kCP + k] = __fdiv_rn(dz[k], fb);
#pragma unroll
        for (int k = kC; k < kCP; ++k) dZ[(long long)r * kCP + k] = 0.0f;
    }
    __syncthreads();
    if (r == 0) {
        float s = 0.0f;
        for (int i = 0; i < B; ++i) s = __fadd_rn(s, row_loss[i]);
        loss_hist[(long long)slot * c.hp_cap + step] = __fdiv_rn(s, (float)B);
    }
}

// ---- bias gradient: db[n] = sum_{r<B} dY[r][n] in row order --------------------------
__global__ void colsum_kernel(StepCtx c, const float* act, long long act_stride, long long dy_off,
                              int ld, int N, float* grad, long long grad_stride, long long db_off) {
    const int slot = c.slots[blockIdx.y];
    const int B = (int)hp_row(c, slot)[3];
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const float* dY = act + act_stride * slot + dy_off;
    float s = 0.0f;
    for (int r = 0; r < B; ++r) s = __fadd_rn(s, dY[(long long)r * ld + n]);
    grad[grad_stride * slot + db_off + n] = s;
}

// Tensor-core mode: the same sums with 8 row-lanes per column and a fixed-order combine
// (deterministic and grouping-invariant; not the oracle's sequential order, which only the exact
// mode promises).  grid: (ceil(N/32), groups), block 256.
__global__ void colsum_fast_kernel(StepCtx c, const float* act, long long act_stride, long long dy_off, int ld, int N,
                                   float* grad, long long grad_stride, long long db_off) {
    const int slot = c.slots[blockIdx.y];
    const int B = (int)hp_row(c, slot)[3];
    const int col = threadIdx.x & 31, lane_r = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + col;
    __shared__ float part[8][33];
    const float* dY = act + act_stride * slot + dy_off;
    float s = 0.0f;
    if (n < N)
        for (int r = lane_r; r < B; r += 8) s = __fadd_rn(s, dY[(long long)r * ld + n]);
    part[lane_r][col] = s;
    __syncthreads();
    if (lane_r == 0 && n < N) {
        float t = part[0][col];
        for (int i = 1; i < 8; ++i) t = __fadd_rn(t, part[i][col]);
        grad[grad_stride * slot + db_off + n] = t;
    }
}

// ---- K5: fused SGD / momentum / weight-decay update ----------------------------------
//   g' = fma(wd, w, g);  m = fma(mu, m, g');  w = fma(-lr, m, w)
// (PyTorch SGD semantics, no dampening / Nesterov).  (lr, mu, wd) come from the
// slot's hp-table row at its current step, so one launch serves every active stage.
// 20 B/param of HBM traffic (read w, g, m; write w, m), 16-byte vectors.
__global__ void __launch_bounds__(256) sgd_update_kernel(StepCtx c, float* slab, long long slab_stride,
                                                         const float* grad, long long grad_stride,
                                                         long long n4) {
    const int slot = c.slots[blockIdx.y];
    const float* hp = hp_row(c, slot);
    const float nlr = -hp[0], mu = hp[1], wd = hp[2];
    float4* w = reinterpret_cast<float4*>(slab + slab_stride * slot);
    float4* m = reinterpret_cast<float4*>(slab + slab_stride * slot + slab_stride / 2);  // [w | m]
    const float4* g = reinterpret_cast<const float4*>(grad + grad_stride * slot);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        float4 wv = w[i], mv = m[i];
        const float4 gv = __ldcs(g + i);
        mv.x = __fmaf_rn(mu, mv.x, __fmaf_rn(wd, wv.x, gv.x));
        mv.y = __fmaf_rn(mu, mv.y, __fmaf_rn(wd, wv.y, gv.y));
        mv.z = __fmaf_rn(mu, mv.z, __fmaf_rn(wd, wv.z, gv.z));
        mv.w = __fmaf_rn(mu, mv.w, __fmaf_rn(wd, wv.w, gv.w));
        wv.x = __fmaf_rn(nlr, mv.x, wv.x);
        wv.y = __fmaf_rn(nlr, mv.y, wv.y);
        wv.z = __fmaf_rn(nlr, mv.z, wv.z);
        wv.w = __fmaf_rn(nlr, mv.w, wv.w);
        w[i] = wv;
        m[i] = mv;
    }
}

// K5 fused into a gradient producer (K3+K5): the same rule as sgd_update_kernel, applied by the
// kernel that computes the parameter's final gradient, so the gradient never round-trips through
// HBM (8 B/param/step).  Bitwise identical to storing g and running sgd_update_kernel.
struct SgdRow {
    float nlr, mu, wd;
};
__device__ __forceinline__ SgdRow sgd_row(const float* hp, int hp_cap, const SlotState* st, int slot) {
    const float* r = hp + ((long long)slot * hp_cap + st[slot].step) * 4;
    return SgdRow{-r[0], r[1], r[2]};
}
__device__ __forceinline__ void sgd_apply(float* w, float* m, long long i, float g, const SgdRow& h) {
    const float mv = __fmaf_rn(h.mu, m[i], __fmaf_rn(h.wd, w[i], g));
    m[i] = mv;
    w[i] = __fmaf_rn(h.nlr, mv, w[i]);
}

// Tensor-core MLP lockstep, after the last weight-gradient GEMM (layer 1, whose epilogue updates
// W1 in place): blocks [0, nb): the layer-1 bias gradient (colsum_fast order) with the update
// fused; blocks [nb, ...): the update of the parameter range [lo, hi) (W2, b2, W3, b3) from the
// gradient slab -- every reader of those weights (the input-gradient GEMMs) has finished.
__global__ void __launch_bounds__(256) colsum_sgd_kernel(StepCtx c, const float* act, long long act_stride,
                                                         long long dy_off, int ld, int N, float* slab,
                                                         long long slab_stride, const float* grad,
                                                         long long grad_stride, long long db_off, int nb,
                                                         long long lo, long long hi) {
    const int slot = c.slots[blockIdx.y];
    const SgdRow h = sgd_row(c.hp, c.hp_cap, c.st, slot);
    float* w = slab + slab_stride * slot;
    float* m = w + slab_stride / 2;
    if ((int)blockIdx.x < nb) {
        const int B = (int)hp_row(c, slot)[3];
        const int col = threadIdx.x & 31, lane_r = threadIdx.x >> 5;
        const int n = blockIdx.x * 32 + col;
        __shared__ float part[8][33];
        const float* dY = act + act_stride * slot + dy_off;
        float s = 0.0f;
        if (n < N)
            for (int r = lane_r; r < B; r += 8) s = __fadd_rn(s, dY[(long long)r * ld + n]);
        part[lane_r][col] = s;
        __syncthreads();
        if (lane_r == 0 && n < N) {
            float t = part[0][col];
            for (int i = 1; i < 8; ++i) t = __fadd_rn(t, part[i][col]);
            sgd_apply(w, m, db_off + n, t, h);
        }
        return;
    }
    const float* g = grad + grad_stride * slot;
    for (long long i = lo + ((long long)blockIdx.x - nb) * blockDim.x + threadIdx.x; i < hi;
         i += (long long)(gridDim.x - nb) * blockDim.x)
        sgd_apply(w, m, i, __ldcs(g + i), h);
}

// Advance each active slot by one step: step += 1, offset += bs.
__global__ void advance_kernel(StepCtx c, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int slot = c.slots[i];
    const int B = (int)hp_row(c, slot)[3];
    c.st[slot].step += 1;
    c.st[slot].offset += B;
}

// ---- K6: fork copy (slot <-> checkpoint pool), batched --------------------------------
struct CopyJob {
    const float4* src;
    float4* dst;
    const SlotState* src_st;
    SlotState* dst_st;
};

// Jobs travel as a kernel parameter (no job-list H2D, no host sync between forks): one launch
// moves up to N (slot, entry) pairs, blockIdx.y = job.  N = 16 for the engine's forks (512 B
// of parameters), 256 for the bench's many-checkpoint K6 measurement.
template <int N>
struct CopyBatch {
    CopyJob j[N];
};

template <int N>
__global__ void __launch_bounds__(256) fork_copy_kernel(const __grid_constant__ CopyBatch<N> jobs, long long n4) {
    const CopyJob j = jobs.j[blockIdx.y];
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    // 4 independent 16-byte loads in flight per thread
    for (; i + 3 * stride < n4; i += 4 * stride) {
        const float4 a = __ldcs(j.src + i), b = __ldcs(j.src + i + stride);
        const float4 cc = __ldcs(j.src + i + 2 * stride), d = __ldcs(j.src + i + 3 * stride);
        j.dst[i] = a;
        j.dst[i + stride] = b;
        j.dst[i + 2 * stride] = cc;
        j.dst[i + 3 * stride] = d;
    }
    for (; i < n4; i += stride) j.dst[i] = __ldcs(j.src + i);
    if (blockIdx.x == 0 && threadIdx.x == 0) *j.dst_st = *j.src_st;
}

// ---- K9: validation loss / accuracy with a fixed reduction order ---------------------
// Per-sample losses go to `scratch`; warp 0 then sums lane-strided partials sequentially and
// folds them with a fixed shuffle tree (the oracle restates exactly this order).
__global__ void eval_reduce_kernel(const int* eval_slots, const float* Z, long long z_stride,
                                   const int* labels, int n_val, float* scratch, double* out) {
    const int g = blockIdx.x;
    const float* Zg = Z + z_stride * g;
    float* lg = scratch + (long long)g * n_val;
    __shared__ int correct_s[256];
    int correct = 0;
    for (int r = threadIdx.x; r < n_val; r += blockDim.x) {
        int am = 0;
        lg[r] = softmax_ce_row(Zg + (long long)r * kCP, labels[r], nullptr, &am);
        correct += (am == labels[r]);
    }
    correct_s[threadIdx.x] = correct;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        float v = 0.0f;
        for (int t = 0; t < n_val / 32; ++t) v = __fadd_rn(v, lg[lane + 32 * t]);
        for (int w = 16; w >= 1; w >>= 1) {
            const float o = __shfl_down_sync(0xffffffffu, v, w);
            if (lane < w) v = __fadd_rn(v, o);
        }
        int cs = 0;
        if (lane == 0) {
            for (int i = 0; i < (int)blockDim.x; ++i) cs += correct_s[i];
            out[g * 2 + 0] = (double)__fdiv_rn(v, (float)n_val);
            out[g * 2 + 1] = (double)cs / (double)n_val;
        }
    }
    (void)eval_slots;
}

}  // namespace smx
