/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle of the stage executor's CNN model.
 *
 * Independent plain-C restatement of the arithmetic the GPU exact mode implements for
 * SMX_MODEL_CNN (conv3x3 3->32 s1, conv3x3 32->64 s2, conv3x3 64->128 s2, ReLU, global average
 * pool, FC 128->10, softmax-CE, PyTorch SGD).  Same rules as trainer.c: compiled with
 * -ffp-contract=off, every dot product is one fmaf chain in the order DESIGN.md §3b states,
 * sums are sequential IEEE adds.  Anchors in the reference: worker_execute,
 * the prefix-only TrainingOracle invariant, PyTorch SGD,
 * the data-offset-in-checkpoint rule.  The model itself is the builder's
 * (SURVEY §8d "small CNN"; the reference ships none) — "parity unpinned" by the reference.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* image: 32 x 32 x 4 (NHWC, channel 3 == 0) */
enum { IMG = 32, CH = 3, CHP = 4, SAMPLE = IMG * IMG * CHP, NC = 10, NCP = 16 };

/* layer geometry: input H, Cin (padded), Cin real, Cout, stride */
static const int LH[4] = {0, 32, 32, 16};
static const int LCI[4] = {0, 4, 32, 64};
static const int LCR[4] = {0, 3, 32, 64};
static const int LCO[4] = {0, 32, 64, 128};
static const int LS[4] = {0, 1, 2, 2};

#define O_W1 0L
#define O_B1 (O_W1 + 32L * 9 * 4)
#define O_W2 (O_B1 + 32)
#define O_B2 (O_W2 + 64L * 9 * 32)
#define O_W3 (O_B2 + 64)
#define O_B3 (O_W3 + 128L * 9 * 64)
#define O_W4 (O_B3 + 128)
#define O_B4 (O_W4 + (long)NCP * 128)
#define O_END (O_B4 + NCP)
#define P_ALLOC ((O_END + 63) / 64 * 64)
#define P_ALGO (32L * 27 + 32 + 64L * 288 + 64 + 128L * 576 + 128 + 10L * 128 + 10)

static const long OW[4] = {0, O_W1, O_W2, O_W3};
static const long OB[4] = {0, O_B1, O_B2, O_B3};

void orc_cnn_layout(int64_t* p_algo, int64_t* p_alloc, int64_t* off) {
    if (p_algo) *p_algo = P_ALGO;
    if (p_alloc) *p_alloc = P_ALLOC;
    if (off) {
        off[0] = O_W1; off[1] = O_B1; off[2] = O_W2; off[3] = O_B2; off[4] = O_W3;
        off[5] = O_B3; off[6] = O_W4; off[7] = O_B4; off[8] = O_END;
    }
}

static uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t key4(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
    return splitmix(seed ^ splitmix((stream << 56) ^ (i << 20) ^ j));
}

/* ---- data: streams 5 (train), 6 (val), 7 (teacher) ------------------ */
static void gen_imgs(uint64_t seed, uint64_t stream, long rows, long n, float* x, int32_t* y) {
    signed char T[CH * 16][NC];
    for (int b = 0; b < CH * 16; ++b)
        for (int c = 0; c < NC; ++c) T[b][c] = (signed char)((int)((key4(seed, 7, (uint64_t)c, (uint64_t)b) >> 8) & 7) - 4);
#pragma omp parallel for schedule(static)
    for (long r = 0; r < rows; ++r) {
        int acc[NC] = {0};
        float* xr = x + r * SAMPLE;
        for (int h = 0; h < IMG; ++h)
            for (int w = 0; w < IMG; ++w) {
                for (int ch = 0; ch < CH; ++ch) {
                    const uint64_t j = (uint64_t)((h * IMG + w) * CH + ch);
                    const int k = (int)(key4(seed, stream, (uint64_t)(r % n), j) & 0xFF) - 128;
                    xr[(h * IMG + w) * CHP + ch] = (float)k * 0.0078125f;
                    const int b = ch * 16 + (h >> 3) * 4 + (w >> 3);
                    for (int c = 0; c < NC; ++c) acc[c] += k * (int)T[b][c];
                }
                xr[(h * IMG + w) * CHP + 3] = 0.0f;
            }
        int best = 0;
        for (int c = 1; c < NC; ++c)
            if (acc[c] > acc[best]) best = c;
        y[r] = best;
    }
}

void orc_cnn_gen_dataset(uint64_t seed, int n_train, int max_batch, int n_val, float* x, int32_t* y, float* vx,
                         int32_t* vy) {
    gen_imgs(seed, 5, (long)n_train + max_batch, n_train, x, y);
    gen_imgs(seed, 6, n_val, n_val, vx, vy);
}

/* ---- init: stream 8 ---------------------------------------------------- */
void orc_cnn_init(uint64_t seed, float* w, float* m) {
    memset(w, 0, sizeof(float) * P_ALLOC);
    memset(m, 0, sizeof(float) * P_ALLOC);
    for (int l = 1; l <= 4; ++l) {
        const int rows = l == 4 ? NC : LCO[l];
        const int fan = l == 4 ? 128 : 9 * LCR[l];
        const float sc = (float)sqrt(6.0 / (double)fan) * (1.0f / 8388608.0f);
        for (int o = 0; o < rows; ++o)
            for (int i = 0; i < fan; ++i) {
                const uint64_t h = key4(seed, 8, ((uint64_t)l << 16) | (uint64_t)o, (uint64_t)i);
                const int s = (int)((h >> 40) & 0xFFFFFF) - 8388608;
                long at;
                if (l == 4) {
                    at = O_W4 + (long)o * 128 + i;
                } else {
                    const int t = i / LCR[l], ci = i % LCR[l];
                    at = OW[l] + ((long)o * 9 + t) * LCI[l] + ci;
                }
                w[at] = (float)s * sc;
            }
    }
}

/* ---- training step ------------------------------------------------------ */
typedef struct {
    float a1[256L * 1024 * 32], a2[256L * 256 * 64], a3[256L * 64 * 128];
    float d1[256L * 1024 * 32], d2[256L * 256 * 64], d3[256L * 64 * 128];
    float g[256 * 128], dz[256 * NCP], dg[256 * 128];
    float wt[9 * 64 * 128];  /* W^T [t][ci][co] of the current layer */
    float acc[128 * 9 * 64];
    float grad[P_ALLOC];
} Work;

/* out[n][p][co] = relu(b[co] + sum_{t valid asc} sum_{ci < Cr asc} in[n][q(p,t)][ci] * W[co][t][ci]) */
/* nt > 1: samples split over OpenMP threads -- every output is still its own sequential chain, so
 * the result is bitwise the nt == 1 result (tested). */
static void conv_fwd(int l, const float* restrict in, int B, const float* restrict w, float* restrict out,
                     Work* wk, int nt) {
    const int H = LH[l], Ci = LCI[l], Cr = LCR[l], Co = LCO[l], S = LS[l], OH = H / S;
    for (int co = 0; co < Co; ++co)
        for (int t = 0; t < 9; ++t)
            for (int ci = 0; ci < Ci; ++ci) wk->wt[((long)t * Ci + ci) * Co + co] = w[OW[l] + ((long)co * 9 + t) * Ci + ci];
    (void)nt;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (int n = 0; n < B; ++n)
        for (int oh = 0; oh < OH; ++oh)
            for (int ow = 0; ow < OH; ++ow) {
                float acc[128];
                for (int co = 0; co < Co; ++co) acc[co] = 0.0f;
                for (int t = 0; t < 9; ++t) {
                    const int ih = oh * S + t / 3 - 1, iw = ow * S + t % 3 - 1;
                    if (ih < 0 || ih >= H || iw < 0 || iw >= H) continue;
                    const float* xin = in + (((long)n * H + ih) * H + iw) * Ci;
                    for (int ci = 0; ci < Cr; ++ci) {
                        const float xv = xin[ci];
                        const float* restrict wr = wk->wt + ((long)t * Ci + ci) * Co;
                        for (int co = 0; co < Co; ++co) acc[co] = fmaf(xv, wr[co], acc[co]);
                    }
                }
                float* o = out + (((long)n * OH + oh) * OH + ow) * Co;
                for (int co = 0; co < Co; ++co) {
                    const float v = acc[co] + w[OB[l] + co];
                    o[co] = v > 0.0f ? v : 0.0f;
                }
            }
}

/* gW[co][t][ci] = sum_{n asc, p asc, valid} dy[n][p][co] * in[n][q(p,t)][ci];  gb[co] = sum dy
 * Accumulated as acc[t][ci][co] (the co loop innermost: contiguous in dy and acc, so it
 * vectorises); the (t, ci) rows are split over OpenMP threads when nt > 1.  Every (co, t, ci)
 * chain keeps its (n asc, p asc) order, so the result is bitwise the nt == 1 result (tested). */
static void conv_wgrad(int l, const float* restrict in, const float* restrict dy, int B, float* restrict grad,
                       Work* wk, int nt) {
    const int H = LH[l], Ci = LCI[l], Cr = LCR[l], Co = LCO[l], S = LS[l], OH = H / S;
    float* restrict acc = wk->acc; /* [t][ci][co] */
    memset(acc, 0, sizeof(float) * (size_t)Co * 9 * Ci);
    float gb[128];
    for (int co = 0; co < Co; ++co) gb[co] = 0.0f;
    const int rows = 9 * Cr;  /* (t, ci) rows with real input channels */
    const int nblk = nt > 1 ? (rows < nt ? rows : nt) : 1;
    (void)nt;
#pragma omp parallel for num_threads(nblk) schedule(static) if (nblk > 1)
    for (int blk = 0; blk < nblk; ++blk) {
        const int r0 = rows * blk / nblk, r1 = rows * (blk + 1) / nblk;
        for (int n = 0; n < B; ++n)
            for (int oh = 0; oh < OH; ++oh)
                for (int ow = 0; ow < OH; ++ow) {
                    const float* restrict d = dy + (((long)n * OH + oh) * OH + ow) * Co;
                    if (blk == 0)
                        for (int co = 0; co < Co; ++co) gb[co] = gb[co] + d[co];
                    for (int r = r0; r < r1; ++r) {
                        const int t = r / Cr, ci = r % Cr;
                        const int ih = oh * S + t / 3 - 1, iw = ow * S + t % 3 - 1;
                        if (ih < 0 || ih >= H || iw < 0 || iw >= H) continue;
                        const float xv = in[(((long)n * H + ih) * H + iw) * Ci + ci];
                        float* restrict a = acc + ((long)t * Ci + ci) * Co;
                        for (int co = 0; co < Co; ++co) a[co] = fmaf(d[co], xv, a[co]);
                    }
                }
    }
    for (int co = 0; co < Co; ++co)
        for (int t = 0; t < 9; ++t)
            for (int ci = 0; ci < Ci; ++ci) grad[OW[l] + ((long)co * 9 + t) * Ci + ci] = acc[((long)t * Ci + ci) * Co + co];
    for (int co = 0; co < Co; ++co) grad[OB[l] + co] = gb[co];
}

/* dx[n][q][ci] = (act[n][q][ci] > 0) ? sum_{t asc valid} sum_{co asc} dy[n][p(q,t)][co] * W[co][t][ci] : 0 */
static void conv_dgrad(int l, const float* restrict dy, const float* restrict w, const float* restrict act, int B,
                       float* restrict dx, int nt) {
    const int H = LH[l], Ci = LCI[l], Co = LCO[l], S = LS[l], OH = H / S;
    (void)nt;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (int n = 0; n < B; ++n)
        for (int ih = 0; ih < H; ++ih)
            for (int iw = 0; iw < H; ++iw) {
                float acc[64];
                for (int ci = 0; ci < Ci; ++ci) acc[ci] = 0.0f;
                for (int t = 0; t < 9; ++t) {
                    const int kh = t / 3, kw = t % 3;
                    const int nh = ih + 1 - kh, nw = iw + 1 - kw;
                    if (nh < 0 || nw < 0 || nh % S || nw % S) continue;
                    const int oh = nh / S, ow = nw / S;
                    if (oh >= OH || ow >= OH) continue;
                    const float* d = dy + (((long)n * OH + oh) * OH + ow) * Co;
                    for (int co = 0; co < Co; ++co) {
                        const float dv = d[co];
                        const float* restrict wr = w + OW[l] + ((long)co * 9 + t) * Ci;
                        for (int ci = 0; ci < Ci; ++ci) acc[ci] = fmaf(dv, wr[ci], acc[ci]);
                    }
                }
                const long at = (((long)n * H + ih) * H + iw) * Ci;
                for (int ci = 0; ci < Ci; ++ci) dx[at + ci] = act[at + ci] > 0.0f ? acc[ci] : 0.0f;
            }
}

/* global average pool + FC: g[n][c] = (sum_{p asc} a3[n][p][c]) * 2^-6;
 * z[n][k] = (fmaf chain over c asc of g[n][c] * W4[k][c]) + b4[k] */
static void head_fwd(const float* restrict a3, int B, const float* restrict w, float* restrict g, float* restrict z,
                     int nt) {
    (void)nt;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (int n = 0; n < B; ++n) {
        for (int c = 0; c < 128; ++c) {
            float s = 0.0f;
            for (int p = 0; p < 64; ++p) s = s + a3[((long)n * 64 + p) * 128 + c];
            g[n * 128 + c] = s * 0.015625f;
        }
        for (int k = 0; k < NCP; ++k) {
            float acc = 0.0f;
            for (int c = 0; c < 128; ++c) acc = fmaf(g[n * 128 + c], w[O_W4 + k * 128 + c], acc);
            z[n * NCP + k] = acc + w[O_B4 + k];
        }
    }
}

float orc_ce_row(const float* z, int y, float* dz, int* am);

static float cnn_step(float* restrict w, float* restrict m, const float* hp, const float* x, const int32_t* y,
                      Work* wk, int nt) {
    const int B = (int)hp[3];
    float z[256 * NCP];
    conv_fwd(1, x, B, w, wk->a1, wk, nt);
    conv_fwd(2, wk->a1, B, w, wk->a2, wk, nt);
    conv_fwd(3, wk->a2, B, w, wk->a3, wk, nt);
    head_fwd(wk->a3, B, w, wk->g, z, nt);
    float lsum = 0.0f;
    const float fb = (float)B;
    for (int n = 0; n < B; ++n) {
        float d[NC];
        lsum = lsum + orc_ce_row(z + n * NCP, y[n], d, NULL);
        for (int k = 0; k < NC; ++k) wk->dz[n * NCP + k] = d[k] / fb;
        for (int k = NC; k < NCP; ++k) wk->dz[n * NCP + k] = 0.0f;
    }
    memset(wk->grad, 0, sizeof wk->grad);
    /* FC grads: gW4[k][c] = fmaf chain over n asc; gb4[k] = sum over n */
    for (int k = 0; k < NCP; ++k) {
        float sb = 0.0f;
        for (int c = 0; c < 128; ++c) {
            float acc = 0.0f;
            for (int n = 0; n < B; ++n) acc = fmaf(wk->dz[n * NCP + k], wk->g[n * 128 + c], acc);
            wk->grad[O_W4 + k * 128 + c] = acc;
        }
        for (int n = 0; n < B; ++n) sb = sb + wk->dz[n * NCP + k];
        wk->grad[O_B4 + k] = sb;
    }
    /* dg[n][c] = fmaf chain over k < 16;  d3 = (a3 > 0) ? dg * 2^-6 : 0 */
    for (int n = 0; n < B; ++n)
        for (int c = 0; c < 128; ++c) {
            float acc = 0.0f;
            for (int k = 0; k < NCP; ++k) acc = fmaf(wk->dz[n * NCP + k], w[O_W4 + k * 128 + c], acc);
            wk->dg[n * 128 + c] = acc * 0.015625f;
        }
    for (int n = 0; n < B; ++n)
        for (int p = 0; p < 64; ++p)
            for (int c = 0; c < 128; ++c) {
                const long i = ((long)n * 64 + p) * 128 + c;
                wk->d3[i] = wk->a3[i] > 0.0f ? wk->dg[n * 128 + c] : 0.0f;
            }
    conv_wgrad(3, wk->a2, wk->d3, B, wk->grad, wk, nt);
    conv_dgrad(3, wk->d3, w, wk->a2, B, wk->d2, nt);
    conv_wgrad(2, wk->a1, wk->d2, B, wk->grad, wk, nt);
    conv_dgrad(2, wk->d2, w, wk->a1, B, wk->d1, nt);
    conv_wgrad(1, x, wk->d1, B, wk->grad, wk, nt);
    /* K5 (same rule as the MLP) */
    const float nlr = -hp[0], mu = hp[1], wd = hp[2];
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (long i = 0; i < P_ALLOC; ++i) {
        const float mv = fmaf(mu, m[i], fmaf(wd, w[i], wk->grad[i]));
        m[i] = mv;
        w[i] = fmaf(nlr, mv, w[i]);
    }
    return lsum / fb;
}

static int cnn_train_slot(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows,
                          int n_steps, const float* x, const int32_t* y, int n_train, float* loss_hist, Work* wk,
                          int nt) {
    for (int i = 0; i < n_steps; ++i) {
        const int64_t s = *step;
        if (s < 0 || s >= hp_rows) return 1;
        const float* row = hp + s * 4;
        const long off = (long)(*offset & (int64_t)(n_train - 1));
        const float l = cnn_step(w, m, row, x + off * SAMPLE, y + off, wk, nt);
        if (loss_hist) loss_hist[s] = l;
        *step = s + 1;
        *offset += (int64_t)row[3];
    }
    return 0;
}

int orc_cnn_train(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows, int n_steps,
                  const float* x, const int32_t* y, int n_train, float* loss_hist) {
    Work* wk = (Work*)malloc(sizeof(Work));
    if (!wk) return 2;
    const int rc = cnn_train_slot(w, m, step, offset, hp, hp_rows, n_steps, x, y, n_train, loss_hist, wk, 1);
    free(wk);
    return rc;
}

int orc_cnn_train_mt(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows,
                     int n_steps, const float* x, const int32_t* y, int n_train, float* loss_hist, int threads) {
    Work* wk = (Work*)malloc(sizeof(Work));
    if (!wk) return 2;
    const int rc = cnn_train_slot(w, m, step, offset, hp, hp_rows, n_steps, x, y, n_train, loss_hist, wk,
                                  threads > 1 ? threads : 1);
    free(wk);
    return rc;
}

int orc_cnn_train_many(int n_slots, float** w, float** m, int64_t* step, int64_t* offset, const float** hp,
                       int64_t hp_rows, int n_steps, const float* x, const int32_t* y, int n_train, float** loss_hist,
                       int threads) {
    int rc = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    (void)threads;
#pragma omp parallel reduction(| : rc)
    {
        Work* wk = (Work*)malloc(sizeof(Work));
#pragma omp for schedule(dynamic, 1)
        for (int s = 0; s < n_slots; ++s)
            rc |= wk ? cnn_train_slot(w[s], m[s], &step[s], &offset[s], hp[s], hp_rows, n_steps, x, y, n_train,
                                      loss_hist ? loss_hist[s] : NULL, wk, 1)
                     : 2;
        free(wk);
    }
    return rc;
}

/* ---- eval (same reduction as the MLP: DESIGN.md §3.5) ------------------------------------- */
void orc_cnn_eval_mt(const float* w, const float* vx, const int32_t* vy, int n_val, double* out, int nt);

void orc_cnn_eval(const float* w, const float* vx, const int32_t* vy, int n_val, double* out) {
    orc_cnn_eval_mt(w, vx, vy, n_val, out, 1);
}

void orc_cnn_eval_mt(const float* w, const float* vx, const int32_t* vy, int n_val, double* out, int nt) {
    if (nt < 1) nt = 1;
    Work* wk = (Work*)malloc(sizeof(Work));
    float* loss = (float*)malloc(sizeof(float) * (size_t)n_val);
    float z[256 * NCP];
    long correct = 0;
    for (int r0 = 0; r0 < n_val; r0 += 256) {
        const int B = n_val - r0 < 256 ? n_val - r0 : 256;
        const float* xb = vx + (long)r0 * SAMPLE;
        conv_fwd(1, xb, B, w, wk->a1, wk, nt);
        conv_fwd(2, wk->a1, B, w, wk->a2, wk, nt);
        conv_fwd(3, wk->a2, B, w, wk->a3, wk, nt);
        head_fwd(wk->a3, B, w, wk->g, z, nt);
        for (int n = 0; n < B; ++n) {
            int am = 0;
            loss[r0 + n] = orc_ce_row(z + n * NCP, vy[r0 + n], NULL, &am);
            correct += (am == vy[r0 + n]);
        }
    }
    float part[32];
    for (int l = 0; l < 32; ++l) {
        float v = 0.0f;
        for (int t = 0; t < n_val / 32; ++t) v = v + loss[l + 32 * t];
        part[l] = v;
    }
    for (int wdt = 16; wdt >= 1; wdt >>= 1)
        for (int l = 0; l < wdt; ++l) part[l] = part[l] + part[l + wdt];
    out[0] = (double)(part[0] / (float)n_val);
    out[1] = (double)correct / (double)n_val;
    free(loss);
    free(wk);
}

/* Test hooks: single-layer pieces on caller buffers (B samples), for the GPU kernel tests. */
void orc_cnn_conv_fwd(int l, const float* in, int B, const float* w, float* out) {
    Work* wk = (Work*)malloc(sizeof(Work));
    conv_fwd(l, in, B, w, out, wk, 1);
    free(wk);
}
void orc_cnn_conv_wgrad(int l, const float* in, const float* dy, int B, float* grad) {
    Work* wk = (Work*)malloc(sizeof(Work));
    conv_wgrad(l, in, dy, B, grad, wk, 1);
    free(wk);
}
void orc_cnn_conv_dgrad(int l, const float* dy, const float* w, const float* act, int B, float* dx) {
    conv_dgrad(l, dy, w, act, B, dx, 1);
}
