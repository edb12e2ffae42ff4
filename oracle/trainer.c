/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle of the stage executor (see oracle.h for the rules and
 * the parity status).
 *
 * This file restates DESIGN.md §3 ("executor arithmetic") in plain C, written independently of
 * paper_2006_11972_b200/csrc.  Every rounding is explicit: the file is compiled with
 * -ffp-contract=off, products/sums are single IEEE operations, and fused multiply-adds appear
 * only where DESIGN.md §3 specifies them (fmaf).  Loops are arranged so every dot product is
 * one fmaf chain in ascending reduction index starting from +0 — the order the GPU exact mode
 * uses — while still vectorising across independent outputs.
 *
 * Reference anchors: the executor semantics it realises are worker_execute (reference
 * LOAD / TRAIN / EVAL / SAVE), the TrainingOracle invariant that metrics
 * depend only on the hp value prefix, the PyTorch SGD rule of the
 * paper's stack and the data-offset-in-checkpoint rule
 * (PAPER.md:400-401).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

enum { D0 = 784, HID = 256, NC = 10, NCP = 16, MAXB = 256 };

/* parameter vector layout (floats) */
#define O_W1 0L
#define O_B1 (O_W1 + (long)HID * D0)
#define O_W2 (O_B1 + HID)
#define O_B2 (O_W2 + (long)HID * HID)
#define O_W3 (O_B2 + HID)
#define O_B3 (O_W3 + (long)NCP * HID)
#define O_END (O_B3 + NCP)
#define P_ALLOC ((O_END + 63) / 64 * 64)
#define P_ALGO ((long)HID * D0 + HID + (long)HID * HID + HID + (long)NC * HID + NC)

void orc_layout(int64_t* p_algo, int64_t* p_alloc, int64_t* off) {
    if (p_algo) *p_algo = P_ALGO;
    if (p_alloc) *p_alloc = P_ALLOC;
    if (off) {
        off[0] = O_W1; off[1] = O_B1; off[2] = O_W2; off[3] = O_B2;
        off[4] = O_W3; off[5] = O_B3; off[6] = O_END;
    }
}

/* ---- hashing ------------------------------------------------------------------------ */
static uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t key4(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
    return splitmix(seed ^ splitmix((stream << 56) ^ (i << 20) ^ j));
}

uint64_t orc_fnv(const void* p, int64_t n, uint64_t h) {
    const unsigned char* b = (const unsigned char*)p;
    for (int64_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* ---- exp / log ------------------------------------------------------ */
static float f_of_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bits_of_f(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

float orc_exp(float x) {
    if (x < -87.0f) return 0.0f;
    const float n = rintf(x * 1.44269504f);
    float r = fmaf(-n, 0.693145751953125f, x);
    r = fmaf(-n, 1.42860682e-06f, r);
    static const float c[8] = {1.98412698e-04f, 1.38888889e-03f, 8.33333333e-03f, 4.16666667e-02f,
                               1.66666667e-01f, 0.5f, 1.0f, 1.0f};
    float p = c[0];
    for (int i = 1; i < 8; ++i) p = fmaf(p, r, c[i]);
    const int e = (int)n;
    return p * f_of_bits((uint32_t)(e + 127) << 23);
}

float orc_log(float x) {
    const uint32_t u = bits_of_f(x);
    int e = (int)(u >> 23) - 127;
    float f = f_of_bits((u & 0x7FFFFFu) | 0x3F800000u);
    if (f > 1.41421356f) {
        f = f * 0.5f;
        e += 1;
    }
    const float s = (f - 1.0f) / (f + 1.0f);
    const float s2 = s * s;
    static const float c[6] = {9.09090909e-02f, 1.11111111e-01f, 1.42857143e-01f, 2.00000000e-01f,
                               3.33333333e-01f, 1.0f};
    float q = c[0];
    for (int i = 1; i < 6; ++i) q = fmaf(q, s2, c[i]);
    const float lf = (s + s) * q;
    return fmaf((float)e, 0.693147182f, lf);
}

/* Row loss of softmax-CE over NC logits; writes p - onehot (unscaled) to dz when non-NULL. */
static float ce_row(const float* z, int y, float* dz, int* am) {
    float mx = z[0];
    int best = 0;
    for (int c = 1; c < NC; ++c)
        if (z[c] > mx) { mx = z[c]; best = c; }
    float e[NC], s = 0.0f;
    for (int c = 0; c < NC; ++c) {
        e[c] = orc_exp(z[c] - mx);
        s = s + e[c];
    }
    if (dz)
        for (int c = 0; c < NC; ++c) dz[c] = e[c] / s - (c == y ? 1.0f : 0.0f);
    if (am) *am = best;
    return orc_log(s) - (z[y] - mx);
}

float orc_ce_row(const float* z, int y, float* dz, int* am) { return ce_row(z, y, dz, am); }

/* ---- data / init ----------------------------------------------- */
static void gen_rows(uint64_t seed, uint64_t stream, long rows, long n, float* x, int32_t* y) {
    signed char T[D0][NC];
    for (int j = 0; j < D0; ++j)
        for (int c = 0; c < NC; ++c) T[j][c] = (signed char)((int)((key4(seed, 3, (uint64_t)c, (uint64_t)j) >> 8) & 7) - 4);
#pragma omp parallel for schedule(static)
    for (long r = 0; r < rows; ++r) {
        int acc[NC] = {0};
        for (int j = 0; j < D0; ++j) {
            const int k = (int)(key4(seed, stream, (uint64_t)(r % n), (uint64_t)j) & 0xFF) - 128;
            x[r * D0 + j] = (float)k * 0.0078125f;
            for (int c = 0; c < NC; ++c) acc[c] += k * (int)T[j][c];
        }
        int best = 0;
        for (int c = 1; c < NC; ++c)
            if (acc[c] > acc[best]) best = c;
        y[r] = best;
    }
}

void orc_gen_dataset(uint64_t seed, int n_train, int max_batch, int n_val, float* x, int32_t* y, float* vx,
                     int32_t* vy) {
    gen_rows(seed, 1, (long)n_train + max_batch, n_train, x, y);
    gen_rows(seed, 2, n_val, n_val, vx, vy);
}

void orc_init(uint64_t seed, float* w, float* m) {
    const int fan[4] = {0, D0, HID, HID};
    const long base[4] = {0, O_W1, O_W2, O_W3};
    const int rows[4] = {0, HID, HID, NC};
    memset(w, 0, sizeof(float) * P_ALLOC);
    memset(m, 0, sizeof(float) * P_ALLOC);
    for (int l = 1; l <= 3; ++l) {
        const float sc = (float)sqrt(6.0 / (double)fan[l]) * (1.0f / 8388608.0f);
        for (int o = 0; o < rows[l]; ++o)
            for (int i = 0; i < fan[l]; ++i) {
                const uint64_t h = key4(seed, 4, ((uint64_t)l << 16) | (uint64_t)o, (uint64_t)i);
                const int s = (int)((h >> 40) & 0xFFFFFF) - 8388608;
                w[base[l] + (long)o * fan[l] + i] = (float)s * sc;
            }
    }
}

/* ---- one training step --------------------------------------------- */
typedef struct {
    float h1[MAXB * HID], h2[MAXB * HID], z[MAXB * NCP], dz[MAXB * NCP], dh2[MAXB * HID], dh1[MAXB * HID];
    float wt1[D0 * HID], wt2[HID * HID], wt3[HID * NCP];
    float acc[D0];
    float g[P_ALLOC];
} Work;

/* out[r][n] = epi(sum_k a[r][k] * wt[k][n]) ; wt is W transposed ([K][N]) */
/* nt > 1 (here and below): independent outputs split over OpenMP threads, every output still one
 * sequential chain -- bitwise the nt == 1 result (tested). */
static void fwd_layer(const float* restrict a, int B, int K, const float* restrict wt, int N,
                      const float* restrict bias, int relu, float* restrict out, int nt) {
    (void)nt;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (int r = 0; r < B; ++r) {
        float acc[HID > NCP ? HID : NCP];
        for (int n = 0; n < N; ++n) acc[n] = 0.0f;
        for (int k = 0; k < K; ++k) {
            const float av = a[(long)r * K + k];
            const float* restrict wk = wt + (long)k * N;
            for (int n = 0; n < N; ++n) acc[n] = fmaf(av, wk[n], acc[n]);
        }
        for (int n = 0; n < N; ++n) {
            float v = acc[n] + bias[n];
            if (relu) v = v > 0.0f ? v : 0.0f;
            out[(long)r * N + n] = v;
        }
    }
}

static void transpose(const float* restrict w, int rows, int cols, float* restrict wt) {
    for (int o = 0; o < rows; ++o)
        for (int i = 0; i < cols; ++i) wt[(long)i * rows + o] = w[(long)o * cols + i];
}

/* gw[o][k] = sum_r dy[r][o] * a[r][k] ; gb[o] = sum_r dy[r][o]  (r ascending) */
static void wgrad(const float* restrict dy, int ldy, int O, const float* restrict a, int K, int B,
                  float* restrict gw, float* restrict gb, int nt) {
    (void)nt;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (int o = 0; o < O; ++o) {
        float acc[D0];
        for (int k = 0; k < K; ++k) acc[k] = 0.0f;
        float sb = 0.0f;
        for (int r = 0; r < B; ++r) {
            const float d = dy[(long)r * ldy + o];
            const float* restrict ar = a + (long)r * K;
            for (int k = 0; k < K; ++k) acc[k] = fmaf(d, ar[k], acc[k]);
            sb = sb + d;
        }
        memcpy(gw + (long)o * K, acc, sizeof(float) * K);
        gb[o] = sb;
    }
}

/* dx[r][k] = (act[r][k] > 0) ? sum_o dy[r][o] * w[o][k] : 0   (o ascending) */
static void dgrad(const float* restrict dy, int ldy, int O, const float* restrict w, int K, int B,
                  const float* restrict act, float* restrict dx, int nt) {
    (void)nt;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (int r = 0; r < B; ++r) {
        float acc[HID];
        for (int k = 0; k < K; ++k) acc[k] = 0.0f;
        for (int o = 0; o < O; ++o) {
            const float d = dy[(long)r * ldy + o];
            const float* restrict wo = w + (long)o * K;
            for (int k = 0; k < K; ++k) acc[k] = fmaf(d, wo[k], acc[k]);
        }
        for (int k = 0; k < K; ++k) dx[(long)r * K + k] = act[(long)r * K + k] > 0.0f ? acc[k] : 0.0f;
    }
}

static float train_step(float* restrict w, float* restrict m, const float* hp, const float* x, const int32_t* y,
                        Work* wk, int nt) {
    const int B = (int)hp[3];
    /* forward */
    transpose(w + O_W1, HID, D0, wk->wt1);
    transpose(w + O_W2, HID, HID, wk->wt2);
    transpose(w + O_W3, NCP, HID, wk->wt3);
    fwd_layer(x, B, D0, wk->wt1, HID, w + O_B1, 1, wk->h1, nt);
    fwd_layer(wk->h1, B, HID, wk->wt2, HID, w + O_B2, 1, wk->h2, nt);
    fwd_layer(wk->h2, B, HID, wk->wt3, NCP, w + O_B3, 0, wk->z, nt);
    /* loss */
    float lsum = 0.0f;
    const float fb = (float)B;
    for (int r = 0; r < B; ++r) {
        float d[NC];
        lsum = lsum + ce_row(wk->z + (long)r * NCP, y[r], d, NULL);
        for (int c = 0; c < NC; ++c) wk->dz[(long)r * NCP + c] = d[c] / fb;
        for (int c = NC; c < NCP; ++c) wk->dz[(long)r * NCP + c] = 0.0f;
    }
    /* backward */
    memset(wk->g, 0, sizeof wk->g);
    wgrad(wk->dz, NCP, NCP, wk->h2, HID, B, wk->g + O_W3, wk->g + O_B3, nt);
    dgrad(wk->dz, NCP, NCP, w + O_W3, HID, B, wk->h2, wk->dh2, nt);
    wgrad(wk->dh2, HID, HID, wk->h1, HID, B, wk->g + O_W2, wk->g + O_B2, nt);
    dgrad(wk->dh2, HID, HID, w + O_W2, HID, B, wk->h1, wk->dh1, nt);
    wgrad(wk->dh1, HID, HID, x, D0, B, wk->g + O_W1, wk->g + O_B1, nt);
    /* K5: g' = fma(wd, w, g); m = fma(mu, m, g'); w = fma(-lr, m, w) */
    const float nlr = -hp[0], mu = hp[1], wd = hp[2];
    const float* restrict g = wk->g;
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
    for (long i = 0; i < P_ALLOC; ++i) {
        const float mv = fmaf(mu, m[i], fmaf(wd, w[i], g[i]));
        m[i] = mv;
        w[i] = fmaf(nlr, mv, w[i]);
    }
    return lsum / fb;
}

static int train_slot(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows,
                      int n_steps, const float* x, const int32_t* y, int n_train, float* loss_hist, Work* wk, int nt) {
    for (int i = 0; i < n_steps; ++i) {
        const int64_t s = *step;
        if (s < 0 || s >= hp_rows) return 1;
        const float* row = hp + s * 4;
        const long off = (long)(*offset & (int64_t)(n_train - 1));
        const float l = train_step(w, m, row, x + off * D0, y + off, wk, nt);
        if (loss_hist) loss_hist[s] = l;
        *step = s + 1;
        *offset += (int64_t)row[3];
    }
    return 0;
}

int orc_train(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows, int n_steps,
              const float* x, const int32_t* y, int n_train, float* loss_hist) {
    Work* wk = (Work*)malloc(sizeof(Work));
    if (!wk) return 2;
    const int rc = train_slot(w, m, step, offset, hp, hp_rows, n_steps, x, y, n_train, loss_hist, wk, 1);
    free(wk);
    return rc;
}

int orc_train_mt(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows, int n_steps,
                 const float* x, const int32_t* y, int n_train, float* loss_hist, int threads) {
    Work* wk = (Work*)malloc(sizeof(Work));
    if (!wk) return 2;
    const int rc = train_slot(w, m, step, offset, hp, hp_rows, n_steps, x, y, n_train, loss_hist, wk,
                              threads > 1 ? threads : 1);
    free(wk);
    return rc;
}

int orc_train_many(int n_slots, float** w, float** m, int64_t* step, int64_t* offset, const float** hp,
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
            rc |= wk ? train_slot(w[s], m[s], &step[s], &offset[s], hp[s], hp_rows, n_steps, x, y, n_train,
                                  loss_hist ? loss_hist[s] : NULL, wk, 1)
                     : 2;
        free(wk);
    }
    return rc;
}

/* ---- eval ----------------------------------------------------------- */
void orc_eval_mt(const float* w, const float* vx, const int32_t* vy, int n_val, double* out, int nt);

void orc_eval(const float* w, const float* vx, const int32_t* vy, int n_val, double* out) {
    orc_eval_mt(w, vx, vy, n_val, out, 1);
}

void orc_eval_mt(const float* w, const float* vx, const int32_t* vy, int n_val, double* out, int nt) {
    if (nt < 1) nt = 1;
    Work* wk = (Work*)malloc(sizeof(Work));
    float* loss = (float*)malloc(sizeof(float) * (size_t)n_val);
    transpose(w + O_W1, HID, D0, wk->wt1);
    transpose(w + O_W2, HID, HID, wk->wt2);
    transpose(w + O_W3, NCP, HID, wk->wt3);
    long correct = 0;
    for (int r0 = 0; r0 < n_val; r0 += MAXB) {
        const int B = n_val - r0 < MAXB ? n_val - r0 : MAXB;
        fwd_layer(vx + (long)r0 * D0, B, D0, wk->wt1, HID, w + O_B1, 1, wk->h1, nt);
        fwd_layer(wk->h1, B, HID, wk->wt2, HID, w + O_B2, 1, wk->h2, nt);
        fwd_layer(wk->h2, B, HID, wk->wt3, NCP, w + O_B3, 0, wk->z, nt);
        for (int r = 0; r < B; ++r) {
            int am = 0;
            loss[r0 + r] = ce_row(wk->z + (long)r * NCP, vy[r0 + r], NULL, &am);
            correct += (am == vy[r0 + r]);
        }
    }
    /* 32 lane partials of stride-32 sequential sums, then a fixed halving tree */
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
