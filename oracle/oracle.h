/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the stage executor.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load liboracle.so, and only as the checker or the timed CPU baseline — never as a product
 * path.
 *
 * PARITY STATUS: the reference ships no training arithmetic at all (sim.cpp
 * is absent, the SPEC's TrainingOracle is synthetic).  The executor's
 * arithmetic is therefore *defined* by DESIGN.md §3 and restated here independently of the
 * CUDA code.  The training numerics are "parity unpinned" by the reference; what this oracle
 * pins is (1) bit-exactness of the GPU exact mode against an independent restatement and
 * (2) the tolerance of the tensor-core mode.  The hp values it consumes come from the product
 * host library, which is itself pinned against the compiled reference (oracle/_ref).
 */
#ifndef ORACLE_H_
#define ORACLE_H_

#include <stdint.h>

void orc_layout(int64_t* p_algo, int64_t* p_alloc, int64_t* off /* 7 offsets: W1 b1 W2 b2 W3 b3 end */);
float orc_exp(float x);
float orc_log(float x);
void orc_gen_dataset(uint64_t seed, int n_train, int max_batch, int n_val, float* x, int32_t* y, float* vx,
                     int32_t* vy);
uint64_t orc_fnv(const void* p, int64_t n, uint64_t h);
void orc_init(uint64_t seed, float* w, float* m);
/* Train one slot for n_steps from (step, offset); hp indexed by absolute step (4 cols).
 * loss_hist indexed by absolute step. */
int orc_train(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows, int n_steps,
              const float* x, const int32_t* y, int n_train, float* loss_hist);
/* Same for many independent slots, OpenMP across slots (the timed CPU baseline). */
int orc_train_many(int n_slots, float** w, float** m, int64_t* step, int64_t* offset, const float** hp,
                   int64_t hp_rows, int n_steps, const float* x, const int32_t* y, int n_train, float** loss_hist,
                   int threads);
void orc_eval(const float* w, const float* vx, const int32_t* vy, int n_val, double* out /* val_loss, val_acc */);
/* The same with every step (eval) split over `threads` OpenMP threads by independent outputs:
 * bitwise the single-thread result.  Used by the plan-driven CPU executor (oracle/cpu_executor.py). */
int orc_train_mt(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows, int n_steps,
                 const float* x, const int32_t* y, int n_train, float* loss_hist, int threads);
void orc_eval_mt(const float* w, const float* vx, const int32_t* vy, int n_val, double* out, int threads);

/* softmax-CE of one row of 10 logits (shared by both models) */
float orc_ce_row(const float* z, int y, float* dz, int* am);

/* ---- CNN model (oracle/cnn.c) ---------------------------------------- */
void orc_cnn_layout(int64_t* p_algo, int64_t* p_alloc, int64_t* off /* 9: W1 b1 W2 b2 W3 b3 W4 b4 end */);
void orc_cnn_gen_dataset(uint64_t seed, int n_train, int max_batch, int n_val, float* x, int32_t* y, float* vx,
                         int32_t* vy);
void orc_cnn_init(uint64_t seed, float* w, float* m);
int orc_cnn_train(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows, int n_steps,
                  const float* x, const int32_t* y, int n_train, float* loss_hist);
int orc_cnn_train_many(int n_slots, float** w, float** m, int64_t* step, int64_t* offset, const float** hp,
                       int64_t hp_rows, int n_steps, const float* x, const int32_t* y, int n_train, float** loss_hist,
                       int threads);
void orc_cnn_eval(const float* w, const float* vx, const int32_t* vy, int n_val, double* out);
int orc_cnn_train_mt(float* w, float* m, int64_t* step, int64_t* offset, const float* hp, int64_t hp_rows,
                     int n_steps, const float* x, const int32_t* y, int n_train, float* loss_hist, int threads);
void orc_cnn_eval_mt(const float* w, const float* vx, const int32_t* vy, int n_val, double* out, int threads);
void orc_cnn_conv_fwd(int l, const float* in, int B, const float* w, float* out);
void orc_cnn_conv_wgrad(int l, const float* in, const float* dy, int B, float* grad);
void orc_cnn_conv_dgrad(int l, const float* dy, const float* w, const float* act, int B, float* dx);

#endif
