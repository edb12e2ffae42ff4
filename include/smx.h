/*
 * smx.h — C ABI of the B200 stage executor (the drop-in boundary).
 *
 * The reference (Hippo / `stagemerge`) executes a stage in `worker_execute(assignment, cost,
 * oracle)` (reference SPEC.md:400-408), simulated there as `steps x sec/step`.  Behind that call
 * sit four things this ABI replaces:
 *
 *   reference interface                                     replaced by
 *   ------------------------------------------------------  ------------------------------------
 *   LOAD of the first stage's resume checkpoint              smx_slot_load / smx_slot_init
 *     (Assignment SPEC.md:315-318;           (kScratch = seeded init,
 *      ResumePoint stage_tree.hpp:21-26)                       stage_tree.hpp:21, :33-34)
 *   TRAIN `steps` under the node's hp values                 smx_hp_upload + smx_train
 *     (values from SearchPlan::value_at
 *      plan.cpp:278-288 -> hpseq.cpp:315-370)
 *   EVAL at declared steps -> MetricRecord                   smx_eval
 *     (TrainingOracle SPEC.md:378-381;
 *      MetricRecord types.hpp:18)
 *   SAVE at stage / request ends -> CkptHandle               smx_slot_save (+ smx_ckpt_* spill)
 *     (record_checkpoint plan.cpp:153-164,
 *      CkptHandle types.hpp:20-21)
 *   cross-worker checkpoint sharing (GlusterFS in the        smx_ckpt_peer_copy (NVLink P2P)
 *     paper)
 *
 * Conventions (mirroring types.hpp:31-43 and SPEC.md:628):
 *   every entry point returns SMX_OK (0), SMX_ECONFIG (1, the host adapter rethrows
 *   ConfigError), SMX_EINTEGRITY (2, rethrows IntegrityError — e.g. loading an empty checkpoint,
 *   the "missing checkpoint" fail-fast of SPEC.md:404) or SMX_EDEVICE (3, CUDA fault).
 *   smx_last_error() returns a thread-local message for the last failure.
 *   Only POD and integer handles cross; host buffers are copied before the call returns
 *   (or, for the async entry points, before the next call on the same context).
 *   One context == one GPU; all calls on a context come from one thread (the reference's
 *   single-owner event loop).  Work is enqueued on the context's stream;
 *   smx_eval / smx_losses / smx_sync / smx_slot_read are the synchronisation points.
 *
 * Numerics: the training arithmetic of one stage-step is a pure function of
 * (w, m, data offset, hp row), independent of which other slots share the launch, so merged
 * (STAGE) and unmerged (TRIAL) execution produce bitwise identical metrics.
 * SMX_GEMM_EXACT reproduces the CPU oracle (oracle/trainer.c) bit for bit;
 * SMX_GEMM_TC runs the GEMMs on tcgen05 tensor cores (3xTF32) within the tolerance stated
 * in DESIGN.md.
 */
#ifndef SMX_H_
#define SMX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMX_OK 0
#define SMX_ECONFIG 1
#define SMX_EINTEGRITY 2
#define SMX_EDEVICE 3

#define SMX_MODEL_MLP 0 /* 784-256-256-10, ReLU, softmax-CE */
#define SMX_MODEL_CNN 1 /* 3x32x32: conv3x3 3->32 s1, 32->64 s2, 64->128 s2, ReLU, GAP, FC 128->10
                           (DESIGN.md §3b); inputs NHWC 32x32x4 (channel 3 = 0) */

#define SMX_GEMM_EXACT 0 /* SIMT fp32, fixed fmaf order: bit-exact with the CPU oracle */
#define SMX_GEMM_TC 1    /* tcgen05 kind::tf32, 3xTF32 split: fp32-level accuracy */

/* hp row layout in smx_hp_upload: one row per absolute training step. */
#define SMX_HP_LR 0
#define SMX_HP_MOMENTUM 1
#define SMX_HP_WD 2
#define SMX_HP_BS 3
#define SMX_HP_COLS 4

/* metrics written by smx_eval, per slot */
#define SMX_MET_VAL_LOSS 0
#define SMX_MET_VAL_ACC 1
#define SMX_MET_COLS 2

typedef struct smx_ctx smx_ctx;

typedef struct smx_model_desc {
    int32_t model;     /* SMX_MODEL_* */
    int32_t max_batch; /* largest bs any step may use (<= 256) */
    int32_t n_train;   /* synthetic training samples, power of two */
    int32_t n_val;     /* validation samples, multiple of 128 */
    int32_t max_steps; /* hp-table / loss-history capacity per slot (absolute steps) */
    int32_t gemm_mode; /* SMX_GEMM_* */
    uint64_t seed;     /* data, teacher and init seed (identical on every GPU) */
} smx_model_desc;

typedef struct smx_stats {
    int64_t launches;      /* kernels launched by this context since open / last reset */
    int64_t locksteps;     /* grouped training steps executed */
    int64_t stage_steps;   /* (slot, step) updates executed */
    int64_t forks;         /* checkpoint copies (save + load + peer) */
    double update_ms;      /* summed CUDA-event time of the K5 update kernel (timing mode only) */
    int64_t update_launches;
    double gemm_ms;        /* summed CUDA-event time of the GEMM kernels (timing mode only) */
    int64_t gemm_launches;
    double fork_ms;        /* summed CUDA-event time of the K6 fork kernel (timing mode only) */
    int64_t fork_launches;
    double lockstep_ms;    /* summed CUDA-event time of whole locksteps (timing mode only) */
} smx_stats;

/* --- lifetime ------------------------------------------------------------------------- */
int smx_open(const smx_model_desc* desc, int device, int n_slots, int n_ckpts, smx_ctx** out);
int smx_close(smx_ctx* ctx);
/* P = algorithmic parameter count; p_alloc = floats per parameter vector in HBM (padded). */
int smx_param_count(const smx_ctx* ctx, int64_t* p, int64_t* p_alloc);
/* FNV-1a over the bytes of the training/validation sets and labels. */
int smx_dataset_digest(smx_ctx* ctx, uint64_t* out);
/* Replace the synthetic dataset with host data: x (n_train + max_batch) x d_in fp32 (rows past
 * n_train repeat the first max_batch rows; d_in = 784 for the MLP, 4096 = 32x32x4 for the CNN),
 * y int32 labels, vx n_val x d_in, vy.  Host->device
 * copies on the context stream; pinned buffers (smx_host_alloc) make them DMA-direct. */
int smx_dataset_upload(smx_ctx* ctx, const float* x, const int32_t* y, const float* vx, const int32_t* vy);
/* Device -> host copy of the context's dataset in the smx_dataset_upload layout (e.g. to stage
 * the synthetic set in pinned memory for the end-to-end path); synchronous. */
int smx_dataset_read(smx_ctx* ctx, float* x, int32_t* y, float* vx, int32_t* vy);
/* Page-locked host buffers for the e2e path. */
int smx_host_alloc(uint64_t bytes, void** out);
int smx_host_free(void* p);

/* --- per-slot state (the model/optimizer state store) ------------------------------- */
/* hp rows [step0, step0+n) for `slot`, each SMX_HP_COLS floats (host-computed values). */
int smx_hp_upload(smx_ctx* ctx, int slot, int64_t step0, int64_t n, const float* hp);
int smx_slot_init(smx_ctx* ctx, int slot);                /* kScratch: seeded init, m=0, step=0 */
int smx_slot_load(smx_ctx* ctx, int slot, int ckpt);      /* LOAD: pool -> slot (HBM copy) */
int smx_slot_save(smx_ctx* ctx, int slot, int ckpt);      /* SAVE: slot -> pool (HBM copy) */
int smx_ckpt_free(smx_ctx* ctx, int ckpt);                /* GC: entry becomes empty */
/* STOP / cancel_trial (reference plan.cpp:204-225): the slot's state is abandoned; it must be
 * re-initialised (smx_slot_init / _load / _write) before it trains or evaluates again. */
int smx_release_slot(smx_ctx* ctx, int slot);
int smx_ckpt_peer_copy(smx_ctx* dst, int dst_ckpt, smx_ctx* src, int src_ckpt); /* NVLink P2P */
int smx_slot_state(smx_ctx* ctx, int slot, int64_t* step, int64_t* offset);
int smx_slot_read(smx_ctx* ctx, int slot, float* w, float* m);  /* p_alloc floats each */
int smx_slot_write(smx_ctx* ctx, int slot, const float* w, const float* m, int64_t step,
                   int64_t offset);
int smx_ckpt_read(smx_ctx* ctx, int ckpt, float* w, float* m, int64_t* step, int64_t* offset);
int smx_ckpt_write(smx_ctx* ctx, int ckpt, const float* w, const float* m, int64_t step,
                   int64_t offset);

/* --- execution ------------------------------------------------------------------------ */
/* n_steps grouped locksteps over `slots`; every slot advances its own step and data offset
 * and reads its own hp row.  Asynchronous. */
int smx_train(smx_ctx* ctx, int n_active, const int* slots, int n_steps);
/* Deterministic validation metrics at each slot's current state; synchronous.
 * out: n x SMX_MET_COLS doubles. */
int smx_eval(smx_ctx* ctx, int n, const int* slots, double* out);
/* Training loss recorded at steps [step0, step0+n) of `slot`; synchronous. */
int smx_losses(smx_ctx* ctx, int slot, int64_t step0, int64_t n, float* out);
int smx_sync(smx_ctx* ctx);

/* --- measurement ---------------------------------------------------------------------- */
int smx_set_timing(smx_ctx* ctx, int enabled); /* CUDA events around every kernel class */
int smx_set_graphs(smx_ctx* ctx, int enabled); /* capture lockstep sequences in CUDA graphs */
int smx_get_stats(smx_ctx* ctx, smx_stats* out);
int smx_reset_stats(smx_ctx* ctx);
/* Standalone launches of one kernel class for roofline measurement: kind 0 = K5 update over
 * `n` slots, 1 = K6 fork copy of `n` checkpoints, 2 = the layer-1 forward GEMM over `n` slots,
 * 3 = the layer-1 weight-gradient GEMM over `n` slots (both at the slots' current batch size);
 * for the CNN, 2 = the conv2 forward implicit GEMM and 3 = the conv2 weight-gradient implicit
 * GEMM (tensor-core mode: the split GEMM alone; exact mode: the SIMT kernel); 4 / 5 = the conv2 /
 * conv3 input gradient, 6 = the conv3 forward, 7 = the conv3 weight gradient (tensor-core mode: the
 * split GEMM alone; exact mode: with its reduction),
 * 8 = the conv1 weight gradient (with its reduction), 9 = the conv1 forward.
 * Returns mean CUDA-event ms per launch. */
int smx_bench_kernel(smx_ctx* ctx, int kind, int n, int reps, double* ms_per_launch);
/* K7 measurement: n <= 16 checkpoint entries 0..n-1 of `src` copied to entries 0..n-1 of `dst` per
 * launch (the fork kernel on dst reading src's pool through peer loads; a staged runtime peer copy
 * without P2P access), `reps` launches timed with CUDA events on dst's stream.  Returns mean ms
 * per entry copied. */
int smx_bench_peer_copy(smx_ctx* dst, smx_ctx* src, int n, int reps, double* ms_per_copy);

/* Test hook: one ungrouped GEMM C[M x N] = A op B on the device through the executor's GEMM
 * kernels (gemm_mode of the context): am/bm = 0 when A(m,k) = A[m*lda+k] / B(n,k) = B[n*ldb+k],
 * 1 when A(m,k) = A[k*lda+m] / B(n,k) = B[k*ldb+n].  Host buffers in and out; synchronous. */
int smx_test_gemm(smx_ctx* ctx, int am, int bm, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                  float* C);

const char* smx_last_error(void);
const char* smx_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SMX_H_ */
