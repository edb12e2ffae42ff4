// Host-only stand-in for libsmx.so (test infrastructure, never shipped): implements every
// entry point of include/smx.h on the CPU with no arithmetic, so the C++ engine (plan, stage
// trees, scheduler, event loop, checkpoint pool, spill tier, tuners) can be tested here without
// a GPU.  Linked only into tests/native/_stagemerge_stub*.so (paper_2006_11972_b200/build.py).
//
// A slot's "model state" is a 64-bit digest of the hp rows it has trained on, chained step by
// step; SAVE / LOAD / peer copies / spills move the digest like the real executor moves w | m.
// smx_eval reports metrics derived from it, so two executions record equal metrics exactly when
// they trained the same hp prefix -- the property the GPU kernels must have bitwise
// -- and a missing hp upload, a wrong LOAD or a lost checkpoint shows up as a
// metric conflict (plan.cpp:172-179) or an explicit error.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/smx.h"

namespace {

thread_local std::string g_err;

struct State {
    int64_t step = 0, offset = 0;
    uint64_t digest = 0;
};

uint64_t mix(uint64_t h, const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

constexpr uint64_t kInit = 0xcbf29ce484222325ull;
constexpr int64_t kPAlloc = 4;  // w[0..1] carry the digest bits through the spill tier

int err(int code, const std::string& m) {
    g_err = m;
    return code;
}

}  // namespace

struct smx_ctx {
    smx_model_desc d{};
    int S = 0, C = 0;
    std::vector<float> hp;  // S x max_steps x 4
    std::vector<char> hp_set;
    std::vector<State> slot, ck;
    std::vector<char> ck_valid;
    smx_stats stats{};
};

extern "C" {

const char* smx_last_error(void) { return g_err.c_str(); }
const char* smx_version(void) { return "smx host stub (tests only)"; }

int smx_open(const smx_model_desc* d, int, int n_slots, int n_ckpts, smx_ctx** out) {
    if (!d || !out || n_slots < 1 || n_ckpts < 0 || d->max_steps < 1) return err(SMX_ECONFIG, "bad open args");
    auto* c = new smx_ctx();
    c->d = *d;
    c->S = n_slots;
    c->C = n_ckpts;
    c->hp.assign(static_cast<size_t>(n_slots) * d->max_steps * SMX_HP_COLS, 0.f);
    c->hp_set.assign(static_cast<size_t>(n_slots) * d->max_steps, 0);
    c->slot.assign(static_cast<size_t>(n_slots), State{});
    c->ck.assign(static_cast<size_t>(n_ckpts), State{});
    c->ck_valid.assign(static_cast<size_t>(n_ckpts), 0);
    *out = c;
    return SMX_OK;
}

int smx_close(smx_ctx* c) {
    delete c;
    return SMX_OK;
}

int smx_param_count(const smx_ctx*, int64_t* p, int64_t* p_alloc) {
    if (p) *p = kPAlloc;
    if (p_alloc) *p_alloc = kPAlloc;
    return SMX_OK;
}

int smx_dataset_digest(smx_ctx*, uint64_t* out) {
    *out = 0;
    return SMX_OK;
}
int smx_dataset_upload(smx_ctx*, const float*, const int32_t*, const float*, const int32_t*) { return SMX_OK; }
int smx_dataset_read(smx_ctx*, float*, int32_t*, float*, int32_t*) { return SMX_OK; }
int smx_host_alloc(uint64_t bytes, void** out) {
    *out = std::malloc(bytes);
    return *out ? SMX_OK : err(SMX_EDEVICE, "malloc");
}
int smx_host_free(void* p) {
    std::free(p);
    return SMX_OK;
}

int smx_hp_upload(smx_ctx* c, int slot, int64_t step0, int64_t n, const float* hp) {
    if (slot < 0 || slot >= c->S) return err(SMX_ECONFIG, "slot out of range");
    if (step0 < 0 || n < 0 || step0 + n > c->d.max_steps) return err(SMX_ECONFIG, "hp rows exceed max_steps");
    for (int64_t i = 0; i < n; ++i) {
        const float bs = hp[i * SMX_HP_COLS + SMX_HP_BS];
        if (!(bs >= 1.0f) || bs > static_cast<float>(c->d.max_batch)) return err(SMX_ECONFIG, "batch size outside [1, max_batch]");
        const size_t r = static_cast<size_t>(slot) * c->d.max_steps + static_cast<size_t>(step0 + i);
        std::memcpy(&c->hp[r * SMX_HP_COLS], hp + i * SMX_HP_COLS, sizeof(float) * SMX_HP_COLS);
        c->hp_set[r] = 1;
    }
    return SMX_OK;
}

int smx_slot_init(smx_ctx* c, int slot) {
    if (slot < 0 || slot >= c->S) return err(SMX_ECONFIG, "slot out of range");
    c->slot[static_cast<size_t>(slot)] = State{0, 0, kInit};
    return SMX_OK;
}

int smx_slot_load(smx_ctx* c, int slot, int ckpt) {
    if (slot < 0 || slot >= c->S || ckpt < 0 || ckpt >= c->C) return err(SMX_ECONFIG, "index out of range");
    if (!c->ck_valid[static_cast<size_t>(ckpt)]) return err(SMX_EINTEGRITY, "load from empty checkpoint entry");
    c->slot[static_cast<size_t>(slot)] = c->ck[static_cast<size_t>(ckpt)];
    c->stats.forks += 1;
    return SMX_OK;
}

int smx_slot_save(smx_ctx* c, int slot, int ckpt) {
    if (slot < 0 || slot >= c->S || ckpt < 0 || ckpt >= c->C) return err(SMX_ECONFIG, "index out of range");
    c->ck[static_cast<size_t>(ckpt)] = c->slot[static_cast<size_t>(slot)];
    c->ck_valid[static_cast<size_t>(ckpt)] = 1;
    c->stats.forks += 1;
    return SMX_OK;
}

int smx_release_slot(smx_ctx* c, int slot) {
    if (slot < 0 || slot >= c->S) return err(SMX_ECONFIG, "slot out of range");
    c->slot[static_cast<size_t>(slot)] = State{-1, 0, 0};  // no state: train / eval fail until init / load
    return SMX_OK;
}

int smx_ckpt_free(smx_ctx* c, int ckpt) {
    if (ckpt < 0 || ckpt >= c->C) return err(SMX_ECONFIG, "checkpoint out of range");
    c->ck_valid[static_cast<size_t>(ckpt)] = 0;
    return SMX_OK;
}

int smx_ckpt_peer_copy(smx_ctx* dst, int dst_ckpt, smx_ctx* src, int src_ckpt) {
    if (dst_ckpt < 0 || dst_ckpt >= dst->C || src_ckpt < 0 || src_ckpt >= src->C) return err(SMX_ECONFIG, "index");
    if (!src->ck_valid[static_cast<size_t>(src_ckpt)]) return err(SMX_EINTEGRITY, "peer copy from empty entry");
    dst->ck[static_cast<size_t>(dst_ckpt)] = src->ck[static_cast<size_t>(src_ckpt)];
    dst->ck_valid[static_cast<size_t>(dst_ckpt)] = 1;
    dst->stats.forks += 1;
    return SMX_OK;
}

int smx_slot_state(smx_ctx* c, int slot, int64_t* step, int64_t* offset) {
    if (slot < 0 || slot >= c->S) return err(SMX_ECONFIG, "slot out of range");
    if (step) *step = c->slot[static_cast<size_t>(slot)].step;
    if (offset) *offset = c->slot[static_cast<size_t>(slot)].offset;
    return SMX_OK;
}

static void put_digest(const State& s, float* w, float* m) {
    if (w) {
        std::memset(w, 0, sizeof(float) * kPAlloc);
        std::memcpy(w, &s.digest, sizeof s.digest);
    }
    if (m) std::memset(m, 0, sizeof(float) * kPAlloc);
}

int smx_slot_read(smx_ctx* c, int slot, float* w, float* m) {
    if (slot < 0 || slot >= c->S) return err(SMX_ECONFIG, "slot out of range");
    put_digest(c->slot[static_cast<size_t>(slot)], w, m);
    return SMX_OK;
}

int smx_slot_write(smx_ctx* c, int slot, const float* w, const float*, int64_t step, int64_t offset) {
    if (slot < 0 || slot >= c->S) return err(SMX_ECONFIG, "slot out of range");
    State s{step, offset, 0};
    std::memcpy(&s.digest, w, sizeof s.digest);
    c->slot[static_cast<size_t>(slot)] = s;
    return SMX_OK;
}

int smx_ckpt_read(smx_ctx* c, int ckpt, float* w, float* m, int64_t* step, int64_t* offset) {
    if (ckpt < 0 || ckpt >= c->C) return err(SMX_ECONFIG, "checkpoint out of range");
    if (!c->ck_valid[static_cast<size_t>(ckpt)]) return err(SMX_EINTEGRITY, "read of empty checkpoint entry");
    const State& s = c->ck[static_cast<size_t>(ckpt)];
    put_digest(s, w, m);
    if (step) *step = s.step;
    if (offset) *offset = s.offset;
    return SMX_OK;
}

int smx_ckpt_write(smx_ctx* c, int ckpt, const float* w, const float*, int64_t step, int64_t offset) {
    if (ckpt < 0 || ckpt >= c->C) return err(SMX_ECONFIG, "checkpoint out of range");
    State s{step, offset, 0};
    std::memcpy(&s.digest, w, sizeof s.digest);
    c->ck[static_cast<size_t>(ckpt)] = s;
    c->ck_valid[static_cast<size_t>(ckpt)] = 1;
    return SMX_OK;
}

int smx_train(smx_ctx* c, int n_active, const int* slots, int n_steps) {
    if (n_active < 0 || n_steps < 0) return err(SMX_ECONFIG, "negative counts");
    std::vector<char> seen(static_cast<size_t>(c->S), 0);
    for (int i = 0; i < n_active; ++i) {
        const int s = slots[i];
        if (s < 0 || s >= c->S || seen[static_cast<size_t>(s)]) return err(SMX_ECONFIG, "bad slot list");
        seen[static_cast<size_t>(s)] = 1;
    }
    for (int k = 0; k < n_steps; ++k)
        for (int i = 0; i < n_active; ++i) {
            State& st = c->slot[static_cast<size_t>(slots[i])];
            if (st.step < 0) return err(SMX_ECONFIG, "slot has no state");
            if (st.step >= c->d.max_steps) return err(SMX_ECONFIG, "step beyond max_steps");
            const size_t r = static_cast<size_t>(slots[i]) * c->d.max_steps + static_cast<size_t>(st.step);
            if (!c->hp_set[r]) return err(SMX_EINTEGRITY, "no hp row uploaded for slot " + std::to_string(slots[i]) +
                                                          " step " + std::to_string(st.step));
            const float* row = &c->hp[r * SMX_HP_COLS];
            st.digest = mix(st.digest, row, sizeof(float) * SMX_HP_COLS);
            st.offset += static_cast<int64_t>(row[SMX_HP_BS]);
            st.step += 1;
        }
    c->stats.locksteps += n_steps;
    c->stats.stage_steps += static_cast<int64_t>(n_steps) * n_active;
    c->stats.launches += n_active ? n_steps : 0;
    return SMX_OK;
}

int smx_eval(smx_ctx* c, int n, const int* slots, double* out) {
    for (int i = 0; i < n; ++i) {
        if (slots[i] < 0 || slots[i] >= c->S) return err(SMX_ECONFIG, "slot out of range");
        const State& s = c->slot[static_cast<size_t>(slots[i])];
        if (s.step < 0) return err(SMX_ECONFIG, "eval of a slot with no state");
        const uint64_t h = mix(s.digest, &s.offset, sizeof s.offset);
        out[i * SMX_MET_COLS + SMX_MET_VAL_LOSS] = static_cast<double>(h >> 11) * 0x1p-53;
        out[i * SMX_MET_COLS + SMX_MET_VAL_ACC] = static_cast<double>(s.step);
    }
    return SMX_OK;
}

int smx_losses(smx_ctx* c, int slot, int64_t step0, int64_t n, float* out) {
    if (slot < 0 || slot >= c->S || step0 < 0 || n < 0 || step0 + n > c->d.max_steps) return err(SMX_ECONFIG, "range");
    std::memset(out, 0, sizeof(float) * static_cast<size_t>(n));
    return SMX_OK;
}

int smx_sync(smx_ctx*) { return SMX_OK; }
int smx_set_timing(smx_ctx*, int) { return SMX_OK; }
int smx_set_graphs(smx_ctx*, int) { return SMX_OK; }
int smx_get_stats(smx_ctx* c, smx_stats* out) {
    *out = c->stats;
    return SMX_OK;
}
int smx_reset_stats(smx_ctx* c) {
    c->stats = smx_stats{};
    return SMX_OK;
}
int smx_bench_kernel(smx_ctx*, int, int, int, double*) { return err(SMX_ECONFIG, "stub has no kernels"); }
int smx_bench_peer_copy(smx_ctx*, smx_ctx*, int, int, double*) { return err(SMX_ECONFIG, "stub has no kernels"); }
int smx_test_gemm(smx_ctx*, int, int, int, int, int, const float*, int, const float*, int, float*) {
    return err(SMX_ECONFIG, "stub has no kernels");
}

}  // extern "C"
