// The engine: deterministic lockstep event loop over the smx executor (see engine.hpp).
#include "stagemerge/engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "smx.h"
#include "stagemerge/partition.hpp"

namespace stagemerge {

namespace {

void smx_ok(int rc, const char* what) {
    if (rc == SMX_OK) return;
    const std::string msg = std::string(what) + ": " + smx_last_error();
    if (rc == SMX_ECONFIG) throw ConfigError(msg);
    if (rc == SMX_EINTEGRITY) throw IntegrityError(msg);
    throw std::runtime_error("device error: " + msg);
}

std::string hex16(std::uint64_t v) {
    char b[20];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
    return b;
}

constexpr const char* kTrialHp = "__trial";  // TRIAL mode: a per-trial constant hp defeats merging

}  // namespace

struct Engine::Gpu {
    int device = 0;
    smx_ctx* ctx = nullptr;
    std::vector<int> free_entries;
    std::map<CkptHandle, int> entry_of;  // checkpoints resident in this GPU's pool
    std::vector<CkptHandle> handle_of;   // entry -> handle ("" = free)
    std::vector<std::uint64_t> last_use; // LRU clock per entry
};

struct Engine::Worker {
    int id = 0, gpu = 0, slot = 0;
    bool busy = false;
    Assignment a;
    std::size_t cur = 0;
    StepCount remaining = 0;
    double cost_us = 0;  // cost model's us per step of the current stage
};

Engine::Engine(CompatKey key, EngineOptions opts) : key_(std::move(key)), opts_(std::move(opts)) {
    if (opts_.devices.empty()) throw ConfigError("engine needs at least one device");
    if (opts_.slots_per_gpu < 1 || opts_.ckpts_per_gpu < 1) throw ConfigError("bad slot / checkpoint counts");
    if (opts_.trial_mode) {
        key_.hp_set.push_back(kTrialHp);
        std::sort(key_.hp_set.begin(), key_.hp_set.end());
    }
    plan_ = std::make_unique<SearchPlan>(key_);
    if (key_.model != "mlp" && key_.model != "cnn")
        throw ConfigError("executor has no model '" + key_.model + "' (supported: mlp, cnn)");
    const int model = key_.model == "cnn" ? SMX_MODEL_CNN : SMX_MODEL_MLP;
    d_in_ = model == SMX_MODEL_CNN ? 32 * 32 * 4 : 784;
    smx_model_desc d{model, opts_.max_batch, opts_.n_train, opts_.n_val, opts_.max_steps, opts_.gemm_mode,
                     opts_.seed};
    for (int dev : opts_.devices) {
        auto g = std::make_unique<Gpu>();
        g->device = dev;
        smx_ok(smx_open(&d, dev, opts_.slots_per_gpu, opts_.ckpts_per_gpu, &g->ctx), "smx_open");
        smx_set_graphs(g->ctx, opts_.use_graphs ? 1 : 0);
        smx_param_count(g->ctx, nullptr, &p_alloc_);
        g->handle_of.assign(static_cast<std::size_t>(opts_.ckpts_per_gpu), "");
        g->last_use.assign(static_cast<std::size_t>(opts_.ckpts_per_gpu), 0);
        for (int e = opts_.ckpts_per_gpu - 1; e >= 0; --e) g->free_entries.push_back(e);
        gpus_.push_back(std::move(g));
    }
    // worker w -> GPU w / S, slot w % S; with several GPUs, paths go to the GPU their nodes are
    // placed on (place_nodes, schedule_placed)
    const int G = static_cast<int>(gpus_.size());
    for (int w = 0; w < G * opts_.slots_per_gpu; ++w) {
        auto wk = std::make_unique<Worker>();
        wk->id = w;
        wk->gpu = w / opts_.slots_per_gpu;
        wk->slot = w % opts_.slots_per_gpu;
        workers_.push_back(std::move(wk));
    }
}

Engine::~Engine() {
    for (auto& g : gpus_)
        if (g->ctx) smx_close(g->ctx);
}

std::vector<smx_ctx*> Engine::contexts() const {
    std::vector<smx_ctx*> v;
    for (const auto& g : gpus_) v.push_back(g->ctx);
    return v;
}

void Engine::reset() {
    for (auto& w : workers_)
        if (w->busy) throw IntegrityError("reset while workers are busy");
    plan_ = std::make_unique<SearchPlan>(key_);
    for (auto& g : gpus_) {
        g->entry_of.clear();
        g->free_entries.clear();
        std::fill(g->last_use.begin(), g->last_use.end(), 0);
        for (int e = opts_.ckpts_per_gpu - 1; e >= 0; --e) {
            g->handle_of[static_cast<std::size_t>(e)].clear();
            g->free_entries.push_back(e);
            smx_ckpt_free(g->ctx, e);
        }
        smx_reset_stats(g->ctx);
    }
    trial_index_.clear();
    trial_cfg_.clear();
    reached_.clear();
    spilled_.clear();
    root_owner_.clear();
    stats_ = EngineStats{};
    next_assignment_ = 0;
    trace_.clear();
    clock_ = 0;
    stopped_.clear();
}

void Engine::emit(int worker, const char* kind, NodeId node, StepCount start, StepCount end, std::string detail) {
    trace_.push_back(TraceEvent{clock_, worker, kind, node, start, end, std::move(detail)});
}

void Engine::upload_dataset(const float* x, const std::int32_t* y, const float* vx, const std::int32_t* vy) {
    for (auto& g : gpus_) smx_ok(smx_dataset_upload(g->ctx, x, y, vx, vy), "smx_dataset_upload");
    const std::int64_t rows = static_cast<std::int64_t>(opts_.n_train) + opts_.max_batch;
    stats_.h2d_bytes += static_cast<std::int64_t>(gpus_.size()) *
                        (rows * d_in_ * 4 + rows * 4 + static_cast<std::int64_t>(opts_.n_val) * (d_in_ * 4 + 4));
}

std::uint64_t Engine::dataset_digest() {
    std::uint64_t h = 0;
    smx_ok(smx_dataset_digest(gpus_.front()->ctx, &h), "smx_dataset_digest");
    return h;
}

InsertOutcome Engine::submit(const TrialRequest& in) {
    TrialRequest req = in;
    if (opts_.trial_mode) {
        HpFunction tag;
        tag.params["value"] = Rational(static_cast<std::int64_t>(in.study) * 1000003 + in.trial + 1);
        req.config.sequences[kTrialHp] = make_sequence(kTrialHp, tag, req.config.total_steps);
    }
    if (req.config.total_steps > opts_.max_steps)
        throw ConfigError("trial longer than the executor's max_steps (" + std::to_string(opts_.max_steps) + ")");
    InsertOutcome out = plan_->insert_trial(req);
    const TrialRef t{in.study, in.trial};
    stopped_.erase(t);
    trial_index_[t] = {req.config.total_steps, out.node};
    trial_cfg_[t] = in.config;
    if (out.kind == InsertOutcome::Kind::kImmediate) credit(t, req.config.total_steps);
    return out;
}

void Engine::credit(const TrialRef& t, StepCount end) {
    StepCount& r = reached_[t];
    if (end > r) {
        stats_.trial_steps += end - r;
        r = end;
    }
}

bool Engine::cancel(const TrialRef& t) {
    stopped_.insert(t);
    const bool changed = plan_->cancel_trial(t);
    if (changed) release_orphans();
    return changed;
}

void Engine::release_orphans() {
    std::set<RequestId> live;
    for (const PendingRequest& p : plan_->pending_requests()) live.insert(p.id);
    for (auto& w : workers_) {
        if (!w->busy) continue;
        // one past the last stage (from the current one) that still serves a pending request
        std::size_t keep = w->cur;
        for (std::size_t i = w->a.stages.size(); i-- > w->cur;) {
            const auto& sv = w->a.stages[i].serves;
            if (std::any_of(sv.begin(), sv.end(), [&](RequestId r) { return live.count(r) > 0; })) {
                keep = i + 1;
                break;
            }
        }
        if (keep == w->cur) {
            smx_ok(smx_release_slot(gpus_[static_cast<std::size_t>(w->gpu)]->ctx, w->slot), "smx_release_slot");
            w->busy = false;
            w->remaining = 0;
            stats_.releases += 1;
            emit(w->id, "IDLE", w->a.stages[w->cur].node, w->a.stages[w->cur].start, w->a.stages[w->cur].end,
                 "released");
        } else if (keep < w->a.stages.size()) {
            w->a.stages.resize(keep);
        }
    }
}

std::set<CkptHandle> Engine::needed_checkpoints() const {
    // what a pending request would resume from now, and what an EXTEND of any live (un-STOPped)
    // trial would resume from; everything else in the pool is dead
    std::set<CkptHandle> need;
    FindCheckpointMemo memo;
    auto add = [&](NodeId node, StepCount step) {
        const ResumePoint rp = find_latest_checkpoint(*plan_, node, step, &memo, nullptr);
        if (rp.kind == ResumeKind::kCheckpoint) need.insert(plan_->node(rp.ckpt.node).ckpts.at(rp.ckpt.step));
    };
    for (const PendingRequest& p : plan_->pending_requests()) add(p.node, p.end);
    for (const auto& [t, ent] : trial_index_)
        if (!stopped_.count(t)) add(ent.second, ent.first);
    return need;
}

int Engine::collect_checkpoints() {
    const std::set<CkptHandle> need = needed_checkpoints();
    int freed = 0;
    for (auto& gp : gpus_) {
        Gpu& g = *gp;
        for (int e = 0; e < opts_.ckpts_per_gpu; ++e) {
            const CkptHandle& h = g.handle_of[static_cast<std::size_t>(e)];
            if (h.empty() || need.count(h)) continue;
            g.entry_of.erase(h);
            g.handle_of[static_cast<std::size_t>(e)].clear();
            smx_ok(smx_ckpt_free(g.ctx, e), "smx_ckpt_free");
            g.free_entries.push_back(e);
            ++freed;
        }
    }
    for (auto it = spilled_.begin(); it != spilled_.end();)
        it = need.count(it->first) ? std::next(it) : spilled_.erase(it);
    stats_.gc_frees += freed;
    return freed;
}

double Engine::step_cost_us(double bs) const {
    if (const auto it = opts_.step_cost_us.find(static_cast<int>(bs)); it != opts_.step_cost_us.end()) return it->second;
    return bs;  // cost model: proportional to the batch size
}

void Engine::calibrate(const std::vector<int>& batch_sizes) {
    for (auto& w : workers_)
        if (w->busy) throw IntegrityError("calibrate while workers are busy");
    smx_ctx* ctx = gpus_.front()->ctx;
    const int k = std::min(opts_.slots_per_gpu, 64);
    std::vector<int> slots(static_cast<std::size_t>(k));
    std::iota(slots.begin(), slots.end(), 0);
    for (int bs : batch_sizes) {
        if (bs < 1 || bs > opts_.max_batch) throw ConfigError("calibrate: batch size outside [1, max_batch]");
        std::vector<float> rows;
        for (int i = 0; i < 4; ++i) rows.insert(rows.end(), {0.01f, 0.9f, 0.0f, static_cast<float>(bs)});
        for (int sl : slots) {
            smx_ok(smx_slot_init(ctx, sl), "smx_slot_init");
            smx_ok(smx_hp_upload(ctx, sl, 0, 4, rows.data()), "smx_hp_upload");
        }
        smx_ok(smx_set_timing(ctx, 1), "smx_set_timing");
        smx_ok(smx_train(ctx, k, slots.data(), 1), "smx_train");
        smx_stats a{}, b{};
        smx_get_stats(ctx, &a);
        smx_ok(smx_train(ctx, k, slots.data(), 3), "smx_train");
        smx_get_stats(ctx, &b);
        smx_ok(smx_set_timing(ctx, 0), "smx_set_timing");
        const double us = (b.lockstep_ms - a.lockstep_ms) * 1e3 / (3.0 * k);
        const double mag = std::pow(10.0, std::floor(std::log10(std::max(us, 1e-9))) - 2);
        opts_.step_cost_us[bs] = std::round(us / mag) * mag;  // 3 significant digits
        for (int sl : slots) smx_ok(smx_release_slot(ctx, sl), "smx_release_slot");
    }
    smx_ok(smx_sync(ctx), "smx_sync");
    smx_reset_stats(ctx);
}

std::vector<TrialRef> Engine::trials() const {
    std::vector<TrialRef> v;
    for (const auto& kv : trial_index_) v.push_back(kv.first);
    return v;
}

StepCount Engine::trial_end(const TrialRef& t) const { return trial_index_.at(t).first; }

MetricHistory Engine::history(const TrialRef& t) const {
    const auto& [end, leaf] = trial_index_.at(t);
    MetricHistory h;
    const auto path = plan_->path_to(leaf);
    for (std::size_t i = 0; i < path.size(); ++i) {
        const PlanNode& n = plan_->node(path[i]);
        const StepCount hi = i + 1 < path.size() ? plan_->node(path[i + 1]).start_step : end;
        for (const auto& [s, rec] : n.metrics)
            if (s > n.start_step && s <= hi) h[s] = rec;
    }
    return h;
}

TimeUs Engine::est_us(NodeId n) const {
    // StepTimeEstimator (stage_tree.hpp:88-90): the node's stored runtime once a stage of it ran
    // (SearchPlan::set_runtime), else the profile table / bs-proportional model at
    // the batch size of the node's start -- a pure function of the plan, so schedules are
    // deterministic
    const PlanNode& node = plan_->node(n);
    if (node.runtime_sec_per_step > 0) return std::max<TimeUs>(1, std::llround(node.runtime_sec_per_step * 1e6));
    double bs = opts_.default_bs;
    if (node.config.count(opts_.hp_bs)) bs = plan_->value_at(n, opts_.hp_bs, node.start_step);
    return std::max<TimeUs>(1, std::llround(step_cost_us(bs)));
}

std::set<NodeId> Engine::owned_roots() const {
    const auto& roots = plan_->roots();
    if (opts_.world <= 1) return {roots.begin(), roots.end()};
    assign_roots(*plan_, opts_.world, root_owner_);  // deterministic: every rank computes the same map
    std::set<NodeId> own;
    for (const auto& [r, o] : root_owner_)
        if (o == opts_.rank) own.insert(r);
    return own;
}

std::set<NodeId> Engine::blocked_nodes() const {
    std::set<NodeId> running;
    for (const auto& w : workers_)
        if (w->busy)
            for (std::size_t i = w->cur; i < w->a.stages.size(); ++i) running.insert(w->a.stages[i].node);
    if (opts_.world > 1) {
        const std::set<NodeId> own = owned_roots();
        for (const PlanNode& n : plan_->nodes())
            if (!own.count(root_of(*plan_, n.id))) running.insert(n.id);
    }
    return running;
}

int Engine::alloc_entry(int gpu) {
    Gpu& g = *gpus_[static_cast<std::size_t>(gpu)];
    if (g.free_entries.empty() && opts_.ckpt_gc) {
        // pool full: free the least recently used dead entry (checkpoint GC, no spill)
        const std::set<CkptHandle> need = needed_checkpoints();
        int victim = -1;
        for (int e = 0; e < opts_.ckpts_per_gpu; ++e)
            if (!need.count(g.handle_of[static_cast<std::size_t>(e)]) &&
                (victim < 0 || g.last_use[static_cast<std::size_t>(e)] < g.last_use[static_cast<std::size_t>(victim)]))
                victim = e;
        if (victim >= 0) {
            g.entry_of.erase(g.handle_of[static_cast<std::size_t>(victim)]);
            g.handle_of[static_cast<std::size_t>(victim)].clear();
            smx_ok(smx_ckpt_free(g.ctx, victim), "smx_ckpt_free");
            g.free_entries.push_back(victim);
            stats_.gc_frees += 1;
        }
    }
    if (g.free_entries.empty()) {
        // every entry is still needed: spill the least recently used one to host memory (the
        // checkpoint spill tier); a later LOAD brings it back with smx_ckpt_write
        int victim = -1;
        for (int e = 0; e < opts_.ckpts_per_gpu; ++e)
            if (victim < 0 || g.last_use[static_cast<std::size_t>(e)] < g.last_use[static_cast<std::size_t>(victim)])
                victim = e;
        const CkptHandle h = g.handle_of[static_cast<std::size_t>(victim)];
        if (!spilled_.count(h)) {
            HostCkpt hc;
            hc.w.resize(static_cast<std::size_t>(p_alloc_));
            hc.m.resize(static_cast<std::size_t>(p_alloc_));
            smx_ok(smx_ckpt_read(g.ctx, victim, hc.w.data(), hc.m.data(), &hc.step, &hc.offset), "smx_ckpt_read");
            stats_.d2h_bytes += 8 * p_alloc_;
            spilled_.emplace(h, std::move(hc));
        }
        g.entry_of.erase(h);
        g.handle_of[static_cast<std::size_t>(victim)].clear();
        smx_ckpt_free(g.ctx, victim);
        g.free_entries.push_back(victim);
        stats_.spills += 1;
    }
    const int e = g.free_entries.back();
    g.free_entries.pop_back();
    g.last_use[static_cast<std::size_t>(e)] = ++use_clock_;
    return e;
}

// Pool entry holding checkpoint `h` on `gpu`, peer-copying it from another GPU if needed (K7).
int Engine::ckpt_on(int gpu, const CkptHandle& h) {
    Gpu& g = *gpus_[static_cast<std::size_t>(gpu)];
    if (auto it = g.entry_of.find(h); it != g.entry_of.end()) {
        g.last_use[static_cast<std::size_t>(it->second)] = ++use_clock_;
        return it->second;
    }
    for (std::size_t o = 0; o < gpus_.size(); ++o) {
        Gpu& src = *gpus_[o];
        auto it = src.entry_of.find(h);
        if (it == src.entry_of.end()) continue;
        const int e = alloc_entry(gpu);
        smx_ok(smx_ckpt_peer_copy(g.ctx, e, src.ctx, it->second), "smx_ckpt_peer_copy");
        g.entry_of[h] = e;
        g.handle_of[static_cast<std::size_t>(e)] = h;
        stats_.peer_copies += 1;
        return e;
    }
    if (auto it = spilled_.find(h); it != spilled_.end()) {
        const int e = alloc_entry(gpu);
        const HostCkpt& hc = it->second;
        smx_ok(smx_ckpt_write(g.ctx, e, hc.w.data(), hc.m.data(), hc.step, hc.offset), "smx_ckpt_write");
        stats_.h2d_bytes += 8 * p_alloc_;
        g.entry_of[h] = e;
        g.handle_of[static_cast<std::size_t>(e)] = h;
        return e;
    }
    return -1;
}

void Engine::upload_hp(Worker& w, const Stage& s) {
    const StepCount n = s.end - s.start;
    if (n <= 0) return;
    std::vector<float> rows(static_cast<std::size_t>(n) * SMX_HP_COLS);
    const auto& cfg = plan_->node(s.node).config;
    const std::string* names[SMX_HP_COLS] = {&opts_.hp_lr, &opts_.hp_momentum, &opts_.hp_wd, &opts_.hp_bs};
    const double defaults[SMX_HP_COLS] = {opts_.default_lr, opts_.default_momentum, opts_.default_wd, opts_.default_bs};
    for (int c = 0; c < SMX_HP_COLS; ++c) {
        const bool tuned = cfg.count(*names[c]) > 0;
        for (StepCount i = 0; i < n; ++i)
            rows[static_cast<std::size_t>(i) * SMX_HP_COLS + c] =
                static_cast<float>(tuned ? plan_->value_at(s.node, *names[c], s.start + i) : defaults[c]);
    }
    smx_ok(smx_hp_upload(gpus_[static_cast<std::size_t>(w.gpu)]->ctx, w.slot, s.start, n, rows.data()), "smx_hp_upload");
    stats_.h2d_bytes += static_cast<std::int64_t>(rows.size() * sizeof(float));
}

void Engine::begin_stage(Worker& w) {
    const Stage& s = w.a.stages[w.cur];
    upload_hp(w, s);
    w.remaining = s.end - s.start;
    const PlanNode& n = plan_->node(s.node);
    w.cost_us = step_cost_us(n.config.count(opts_.hp_bs) ? plan_->value_at(s.node, opts_.hp_bs, s.start) : opts_.default_bs);
    if (s.end > s.start) emit(w.id, "TRAIN", s.node, s.start, s.end);
}

void Engine::start(const Assignment& a) {
    Worker& w = *workers_[static_cast<std::size_t>(a.worker)];
    w.busy = true;
    w.a = a;
    w.cur = 0;
    smx_ctx* ctx = gpus_[static_cast<std::size_t>(w.gpu)]->ctx;
    const Stage& first = a.stages.front();
    if (first.resume) {
        const PlanNode& n = plan_->node(first.resume->node);
        const auto it = n.ckpts.find(first.resume->step);
        if (it == n.ckpts.end())
            throw IntegrityError("resume checkpoint missing at node " + std::to_string(first.resume->node));
        const int e = ckpt_on(w.gpu, it->second);
        if (e < 0) throw IntegrityError("checkpoint " + it->second + " is not resident on any GPU");
        smx_ok(smx_slot_load(ctx, w.slot, e), "smx_slot_load");
        stats_.loads += 1;
        emit(w.id, "LOAD", first.resume->node, first.resume->step, first.resume->step, it->second);
    } else {
        if (first.start != 0) throw IntegrityError("scratch stage must start at step 0");
        smx_ok(smx_slot_init(ctx, w.slot), "smx_slot_init");
        stats_.inits += 1;
        emit(w.id, "LOAD", first.node, 0, 0, "init");
    }
    stats_.assignments += 1;
    begin_stage(w);
}

void Engine::dispatch() {
    std::vector<int> idle;
    for (const auto& w : workers_)
        if (!w->busy) idle.push_back(w->id);
    if (idle.empty() || !plan_->has_pending()) return;
    TreeBuildContext ctx;
    ctx.running = blocked_nodes();
    ctx.eval_intervals = opts_.eval_intervals;
    const auto est = [this](NodeId n) { return est_us(n); };
    std::vector<Assignment> as;
    if (gpus_.size() == 1) {
        as = schedule(*plan_, ctx, idle, est, next_assignment_);
    } else {
        const std::map<NodeId, int> place = place_nodes(*plan_, static_cast<int>(gpus_.size()));
        std::vector<std::vector<int>> by_dev(gpus_.size());
        for (int w : idle) by_dev[static_cast<std::size_t>(workers_[static_cast<std::size_t>(w)]->gpu)].push_back(w);
        as = schedule_placed(*plan_, ctx, by_dev, [&place](NodeId n) { return place.at(n); }, est, next_assignment_);
    }
    next_assignment_ += static_cast<int>(as.size());
    for (const Assignment& a : as) start(a);
}

void Engine::finish_stages(std::vector<Worker*>& done) {
    // SAVE (every stage end) in worker order
    for (Worker* w : done) {
        const Stage& s = w->a.stages[w->cur];
        if (s.end <= s.start) continue;
        const CkptHandle h = hex16(plan_->prefix_digest_at(s.node, s.end));
        const PlanNode& n = plan_->node(s.node);
        Gpu& g = *gpus_[static_cast<std::size_t>(w->gpu)];
        bool resident = false;
        for (const auto& og : gpus_) resident = resident || og->entry_of.count(h);
        resident = resident || spilled_.count(h);
        if (!resident) {
            const int e = alloc_entry(w->gpu);
            smx_ok(smx_slot_save(g.ctx, w->slot, e), "smx_slot_save");
            g.entry_of[h] = e;
            g.handle_of[static_cast<std::size_t>(e)] = h;
            stats_.saves += 1;
        }
        emit(w->id, "SAVE", s.node, s.end, s.end, resident ? "resident:" + h : h);
        plan_->record_checkpoint(s.node, s.end, h);
        // the node's runtime after its first executed stage: the profiled cost
        // of its batch size (SearchPlan::set_runtime, plan.cpp:290-292)
        if (n.runtime_sec_per_step <= 0) {
            const double bs = n.config.count(opts_.hp_bs) ? plan_->value_at(s.node, opts_.hp_bs, s.start) : opts_.default_bs;
            plan_->set_runtime(s.node, step_cost_us(bs) * 1e-6);
        }
    }
    // EVAL, batched per GPU
    std::map<int, std::vector<Worker*>> by_gpu;
    for (Worker* w : done)
        if (w->a.stages[w->cur].eval_at_end) by_gpu[w->gpu].push_back(w);
    std::map<int, MetricRecord> records;
    for (auto& [gi, ws] : by_gpu) {
        std::vector<int> slots;
        for (Worker* w : ws) slots.push_back(w->slot);
        std::vector<double> out(slots.size() * SMX_MET_COLS);
        smx_ok(smx_eval(gpus_[static_cast<std::size_t>(gi)]->ctx, static_cast<int>(slots.size()), slots.data(), out.data()),
               "smx_eval");
        stats_.evals += static_cast<std::int64_t>(slots.size());
        stats_.d2h_bytes += static_cast<std::int64_t>(out.size() * sizeof(double));
        for (std::size_t i = 0; i < ws.size(); ++i)
            records[ws[i]->id] = MetricRecord{{"val_acc", out[i * SMX_MET_COLS + SMX_MET_VAL_ACC]},
                                              {"val_loss", out[i * SMX_MET_COLS + SMX_MET_VAL_LOSS]}};
    }
    // aggregate: record metrics, fan out completions, advance workers (ascending id)
    for (Worker* w : done) {
        if (!w->busy) continue;  // released by a STOP issued from an earlier completion callback
        const Stage s = w->a.stages[w->cur];
        if (auto it = records.find(w->id); it != records.end()) {
            const std::vector<CompletedRequest> comp = plan_->record_metrics(s.node, s.end, it->second);
            char buf[96];
            std::snprintf(buf, sizeof buf, "val_acc=%.17g;val_loss=%.17g", it->second.at("val_acc"),
                          it->second.at("val_loss"));
            std::string detail = buf;
            std::string who;
            for (const CompletedRequest& c : comp)
                for (const TrialRef& t : c.subscribers) who += (who.empty() ? "" : ",") + std::to_string(t.study) + ":" + std::to_string(t.trial);
            if (!who.empty()) detail += ";trials=" + who;
            emit(w->id, "EVAL", s.node, s.end, s.end, detail);
            for (const CompletedRequest& c : comp) {
                for (const TrialRef& t : c.subscribers) credit(t, c.end);
                if (on_complete_) on_complete_(*this, c);
            }
        }
        if (!w->busy) continue;  // this worker's own remaining path was released by the callback
        w->cur += 1;
        if (w->cur < w->a.stages.size()) {
            begin_stage(*w);
        } else {
            w->busy = false;
            emit(w->id, "IDLE", s.node, s.end, s.end);
        }
    }
}

void Engine::run() {
    static const bool trace = std::getenv("SMX_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const int G = static_cast<int>(gpus_.size());
    for (;;) {
        dispatch();
        // stages with nothing (left) to train finish immediately: eval-only stages
        for (;;) {
            std::vector<Worker*> done;
            for (auto& w : workers_)
                if (w->busy && w->remaining == 0) done.push_back(w.get());
            if (done.empty()) break;
            finish_stages(done);
            dispatch();
        }
        std::vector<Worker*> active;
        for (auto& w : workers_)
            if (w->busy) active.push_back(w.get());
        if (active.empty()) break;
        StepCount k = active.front()->remaining;
        for (Worker* w : active) k = std::min(k, w->remaining);
        if (trace) std::fprintf(stderr, "[engine] active=%zu k=%lld stage_steps=%lld\n", active.size(),
                                static_cast<long long>(k), static_cast<long long>(stats_.stage_steps));
        for (int gi = 0; gi < G; ++gi) {
            std::vector<int> slots;
            for (Worker* w : active)
                if (w->gpu == gi) slots.push_back(w->slot);
            if (slots.empty()) continue;
            smx_ok(smx_train(gpus_[static_cast<std::size_t>(gi)]->ctx, static_cast<int>(slots.size()), slots.data(),
                             static_cast<int>(k)),
                   "smx_train");
            stats_.locksteps += k;
        }
        double busy = 0, slowest = 0;
        for (Worker* w : active) {
            w->remaining -= k;
            busy += w->cost_us;
            slowest = std::max(slowest, w->cost_us);
        }
        stats_.model_busy_us += busy * static_cast<double>(k);
        stats_.model_wall_us += slowest * static_cast<double>(k);
        stats_.stage_steps += k * static_cast<StepCount>(active.size());
        clock_ += k;
    }
    for (auto& g : gpus_) smx_ok(smx_sync(g->ctx), "smx_sync");
    std::int64_t launches = 0;
    for (auto& g : gpus_) {
        smx_stats st{};
        smx_get_stats(g->ctx, &st);
        launches += st.launches;
    }
    stats_.kernel_launches = launches;
    stats_.wall_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace stagemerge
