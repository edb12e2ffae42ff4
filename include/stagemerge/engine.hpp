// stagemerge/engine.hpp — the event loop that drives the B200 stage executor.
//
// Replaces the reference's simulator loop (sim.cpp is missing from the
// reference, core/CMakeLists.txt:8) with real execution: schedule() hands critical paths to
// workers, and each worker's worker_execute runs on a GPU slot through the smx
// C ABI (include/smx.h): LOAD (smx_slot_load / smx_slot_init), TRAIN (smx_hp_upload +
// grouped smx_train locksteps), SAVE at every stage end (smx_slot_save), EVAL at
// declared steps (smx_eval).  aggregate becomes record_checkpoint /
// record_metrics on the plan, and completions fan out to a callback (the tuner hook).
//
// Determinism: time is counted in locksteps, not wall-clock.  Per lockstep every active worker
// advances the same number of steps; stage ends are processed in ascending worker id; the cost
// estimate is a pure function of the plan.  So the plan evolves identically on every run
// (SURVEY App. B.3), and the GPU kernels' grouping invariance makes STAGE and TRIAL metric
// histories bitwise equal.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "stagemerge/plan.hpp"
#include "stagemerge/scheduler.hpp"

struct smx_ctx;

namespace stagemerge {

struct EngineOptions {
    std::vector<int> devices{0};
    int slots_per_gpu = 64;    // workers per GPU (each owns one slot of the slab)
    int ckpts_per_gpu = 1024;  // checkpoint pool entries per GPU
    int gemm_mode = 0;         // SMX_GEMM_EXACT / SMX_GEMM_TC
    int max_steps = 4096;      // hp-table capacity (absolute steps)
    int max_batch = 256;
    int n_train = 65536;
    int n_val = 4096;
    std::uint64_t seed = 2006'11972;
    std::vector<StepCount> eval_intervals;  // extra eval marks (request ends always evaluate)
    bool trial_mode = false;                // no merging: every trial runs on its own path
    bool use_graphs = true;
    // hp names the executor reads (absent hps take the defaults)
    std::string hp_lr = "lr", hp_momentum = "momentum", hp_wd = "weight_decay", hp_bs = "batch_size";
    double default_lr = 0.1, default_momentum = 0.9, default_wd = 0.0, default_bs = 128;
    // multi-process partition: this process executes only the root subtrees LPT assigns to `rank`
    int rank = 0, world = 1;
    // profiled seconds-per-step table (batch size -> microseconds per stage-step); after a node's
    // first executed stage its entry is stored with SearchPlan::set_runtime and
    // the scheduler's estimator reads it.  Empty: the bs-proportional cost model.
    std::map<int, double> step_cost_us;
    // checkpoint GC (plan.hpp:45 ref_count; policy ours): when the
    // pool is full, an entry no pending request resumes from and no live (un-STOPped) trial can
    // be extended from is freed instead of spilled to host memory
    bool ckpt_gc = true;
};

/// One event of the execution trace (SPEC.md:436 columns time_us,worker,kind,node,start,end,
/// detail).  Time is the engine's logical lockstep clock in training steps, so repeated runs
/// give byte-identical traces (acceptance 10); device time is in EngineStats.
struct TraceEvent {
    StepCount time = 0;
    int worker = 0;
    std::string kind;  // LOAD, TRAIN, SAVE, EVAL, IDLE
    NodeId node = -1;
    StepCount start = 0, end = 0;
    std::string detail;
};

struct EngineStats {
    double wall_s = 0;            // host wall time spent inside run()
    std::int64_t locksteps = 0;   // grouped training launches (sum over GPUs)
    std::int64_t stage_steps = 0; // (slot, step) updates executed
    std::int64_t trial_steps = 0; // sum over trials of the furthest end step reported to them
                                  // (the work TRIAL mode would do; extensions count once)
    std::int64_t saves = 0, loads = 0, inits = 0, peer_copies = 0, evals = 0, assignments = 0, spills = 0;
    std::int64_t releases = 0;    // in-flight slots freed because STOP cancelled every request they served
    std::int64_t gc_frees = 0;    // pool entries freed by checkpoint GC (no spill)
    // the cost model's time of the executed schedule (deterministic, SPEC.md:403/:428 semantics
    // with zero save/load/eval overheads): busy = sum over workers, wall = per lockstep the
    // slowest active worker
    double model_busy_us = 0, model_wall_us = 0;
    std::int64_t kernel_launches = 0;
    std::int64_t h2d_bytes = 0, d2h_bytes = 0;
};

/// One trial's metric history along its plan path: step -> record.
using MetricHistory = std::map<StepCount, MetricRecord>;

class Engine {
public:
    Engine(CompatKey key, EngineOptions opts);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    /// Inserts a trial into the plan (in TRIAL mode onto its own unmerged path).
    InsertOutcome submit(const TrialRequest& req);
    /// STOP / cancel_trial (plan.cpp:204-225): drops the trial's pending request; in-flight
    /// assignments are cut after their last stage that still serves a pending request, and a
    /// worker left with nothing to serve releases its slot (smx_release_slot).  Shared stages
    /// keep running.
    bool cancel(const TrialRef& t);

    using CompletionFn = std::function<void(Engine&, const CompletedRequest&)>;
    void on_complete(CompletionFn fn) { on_complete_ = std::move(fn); }
    const CompletionFn& completion_callback() const { return on_complete_; }

    /// Runs until no schedulable work remains.
    void run();

    /// Fresh plan (same key), keeping the GPU contexts and the dataset.  Checkpoint pools are
    /// emptied.
    void reset();

    /// Overwrites the synthetic dataset with host data (pinned-copy path used by the e2e bench).
    void upload_dataset(const float* x, const std::int32_t* y, const float* vx, const std::int32_t* vy);
    std::uint64_t dataset_digest();

    const SearchPlan& plan() const { return *plan_; }
    const EngineStats& stats() const { return stats_; }
    const std::vector<TraceEvent>& trace() const { return trace_; }
    /// Frees every checkpoint-pool entry the GC policy considers dead; returns how many.
    int collect_checkpoints();
    /// Profiles microseconds per stage-step for each batch size (timed locksteps on idle slots of
    /// the first GPU, 3 significant digits) into options().step_cost_us.  Needs idle workers.
    void calibrate(const std::vector<int>& batch_sizes);
    const EngineOptions& options() const { return opts_; }
    MetricHistory history(const TrialRef& t) const;
    std::vector<TrialRef> trials() const;
    StepCount trial_end(const TrialRef& t) const;
    /// Root subtrees owned by this rank (all roots when world == 1).
    std::set<NodeId> owned_roots() const;
    std::vector<smx_ctx*> contexts() const;

private:
    struct Worker;
    struct Gpu;
    void dispatch();
    void start(const Assignment& a);
    void begin_stage(Worker& w);
    void finish_stages(std::vector<Worker*>& done);
    void upload_hp(Worker& w, const Stage& s);
    int ckpt_on(int gpu, const CkptHandle& h);
    int alloc_entry(int gpu);
    TimeUs est_us(NodeId n) const;
    std::set<NodeId> blocked_nodes() const;
    void release_orphans();
    std::set<CkptHandle> needed_checkpoints() const;
    double step_cost_us(double bs) const;
    void emit(int worker, const char* kind, NodeId node, StepCount start, StepCount end, std::string detail = {});

    CompatKey key_;
    EngineOptions opts_;
    std::unique_ptr<SearchPlan> plan_;
    std::vector<std::unique_ptr<Gpu>> gpus_;
    std::vector<std::unique_ptr<Worker>> workers_;
    std::map<TrialRef, std::pair<StepCount, NodeId>> trial_index_;  // trial -> (end, terminal node)
    std::map<TrialRef, TrialConfig> trial_cfg_;
    std::map<TrialRef, StepCount> reached_;  // furthest end reported per trial
    void credit(const TrialRef& t, StepCount end);
    CompletionFn on_complete_;
    EngineStats stats_;
    int next_assignment_ = 0;
    mutable std::map<NodeId, int> root_owner_;
    struct HostCkpt {
        std::vector<float> w, m;
        std::int64_t step = 0, offset = 0;
    };
    std::map<CkptHandle, HostCkpt> spilled_;  // host spill tier of the checkpoint pool
    std::uint64_t use_clock_ = 0;
    std::vector<TraceEvent> trace_;
    StepCount clock_ = 0;               // logical lockstep clock (training steps)
    std::set<TrialRef> stopped_;        // trials STOPped / cancelled (never extended again)
    std::int64_t p_alloc_ = 0;
    std::int64_t d_in_ = 784;  // floats per input sample of the model
};

}  // namespace stagemerge
