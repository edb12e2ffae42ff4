// stagemerge/tuner.hpp — HPO tuners that submit, extend and stop trials from returned metrics,
// and the driver that runs them over the engine (reference SPEC.md [MODULE] tuners, :447-530).
//
// A tuner is a pure state machine: start() and on_result() return TunerActions
// (SUBMIT / EXTEND / STOP / DONE, SPEC.md TunerAction) and never touch the plan, so its decisions
// are a function of (spec, metric history) alone (SPEC.md "Invariants & Properties").  The driver
// turns SUBMIT / EXTEND into fresh TrialRequests over a truncated copy of the trial's config —
// EXTEND is "a fresh TrialRequest with the same prefix and a larger end step, which the plan
// merges" (SPEC.md DESIGN DECISIONS) — and STOP into Engine::cancel (plan.cpp:204-225).
//
// Kinds (study spec key "tuner"):
//   {"kind": "grid"}                        every trial to max_steps, DONE with the best
//   {"kind": "sha", "reduction": 4, "min": 15, "max": 120}          (iterations; wait_all rungs)
//   {"kind": "sha", "milestones": [[5, 8], [10, 4]]}                (Fig. 10 MilestoneSchedule)
//   {"kind": "asha", "reduction": 4, "min": 15, "max": 120, "parallelism": 64}   (wait_any)
//   {"kind": "median", "interval": 10, "min": 10, "parallelism": 64}  (median stopping, iterations)
// plus "metric" (default "val_loss") and "mode" ("min" | "max", default "min").  Ties on equal
// metrics: the smaller trial id ranks first (SPEC.md DESIGN DECISIONS).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "stagemerge/plan.hpp"
#include "stagemerge/study.hpp"

namespace stagemerge {

class Engine;

struct TunerAction {
    enum class Kind { kSubmit, kExtend, kStop, kDone };
    Kind kind = Kind::kSubmit;
    TrialId trial = 0;
    StepCount end = 0;               // SUBMIT / EXTEND: requested end step
    std::vector<TrialId> winners;    // DONE
    std::string to_string() const;   // "SUBMIT 3 150", "EXTEND 3 600", "STOP 7", "DONE 1,4"
};

struct TunerParams {
    std::string kind = "grid";     // grid | sha | asha | median
    int reduction = 4;             // eta
    StepCount min_steps = 0;       // first rung / first median milestone (steps)
    StepCount max_steps = 0;       // last rung (steps)
    StepCount interval = 0;        // median: milestone spacing (steps)
    std::vector<std::pair<StepCount, int>> milestones;  // (step, survivors entering that rung)
    int parallelism = 0;           // asha / median: trials in flight (0 = all)
    std::string metric = "val_loss";
    bool maximize = false;
};

/// Parses the "tuner" object of a study spec; iteration counts are scaled by the spec's
/// steps_per_iteration.  A spec without "tuner" gets {"kind": "grid"}.
TunerParams parse_tuner(const std::string& spec_json, const StudySpec& spec);

/// SHA rung ends (steps) and survivor counts entering each rung (SPEC.md sha_step:
/// min * eta^i capped at max; n_{i+1} = ceil(n_i / eta)).
struct Rungs {
    std::vector<StepCount> ends;
    std::vector<int> survivors;
};
Rungs sha_rungs(const TunerParams& p, int n_trials);

class Tuner {
public:
    virtual ~Tuner() = default;
    virtual std::vector<TunerAction> start() = 0;
    /// Metrics of `trial` at step `end` (one of the ends it was submitted / extended to).
    virtual std::vector<TunerAction> on_result(TrialId trial, StepCount end, const MetricRecord& m) = 0;
    bool done() const { return done_; }
    const std::vector<TrialId>& winners() const { return winners_; }

protected:
    bool done_ = false;
    std::vector<TrialId> winners_;
};

std::unique_ptr<Tuner> make_tuner(const TunerParams& p, int n_trials, StepCount max_steps);

/// Outcome of one tuned study run through the engine.
struct StudyOutcome {
    StudyId study = 0;
    std::vector<TrialId> winners;
    std::vector<std::string> actions;         // in issue order
    std::map<TrialId, StepCount> trained_to;  // furthest end reported per trial
    std::int64_t trial_steps = 0;             // sum of trained_to (TRIAL-mode work of the study)
};

/// Runs studies, each under its own tuner, on one engine until every tuner is DONE (SPEC.md
/// "Tuners run as cooperative tasks over the engine's request handles").  Studies get ids
/// base_study, base_study + 1, ...; request ids are (study << 32) | sequence.
std::vector<StudyOutcome> run_tuned_studies(Engine& engine, const std::vector<std::string>& spec_jsons,
                                            StudyId base_study = 0);

}  // namespace stagemerge
