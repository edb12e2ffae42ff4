// stagemerge/study.hpp — study specs and samplers.
//
// A study spec is JSON (schema 1):
//   {"schema": 1, "name": "c1", "model": "mlp", "dataset": "synthetic",
//    "steps_per_iteration": 1, "max_steps": 200, "eval_interval": 0,
//    "space": {"lr": [<function>, ...], "momentum": [...]},
//    "sampler": {"kind": "grid"} | {"kind": "random", "trials": 256, "seed": 0},
//    "trials": [{"hps": {"lr": <function>}}]            (optional explicit trials)}
// where <function> is the plan-file function encoding ({"family": ..., params...}, with
// {"epochs": n} wrappers scaled by steps_per_iteration) applied over [0, max_steps).
// Grid order: Cartesian product over hp names in lexicographic order, each in declaration
// order, the last name varying fastest.
#pragma once

#include <string>
#include <vector>

#include "stagemerge/plan.hpp"

namespace stagemerge {

struct StudySpec {
    std::string name;
    CompatKey key;
    StepCount steps_per_iteration = 1;
    StepCount max_steps = 0;
    StepCount eval_interval = 0;
    std::vector<TrialConfig> trials;  // expanded, in submission order
};

StudySpec parse_study(const std::string& json_text);

/// Requests for one study: ids (study << 32) | index, trial ids = index.
std::vector<TrialRequest> study_requests(const StudySpec& spec, StudyId study);

/// Merge rate p of a set of trial configs: total steps / unique steps of the
/// merged plan (sum of node step extents).  Returned as (total, unique).
std::pair<StepCount, StepCount> merge_rate(const CompatKey& key, const std::vector<TrialConfig>& trials);

}  // namespace stagemerge
