// stagemerge/scheduler.hpp — the stateless critical-path scheduler (paper §4.3, PAPER.md:365-384;
// SPEC.md:304-363).  Missing from the reference (scheduler.cpp, core/CMakeLists.txt:5); restated
// from the SPEC.
#pragma once

#include <vector>

#include "stagemerge/stage_tree.hpp"

namespace stagemerge {

/// One worker's unit of work: a root-to-leaf run of consecutive stages of one tree
/// (SPEC.md:315-318).  The first stage carries the only LOAD; SAVE happens at every stage end
/// (SPEC.md:349); EVAL where Stage::eval_at_end.
struct Assignment {
    int id = 0;
    int worker = 0;
    std::vector<Stage> stages;
};

/// Builds a fresh tree from the plan snapshot and hands out critical paths to idle workers,
/// lowest worker id first, until workers or unscheduled root paths run out.  Holds no state.
std::vector<Assignment> schedule(const SearchPlan& plan, const TreeBuildContext& ctx, const std::vector<int>& idle_workers,
                                 const StepTimeEstimator& step_us, int first_assignment_id = 0);

}  // namespace stagemerge
