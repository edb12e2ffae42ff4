// stagemerge/scheduler.hpp — the stateless critical-path scheduler (paper §4.3, PAPER.md:365-384;
// SPEC.md:304-363).  Missing from the reference (scheduler.cpp, core/CMakeLists.txt:5); restated
// from the SPEC.
#pragma once

#include <functional>
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

/// Multi-GPU form ("fill the least-loaded GPU's free slots" behind the same
/// critical-path rule): idle workers grouped per device; a critical path goes to the lowest-id
/// idle worker of the device its first stage's node is placed on, cut before its first stage on
/// another device (that remainder resumes from the cut's checkpoint -- saved at the stage end --
/// in a later round, on its own device, via a peer copy).  A path whose device has no idle
/// worker is passed over this round.  With one device this is exactly schedule().
std::vector<Assignment> schedule_placed(const SearchPlan& plan, const TreeBuildContext& ctx,
                                        const std::vector<std::vector<int>>& idle_by_device,
                                        const std::function<int(NodeId)>& device_of, const StepTimeEstimator& step_us,
                                        int first_assignment_id = 0);

}  // namespace stagemerge
