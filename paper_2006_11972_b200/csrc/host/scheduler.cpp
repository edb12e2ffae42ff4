// Stateless critical-path scheduler: fresh tree per call, repeated
// critical_path extraction, lowest-id idle worker first.
#include <algorithm>

#include "stagemerge/scheduler.hpp"

namespace stagemerge {

std::vector<Assignment> schedule(const SearchPlan& plan, const TreeBuildContext& ctx, const std::vector<int>& idle_workers,
                                 const StepTimeEstimator& step_us, int first_assignment_id) {
    std::vector<Assignment> out;
    if (idle_workers.empty()) return out;
    const StageTree tree = build_stage_tree(plan, ctx);
    std::vector<bool> taken(tree.stages.size(), false);
    std::vector<int> workers = idle_workers;
    std::sort(workers.begin(), workers.end());
    for (int w : workers) {
        const std::vector<int> path = critical_path(tree, step_us, &taken);
        if (path.empty()) break;
        Assignment a;
        a.id = first_assignment_id + static_cast<int>(out.size());
        a.worker = w;
        for (int s : path) {
            taken[static_cast<std::size_t>(s)] = true;
            a.stages.push_back(tree.stages[static_cast<std::size_t>(s)]);
        }
        out.push_back(std::move(a));
    }
    return out;
}

}  // namespace stagemerge
