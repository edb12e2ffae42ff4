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

std::vector<Assignment> schedule_placed(const SearchPlan& plan, const TreeBuildContext& ctx,
                                        const std::vector<std::vector<int>>& idle_by_device,
                                        const std::function<int(NodeId)>& device_of, const StepTimeEstimator& step_us,
                                        int first_assignment_id) {
    std::vector<Assignment> out;
    std::vector<std::vector<int>> idle = idle_by_device;
    std::size_t free_total = 0;
    for (auto& v : idle) {
        std::sort(v.begin(), v.end(), std::greater<int>());  // pop_back = lowest id
        free_total += v.size();
    }
    if (free_total == 0) return out;
    const StageTree tree = build_stage_tree(plan, ctx);
    std::vector<bool> taken(tree.stages.size(), false);
    for (;;) {
        const std::vector<int> path = critical_path(tree, step_us, &taken);
        if (path.empty() || free_total == 0) break;
        const int d = device_of(tree.stages[static_cast<std::size_t>(path.front())].node);
        std::size_t cut = 0;
        while (cut < path.size() && device_of(tree.stages[static_cast<std::size_t>(path[cut])].node) == d) ++cut;
        auto& pool = idle.at(static_cast<std::size_t>(d));
        if (pool.empty()) {  // no slot on that GPU this round: pass the whole path over
            for (int s : path) taken[static_cast<std::size_t>(s)] = true;
            continue;
        }
        Assignment a;
        a.id = first_assignment_id + static_cast<int>(out.size());
        a.worker = pool.back();
        pool.pop_back();
        --free_total;
        for (std::size_t i = 0; i < path.size(); ++i) {
            taken[static_cast<std::size_t>(path[i])] = true;  // the remainder waits for the cut's checkpoint
            if (i < cut) a.stages.push_back(tree.stages[static_cast<std::size_t>(path[i])]);
        }
        out.push_back(std::move(a));
    }
    return out;
}

}  // namespace stagemerge
