// Root-subtree LPT partition (see stagemerge/partition.hpp).
#include "stagemerge/partition.hpp"

#include <algorithm>
#include <vector>

namespace stagemerge {

NodeId root_of(const SearchPlan& plan, NodeId node) {
    while (const auto& p = plan.node(node).parent) node = *p;
    return node;
}

std::map<NodeId, StepCount> root_work(const SearchPlan& plan) {
    std::map<NodeId, StepCount> work;
    for (NodeId r : plan.roots()) work[r] = 0;
    for (const PlanNode& n : plan.nodes()) {
        StepCount hi = n.start_step;
        for (const auto& e : n.requests) hi = std::max(hi, e.end);
        for (NodeId c : n.children) hi = std::max(hi, plan.node(c).start_step);
        work[root_of(plan, n.id)] += hi - n.start_step;
    }
    return work;
}

void assign_roots(const SearchPlan& plan, int world, std::map<NodeId, int>& owner) {
    if (world < 1) throw ConfigError("partition: world must be >= 1");
    std::vector<NodeId> fresh;
    for (NodeId r : plan.roots())
        if (!owner.count(r)) fresh.push_back(r);
    if (fresh.empty()) return;
    const auto work = root_work(plan);
    std::vector<StepCount> load(static_cast<std::size_t>(world), 0);
    for (const auto& [r, o] : owner) load[static_cast<std::size_t>(o)] += work.count(r) ? work.at(r) : 0;
    // heaviest first; equal work keeps root-id order (stable sort over ascending ids)
    std::stable_sort(fresh.begin(), fresh.end(), [&](NodeId a, NodeId b) { return work.at(a) > work.at(b); });
    for (NodeId r : fresh) {
        const auto o = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        owner[r] = o;
        load[static_cast<std::size_t>(o)] += work.at(r);
    }
}

}  // namespace stagemerge
