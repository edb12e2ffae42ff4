// Root-subtree LPT partition (see stagemerge/partition.hpp).
#include "stagemerge/partition.hpp"

#include <algorithm>
#include <set>
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

std::map<NodeId, int> place_nodes(const SearchPlan& plan, int devices) {
    if (devices < 1) throw ConfigError("placement: devices must be >= 1");
    const auto& nodes = plan.nodes();
    const std::size_t nn = nodes.size();
    std::vector<StepCount> own(nn, 0), sub(nn, 0);
    for (const PlanNode& n : nodes) {
        StepCount hi = n.start_step;
        for (const auto& e : n.requests) hi = std::max(hi, e.end);
        for (NodeId c : n.children) hi = std::max(hi, plan.node(c).start_step);
        own[static_cast<std::size_t>(n.id)] = hi - n.start_step;
    }
    for (std::size_t i = nn; i-- > 0;) {  // children have larger ids than their parents
        sub[i] += own[i];
        if (const auto& p = nodes[i].parent) sub[static_cast<std::size_t>(*p)] += sub[i];
    }
    std::set<NodeId> heads(plan.roots().begin(), plan.roots().end());
    // weight of a unit = its head's subtree minus the subtrees of heads below it
    auto weight = [&](NodeId h) {
        StepCount w = sub[static_cast<std::size_t>(h)];
        std::vector<NodeId> st(nodes[static_cast<std::size_t>(h)].children.begin(),
                               nodes[static_cast<std::size_t>(h)].children.end());
        while (!st.empty()) {
            const NodeId c = st.back();
            st.pop_back();
            if (heads.count(c)) {
                w -= sub[static_cast<std::size_t>(c)];
                continue;
            }
            for (NodeId g : nodes[static_cast<std::size_t>(c)].children) st.push_back(g);
        }
        return w;
    };
    StepCount total = 0;
    for (NodeId r : plan.roots()) total += sub[static_cast<std::size_t>(r)];
    const StepCount cap = devices > 1 ? (total + devices - 1) / devices : total;
    for (bool again = devices > 1; again;) {
        again = false;
        NodeId top = -1;
        StepCount tw = -1;
        for (NodeId h : heads) {
            const StepCount w = weight(h);
            if (w > tw) tw = w, top = h;
        }
        if (top < 0 || tw <= cap) break;
        // first branch point of the unit (breadth first): a member with >= 2 member children
        std::vector<NodeId> q{top};
        for (std::size_t qi = 0; qi < q.size() && !again; ++qi) {
            std::vector<NodeId> kids;
            for (NodeId c : nodes[static_cast<std::size_t>(q[qi])].children)
                if (!heads.count(c)) kids.push_back(c);
            if (kids.size() >= 2) {
                std::stable_sort(kids.begin(), kids.end(), [&](NodeId a, NodeId b) {
                    return sub[static_cast<std::size_t>(a)] > sub[static_cast<std::size_t>(b)];
                });
                for (std::size_t k = 1; k < kids.size(); ++k) heads.insert(kids[k]);
                again = true;
            }
            for (NodeId c : kids) q.push_back(c);
        }
    }
    // LPT over the units
    std::vector<std::pair<StepCount, NodeId>> units;
    for (NodeId h : heads) units.emplace_back(weight(h), h);
    std::stable_sort(units.begin(), units.end(), [](const auto& a, const auto& b) {
        return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    std::vector<StepCount> load(static_cast<std::size_t>(devices), 0);
    std::map<NodeId, int> unit_dev;
    for (const auto& [w, h] : units) {
        const auto d = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        unit_dev[h] = d;
        load[static_cast<std::size_t>(d)] += w;
    }
    std::map<NodeId, int> place;
    for (const PlanNode& n : nodes) {  // parents first: inherit unless the node heads a unit
        if (heads.count(n.id))
            place[n.id] = unit_dev.at(n.id);
        else
            place[n.id] = place.at(*n.parent);
    }
    return place;
}

}  // namespace stagemerge
