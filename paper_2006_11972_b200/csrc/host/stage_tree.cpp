// Stage-tree generation (paper Alg. 1 "Build Stage Tree"; Fig. 6 -> Fig. 7;
// SPEC.md:225-300) and critical-path extraction (paper §4.3).
//
// The reference declares this API (stage_tree.hpp:15-100) but ships no implementation; this is
// a restatement from the header contract, the paper and the SPEC, checked by
// tests/test_stage_tree.py against the Fig. 6 -> Fig. 7 example (SPEC acceptance 1) and against
// an independent non-memoised backward-walk oracle on random plans (acceptance 2).
#include <algorithm>
#include <sstream>

#include "stagemerge/stage_tree.hpp"

namespace stagemerge {

ResumePoint find_latest_checkpoint(const SearchPlan& plan, NodeId node, StepCount step, FindCheckpointMemo* memo,
                                   const std::set<NodeId>* running) {
    const auto key = std::make_pair(node, step);
    if (memo)
        if (auto it = memo->find(key); it != memo->end()) return it->second;
    ResumePoint rp;
    const PlanNode& n = plan.node(node);
    if (running && running->count(node)) {
        // Alg. 1 lines 15-16: a running config blocks the request -- unless the in-flight worker
        // has already saved the exact step asked for, in which case that NewCheckpoint unlocks it
        // (acceptance 8).  Any other step stays blocked: the
        // running worker will produce it.
        if (n.ckpts.count(step) && step > n.start_step) {
            rp.kind = ResumeKind::kCheckpoint;
            rp.ckpt = CkptRef{node, step};
        } else {
            rp.kind = ResumeKind::kBlocked;
        }
    } else if (auto it = n.ckpts.upper_bound(step); it != n.ckpts.begin() && std::prev(it)->first > n.start_step) {
        rp.kind = ResumeKind::kCheckpoint;  // scan step, step-1, ..., start (lines 21-24)
        rp.ckpt = CkptRef{node, std::prev(it)->first};
    } else if (n.parent) {
        rp = find_latest_checkpoint(plan, *n.parent, n.start_step, memo, running);  // line 27
    } else {
        rp.kind = ResumeKind::kScratch;
    }
    if (memo) memo->emplace(key, rp);
    return rp;
}

namespace {

struct Piece {
    NodeId node;
    StepCount lo, hi;
};

// Root-to-leaf training pieces of one request, from its resume point to its end.
std::vector<Piece> request_chain(const SearchPlan& plan, NodeId node, StepCount end, const ResumePoint& rp) {
    std::vector<Piece> rev;
    StepCount hi = end;
    for (NodeId cur = node;;) {
        const PlanNode& n = plan.node(cur);
        const bool resumes_here = rp.kind == ResumeKind::kCheckpoint && rp.ckpt.node == cur;
        const StepCount lo = resumes_here ? rp.ckpt.step : n.start_step;
        if (lo < hi || rev.empty()) rev.push_back(Piece{cur, lo, hi});
        if (resumes_here || !n.parent) break;
        hi = n.start_step;
        cur = *n.parent;
    }
    return {rev.rbegin(), rev.rend()};
}

using StageKey = std::tuple<StepCount, NodeId, StepCount>;  // (lo, node, hi): parents sort first

}  // namespace

std::size_t StageTree::leaf_count() const {
    return static_cast<std::size_t>(
        std::count_if(stages.begin(), stages.end(), [](const Stage& s) { return s.children.empty(); }));
}

std::string StageTree::to_dot() const {
    std::ostringstream os;
    os << "digraph stages {\n  rankdir=LR;\n  node [shape=box, fontname=\"monospace\"];\n";
    for (const Stage& s : stages) {
        os << "  s" << s.id << " [label=\"s" << s.id << " n" << s.node << " [" << s.start << "," << s.end << ")";
        if (s.resume) os << "\\nresume n" << s.resume->node << "@" << s.resume->step;
        if (!s.serves.empty()) {
            os << "\\nserves";
            for (RequestId r : s.serves) os << " " << r;
        }
        if (s.eval_at_end) os << "\\neval";
        os << "\"" << (s.resume ? ", style=filled" : "") << "];\n";
        if (s.parent) os << "  s" << *s.parent << " -> s" << s.id << ";\n";
    }
    os << "}\n";
    return os.str();
}

StageTree build_stage_tree(const SearchPlan& plan, const TreeBuildContext& ctx) {
    FindCheckpointMemo memo;
    struct Req {
        RequestId id;
        NodeId node;
        StepCount end;
        ResumePoint rp;
        std::vector<Piece> chain;
    };
    std::vector<Req> reqs;
    std::map<NodeId, std::set<StepCount>> cuts;  // split points per node
    for (const PendingRequest& p : plan.pending_requests()) {
        const ResumePoint rp = find_latest_checkpoint(plan, p.node, p.end, ctx.use_memo ? &memo : nullptr, &ctx.running);
        if (rp.kind == ResumeKind::kBlocked) continue;
        Req r{p.id, p.node, p.end, rp, request_chain(plan, p.node, p.end, rp)};
        for (const Piece& pc : r.chain) {
            auto& c = cuts[pc.node];
            c.insert(pc.lo);
            c.insert(pc.hi);
            for (StepCount iv : ctx.eval_intervals) {
                if (iv <= 0) continue;
                for (StepCount m = (pc.lo / iv + 1) * iv; m < pc.hi; m += iv) c.insert(m);
            }
        }
        reqs.push_back(std::move(r));
    }

    // split every chain at its node's cut points and merge identical (node, range) stages
    struct Proto {
        std::optional<CkptRef> resume;
        std::optional<StageKey> parent;
        std::set<RequestId> serves;
        bool ends_request = false;
    };
    std::map<StageKey, Proto> protos;
    for (const Req& r : reqs) {
        std::optional<StageKey> prev;
        for (const Piece& pc : r.chain) {
            const auto& c = cuts[pc.node];
            std::vector<StepCount> marks{pc.lo};
            for (auto it = c.upper_bound(pc.lo); it != c.end() && *it < pc.hi; ++it) marks.push_back(*it);
            marks.push_back(pc.hi);
            for (std::size_t i = 0; i + 1 < marks.size(); ++i) {
                const StageKey key{marks[i], pc.node, marks[i + 1]};
                Proto& p = protos[key];
                const std::optional<CkptRef> resume =
                    (!prev && r.rp.kind == ResumeKind::kCheckpoint) ? std::optional<CkptRef>(r.rp.ckpt) : std::nullopt;
                if (!p.serves.empty() && (p.parent != prev || p.resume != resume))
                    throw IntegrityError("stage tree: inconsistent history for node " + std::to_string(pc.node) +
                                         " [" + std::to_string(marks[i]) + "," + std::to_string(marks[i + 1]) + ")");
                p.parent = prev;
                p.resume = resume;
                p.serves.insert(r.id);
                prev = key;
            }
        }
        protos[*prev].ends_request = true;
    }

    StageTree tree;
    tree.generation = plan.version();
    std::map<StageKey, int> ids;
    for (const auto& kv : protos) ids.emplace(kv.first, static_cast<int>(ids.size()));
    for (const auto& [key, p] : protos) {
        Stage s;
        s.id = ids.at(key);
        s.start = std::get<0>(key);
        s.node = std::get<1>(key);
        s.end = std::get<2>(key);
        s.resume = p.resume;
        if (p.parent) s.parent = ids.at(*p.parent);
        s.serves.assign(p.serves.begin(), p.serves.end());
        s.eval_at_end = p.ends_request;
        for (StepCount iv : ctx.eval_intervals)
            if (iv > 0 && s.end > s.start && s.end % iv == 0) s.eval_at_end = true;
        tree.stages.push_back(std::move(s));
    }
    for (Stage& s : tree.stages) {
        if (s.parent)
            tree.stages[static_cast<std::size_t>(*s.parent)].children.push_back(s.id);
        else
            tree.roots.push_back(s.id);
    }
    return tree;
}

std::map<RequestId, std::vector<std::tuple<NodeId, StepCount, StepCount>>> request_intervals(const StageTree& tree) {
    std::map<RequestId, std::vector<const Stage*>> by_req;
    for (const Stage& s : tree.stages)
        for (RequestId r : s.serves) by_req[r].push_back(&s);
    std::map<RequestId, std::vector<std::tuple<NodeId, StepCount, StepCount>>> out;
    for (auto& [r, ss] : by_req) {
        std::sort(ss.begin(), ss.end(), [](const Stage* a, const Stage* b) {
            return std::tie(a->start, a->end) < std::tie(b->start, b->end);
        });
        auto& v = out[r];
        for (const Stage* s : ss) {
            if (!v.empty() && std::get<0>(v.back()) == s->node && std::get<2>(v.back()) == s->start)
                std::get<2>(v.back()) = s->end;
            else
                v.emplace_back(s->node, s->start, s->end);
        }
    }
    return out;
}

namespace {

TimeUs stage_us(const Stage& s, const StepTimeEstimator& est) { return (s.end - s.start) * est(s.node); }

}  // namespace

std::vector<int> critical_path(const StageTree& tree, const StepTimeEstimator& step_us,
                               const std::vector<bool>* scheduled) {
    const auto n = tree.stages.size();
    auto open = [&](int id) { return !scheduled || !(*scheduled)[static_cast<std::size_t>(id)]; };
    // best[s]: longest estimated duration of an unscheduled path starting at s (children have
    // larger ids than parents, so one reverse sweep suffices)
    std::vector<TimeUs> best(n, 0);
    std::vector<int> next(n, -1);
    auto better = [&](int a, int b) {  // is a preferred over b?
        if (b < 0) return true;
        if (best[a] != best[b]) return best[a] > best[b];
        const Stage &x = tree.stages[a], &y = tree.stages[b];
        return std::tie(x.node, x.start) < std::tie(y.node, y.start);
    };
    for (std::size_t i = n; i-- > 0;) {
        const Stage& s = tree.stages[i];
        int pick = -1;
        for (int c : s.children)
            if (open(c) && better(c, pick)) pick = c;
        next[i] = pick;
        best[i] = stage_us(s, step_us) + (pick >= 0 ? best[pick] : 0);
    }
    int head = -1;
    for (int r : tree.roots)
        if (open(r) && better(r, head)) head = r;
    std::vector<int> path;
    for (int s = head; s >= 0; s = next[s]) path.push_back(s);
    return path;
}

TimeUs path_duration_us(const StageTree& tree, const std::vector<int>& path, const StepTimeEstimator& step_us) {
    TimeUs t = 0;
    for (int id : path) t += stage_us(tree.stages.at(static_cast<std::size_t>(id)), step_us);
    return t;
}

}  // namespace stagemerge
