// JSON command interface over the host library (smh_call).  It accepts exactly the commands
// oracle/ref_shim.cpp accepts for the compiled reference, so tests/test_host_vs_reference.py can
// replay one script through both and compare the answers byte for byte.  Extra commands
// ("tree" inside "plan") expose the stage-tree / scheduler restatement.
#include <cstring>
#include <string>

#include "json_codec.hpp"
#include "stagemerge/hpseq.hpp"
#include "stagemerge/partition.hpp"
#include "stagemerge/plan.hpp"
#include "stagemerge/scheduler.hpp"
#include "stagemerge/stage_tree.hpp"

namespace stagemerge::api {
namespace {

using namespace stagemerge;
using codec::json;

HpSequence seq_from_json(const std::string& name, const json& j) {
    HpSequence s;
    s.hp_name = name;
    for (const auto& sj : j) {
        Segment seg;
        seg.function = codec::function_in(sj.at("fn"), name, 1);
        seg.local_start = sj.value("local_start", StepCount{0});
        seg.duration = sj.at("duration").get<StepCount>();
        s.segments.push_back(std::move(seg));
    }
    return s;
}

TrialConfig cfg_from_json(const json& j) {
    TrialConfig c;
    c.total_steps = j.at("total_steps").get<StepCount>();
    for (const auto& [name, sj] : j.at("hps").items()) c.sequences.emplace(name, seq_from_json(name, sj));
    return c;
}

json canon_to_json(const std::vector<CanonSegment>& v) {
    json out = json::array();
    for (const auto& s : v) out.push_back({s.desc.to_string(), s.start, s.duration});
    return out;
}

std::string hex64(std::uint64_t h) {
    char b[20];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(h));
    return b;
}

json metrics_json(const MetricRecord& m) {
    json j = json::object();
    for (const auto& [k, v] : m) j[k] = v;
    return j;
}


json tree_json(const SearchPlan& plan, const json& t) {
    TreeBuildContext ctx;
    for (const auto& n : t.value("running", json::array())) ctx.running.insert(n.get<NodeId>());
    for (const auto& e : t.value("eval_intervals", json::array())) ctx.eval_intervals.push_back(e.get<StepCount>());
    ctx.use_memo = t.value("use_memo", true);
    const StageTree tree = build_stage_tree(plan, ctx);
    json out;
    json stages = json::array();
    for (const Stage& s : tree.stages) {
        json sj = {{"id", s.id}, {"node", s.node}, {"start", s.start}, {"end", s.end},
                   {"resume", s.resume ? json{s.resume->node, s.resume->step} : json(nullptr)},
                   {"parent", s.parent ? json(*s.parent) : json(nullptr)}, {"children", s.children},
                   {"serves", s.serves}, {"eval_at_end", s.eval_at_end}};
        stages.push_back(sj);
    }
    out["stages"] = stages;
    out["roots"] = tree.roots;
    out["leaf_count"] = tree.leaf_count();
    json iv = json::object();
    for (const auto& [r, pieces] : request_intervals(tree)) {
        json a = json::array();
        for (const auto& [n, lo, hi] : pieces) a.push_back({n, lo, hi});
        iv[std::to_string(r)] = a;
    }
    out["intervals"] = iv;
    // per-node step cost in us (default 1) for critical paths
    std::map<NodeId, TimeUs> cost;
    const json step_us = t.value("step_us", json::object());
    for (const auto& [k, v] : step_us.items()) cost[std::stoll(k)] = v.get<TimeUs>();
    StepTimeEstimator est = [&](NodeId n) { auto it = cost.find(n); return it == cost.end() ? TimeUs{1} : it->second; };
    out["critical_path"] = critical_path(tree, est);
    out["critical_us"] = path_duration_us(tree, critical_path(tree, est), est);
    if (t.contains("workers")) {
        json as = json::array();
        for (const Assignment& a : schedule(plan, ctx, t.at("workers").get<std::vector<int>>(), est)) {
            json ids = json::array();
            for (const Stage& s : a.stages) ids.push_back(s.id);
            as.push_back({{"id", a.id}, {"worker", a.worker}, {"stages", ids}});
        }
        out["assignments"] = as;
    }
    out["dot"] = tree.to_dot();
    return out;
}

json run(const json& cmd) {
    const std::string op = cmd.at("op").get<std::string>();
    json out;
    if (op == "value_at") {
        HpFunction f = codec::function_in(cmd.at("fn"), "fn", 1);
        validate_function(f);
        json vals = json::array();
        for (const auto& s : cmd.at("steps")) vals.push_back(value_at(f, s.get<StepCount>()));
        out["values"] = vals;
    } else if (op == "sequence") {
        TrialConfig c = cfg_from_json(cmd.at("config"));
        validate_config(c);
        json per = json::object();
        for (const auto& [name, seq] : c.sequences) {
            json e;
            e["canon"] = canon_to_json(canonical_segments(seq));
            json vals = json::array();
            for (StepCount s = 0; s < c.total_steps; ++s) vals.push_back(sequence_value_at(seq, s));
            e["values"] = vals;
            if (cmd.contains("split")) {
                auto [l, r] = split_at(seq, cmd.at("split").get<StepCount>());
                json lv = json::array(), rv = json::array();
                for (StepCount s = 0; s < l.length(); ++s) lv.push_back(sequence_value_at(l, s));
                for (StepCount s = 0; s < r.length(); ++s) rv.push_back(sequence_value_at(r, s));
                e["split_left"] = lv;
                e["split_right"] = rv;
            }
            per[name] = e;
        }
        out["hps"] = per;
        json comb = json::array();
        for (const auto& cs : combined_segments(c)) {
            json d = json::object();
            for (const auto& [n, desc] : cs.descs) d[n] = desc.to_string();
            comb.push_back({cs.start, cs.duration, d});
        }
        out["combined"] = comb;
        json dig = json::array();
        for (const auto& s : cmd.value("digest_steps", json::array()))
            dig.push_back(hex64(prefix_digest(c, s.get<StepCount>())));
        out["digests"] = dig;
    } else if (op == "common_prefix") {
        out["n"] = common_prefix_steps(cfg_from_json(cmd.at("a")), cfg_from_json(cmd.at("b")));
    } else if (op == "rational") {
        json r = json::array();
        for (const auto& t : cmd.at("texts")) {
            Rational q = Rational::from_string(t.get<std::string>());
            r.push_back({q.to_string(), q.num(), q.den()});
        }
        out["rationals"] = r;
    } else if (op == "plan") {
        const auto& k = cmd.at("key");
        CompatKey key{k.at("model").get<std::string>(), k.at("dataset").get<std::string>(),
                      k.at("hp_set").get<std::vector<std::string>>()};
        SearchPlan plan(key);
        json results = json::array();
        for (const auto& a : cmd.at("actions")) {
            json r;
            try {
                const std::string kind = a.at("kind").get<std::string>();
                if (kind == "insert") {
                    TrialRequest req;
                    req.id = a.at("id").get<RequestId>();
                    req.study = a.at("study").get<StudyId>();
                    req.trial = a.at("trial").get<TrialId>();
                    req.config = cfg_from_json(a.at("config"));
                    InsertOutcome o = plan.insert_trial(req);
                    r = {{"kind", o.kind == InsertOutcome::Kind::kImmediate ? "immediate" : "pending"},
                         {"request", o.request_id}, {"node", o.node}, {"attached", o.attached},
                         {"metrics", metrics_json(o.metrics)}};
                } else if (kind == "ckpt") {
                    r = {{"new", plan.record_checkpoint(a.at("node").get<NodeId>(), a.at("step").get<StepCount>(),
                                                        a.at("handle").get<std::string>())}};
                } else if (kind == "metrics") {
                    MetricRecord m;
                    for (const auto& [mk, mv] : a.at("record").items()) m[mk] = mv.get<double>();
                    json done = json::array();
                    for (const auto& c : plan.record_metrics(a.at("node").get<NodeId>(),
                                                             a.at("step").get<StepCount>(), m)) {
                        json subs = json::array();
                        for (const auto& t : c.subscribers) subs.push_back({t.study, t.trial});
                        done.push_back({{"id", c.id}, {"node", c.node}, {"end", c.end}, {"subscribers", subs}});
                    }
                    r = {{"completed", done}};
                } else if (kind == "cancel") {
                    r = {{"changed", plan.cancel_trial(TrialRef{a.at("study").get<StudyId>(),
                                                                a.at("trial").get<TrialId>()})}};
                } else if (kind == "value_at") {
                    r = {{"value", plan.value_at(a.at("node").get<NodeId>(), a.at("hp").get<std::string>(),
                                                 a.at("step").get<StepCount>())}};
                } else if (kind == "digest_at") {
                    r = {{"digest", hex64(plan.prefix_digest_at(a.at("node").get<NodeId>(),
                                                                a.at("step").get<StepCount>()))}};
                } else {
                    throw ConfigError("unknown action " + kind);
                }
            } catch (const ConfigError& e) {
                r = {{"error", "ConfigError"}, {"what", e.what()}};
            } catch (const IntegrityError& e) {
                r = {{"error", "IntegrityError"}, {"what", e.what()}};
            } catch (const std::out_of_range& e) {
                r = {{"error", "out_of_range"}, {"what", e.what()}};
            }
            results.push_back(r);
        }
        out["results"] = results;
        out["signature"] = plan.signature();
        out["json"] = plan.to_json(cmd.value("indent", 2));
        out["dot"] = plan.to_dot();
        out["version"] = plan.version();
        out["node_count"] = plan.node_count();
        json pend = json::array();
        for (const auto& p : plan.pending_requests()) {
            json subs = json::array();
            for (const auto& t : p.subscribers) subs.push_back({t.study, t.trial});
            pend.push_back({{"node", p.node}, {"id", p.id}, {"end", p.end}, {"subscribers", subs}});
        }
        out["pending"] = pend;
        if (cmd.contains("kwise")) {
            try {
                out["kwise_signature"] =
                    kwise_view(plan, cmd.at("kwise").get<std::vector<StudyId>>()).signature();
            } catch (const ConfigError& e) {
                out["kwise_signature"] = {{"error", "ConfigError"}, {"what", e.what()}};
            }
        }
        if (cmd.value("roundtrip", false))
            out["roundtrip_signature"] = SearchPlan::from_json(plan.to_json()).signature();
        out["file_name"] = PlanStore::file_name(key);
        if (cmd.contains("tree")) out["tree"] = tree_json(plan, cmd.at("tree"));
        if (cmd.contains("partition")) {
            std::map<NodeId, int> owner;
            assign_roots(plan, cmd.at("partition").get<int>(), owner);
            json own = json::object();
            for (const auto& [r, o] : owner) own[std::to_string(r)] = o;
            json work = json::object();
            for (const auto& [r, w] : root_work(plan)) work[std::to_string(r)] = w;
            out["partition"] = {{"owner", own}, {"work", work}};
        }
        if (cmd.contains("placement")) {
            json pl = json::object();
            for (const auto& [n, d] : place_nodes(plan, cmd.at("placement").get<int>())) pl[std::to_string(n)] = d;
            out["placement"] = pl;
        }
    } else {
        throw ConfigError("unknown op " + op);
    }
    return out;
}

}  // namespace

std::string call(const std::string& text) {
    json out;
    try {
        out = run(json::parse(text));
    } catch (const ConfigError& e) {
        out = {{"error", "ConfigError"}, {"what", e.what()}};
    } catch (const IntegrityError& e) {
        out = {{"error", "IntegrityError"}, {"what", e.what()}};
    } catch (const std::out_of_range& e) {
        out = {{"error", "out_of_range"}, {"what", e.what()}};
    } catch (const std::exception& e) {
        out = {{"error", "exception"}, {"what", e.what()}};
    }
    return out.dump();
}

}  // namespace stagemerge::api

extern "C" __attribute__((visibility("default"))) const char* smh_call(const char* text) {
    thread_local std::string out;
    out = stagemerge::api::call(text);
    return out.c_str();
}
