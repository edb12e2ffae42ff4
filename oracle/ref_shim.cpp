// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Differential-test shim around the *reference* host library.  The recipe in
// oracle/Makefile compiles /root/reference/proj/core/src/{hpseq,plan}.cpp as
// they lie (no copies), adds this file, and produces oracle/_ref/libstagemerge_ref.so.
// Only tests/ may load it (as the checker for the product host library in
// paper_2006_11972_b200/csrc/host).
//
// Two things live here:
//  1. stagemerge::detail::function_from_json — declared at
//     reference proj/core/src/json_util.hpp:44-45 but never defined in the
//     reference.  Restated from its documented contract: the
//     inverse of function_to_json (json_util.hpp:29-41) plus the {"epochs": n}
//     wrapper of SPEC.md:640 scaled by steps_per_iteration.
//  2. ref_call(json) — a JSON command interface exercising the reference's
//     public API (hpseq.hpp / plan.hpp).  The product exposes the very same
//     command interface (smh_call) so tests can compare the two byte for byte.
#include <algorithm>
#include <cstring>
#include <string>

#include "json_util.hpp"
#include "stagemerge/hpseq.hpp"
#include "stagemerge/plan.hpp"

namespace stagemerge::detail {

static Rational scaled(const json& j, const std::string& where, StepCount spi) {
    if (j.is_object() && j.contains("epochs"))
        return rational_from_json(j.at("epochs"), where) * Rational(spi);
    return rational_from_json(j, where);
}

HpFunction function_from_json(const json& j, const std::string& where,
                              StepCount steps_per_iteration) {
    if (!j.is_object()) throw ConfigError(where + ": expected an object");
    HpFunction f;
    f.family = family_from_name(j.at("family").get<std::string>());
    for (const auto& [k, v] : j.items()) {
        if (k == "family") continue;
        if (k == "inner") {
            f.inner = std::make_shared<HpFunction>(
                function_from_json(v, where + ".inner", steps_per_iteration));
            continue;
        }
        const bool step_like = k == "milestones" || k == "total" || k == "t0" ||
                               k == "duration" || k == "step_size_up" || k == "step_size_down";
        const StepCount spi = step_like ? steps_per_iteration : 1;
        if (v.is_array() || (v.is_object() && v.contains("epochs") && v.at("epochs").is_array())) {
            std::vector<Rational> vals;
            if (v.is_array()) {
                for (const auto& e : v) vals.push_back(scaled(e, where + "." + k, spi));
            } else {
                for (const auto& e : v.at("epochs"))
                    vals.push_back(rational_from_json(e, where + "." + k) * Rational(spi));
            }
            f.lists[k] = std::move(vals);
        } else {
            f.params[k] = scaled(v, where + "." + k, spi);
        }
    }
    return f;
}

}  // namespace stagemerge::detail

namespace {

using namespace stagemerge;
using detail::json;

HpSequence seq_from_json(const std::string& name, const json& j) {
    HpSequence s;
    s.hp_name = name;
    for (const auto& sj : j) {
        Segment seg;
        // "spi": steps per logical iteration of {"epochs": n} values; 1 = plain steps
        seg.function = detail::function_from_json(sj.at("fn"), name, sj.value("spi", StepCount{1}));
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

json run(const json& cmd) {
    const std::string op = cmd.at("op").get<std::string>();
    json out;
    if (op == "value_at") {
        HpFunction f = detail::function_from_json(cmd.at("fn"), "fn", 1);
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
        if (cmd.value("values", false)) {
            // the plan as an executable tree for the CPU executor (oracle/cpu_executor.py): each
            // node's step range [start, hi) and its hp values there, straight from the
            // reference's SearchPlan::value_at (plan.cpp:278-288)
            json nv = json::array();
            for (const PlanNode& n : plan.nodes()) {
                StepCount hi = n.start_step;
                json reqs = json::array();
                for (const auto& e : n.requests) {
                    hi = std::max(hi, e.end);
                    json subs = json::array();
                    for (const auto& t : e.subscribers) subs.push_back({t.study, t.trial});
                    reqs.push_back({{"id", e.id}, {"end", e.end}, {"subscribers", subs}});
                }
                json kids = json::array();
                for (NodeId c : n.children) {
                    hi = std::max(hi, plan.node(c).start_step);
                    kids.push_back(c);
                }
                json hps = json::object();
                for (const auto& h : key.hp_set) {
                    json v = json::array();
                    for (StepCount s = n.start_step; s < hi; ++s) v.push_back(plan.value_at(n.id, h, s));
                    hps[h] = v;
                }
                nv.push_back({{"id", n.id}, {"parent", n.parent ? json(*n.parent) : json(nullptr)},
                              {"start", n.start_step}, {"hi", hi}, {"children", kids}, {"requests", reqs},
                              {"hps", hps}});
            }
            out["node_values"] = nv;
        }
    } else {
        throw ConfigError("unknown op " + op);
    }
    return out;
}

thread_local std::string g_out;

}  // namespace

extern "C" const char* ref_call(const char* text) {
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
    g_out = out.dump();
    return g_out.c_str();
}
