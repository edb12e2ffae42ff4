// Private JSON codec for hp functions, descriptors and trial configs (nlohmann::ordered_json).
//
// The on-disk formats are interfaces: a plan file written by the reference
// (reference plan.cpp:347-437 via json_util.hpp:17-71) must load here and vice versa, so the
// encoders emit the same keys in the same order.  function_from_json is declared but never
// defined in the reference (json_util.hpp:44-45); it is restated from its contract: the
// inverse of function_to_json plus the {"epochs": n} wrapper of SPEC.md:640, scaled by
// steps-per-iteration for step-valued parameters.
#pragma once

#include <json.hpp>
#include <string>

#include "stagemerge/hpseq.hpp"

namespace stagemerge::codec {

using json = nlohmann::ordered_json;

inline Rational rational_in(const json& j, const std::string& where) {
    if (j.is_string()) return Rational::from_string(j.get<std::string>());
    if (j.is_number_integer()) return Rational(j.get<std::int64_t>());
    if (j.is_number_float()) return Rational::from_double(j.get<double>());
    throw ConfigError(where + ": expected a number or numeric string");
}

inline json rational_out(const Rational& r) { return r.is_integer() ? json(r.num()) : json(r.to_string()); }

inline json function_out(const HpFunction& f) {
    json j;
    j["family"] = family_name(f.family);
    for (const auto& [k, v] : f.params) j[k] = rational_out(v);
    for (const auto& [k, vs] : f.lists) {
        json a = json::array();
        for (const auto& v : vs) a.push_back(rational_out(v));
        j[k] = std::move(a);
    }
    if (f.inner) j["inner"] = function_out(*f.inner);
    return j;
}

inline bool step_valued(const std::string& k) {
    return k == "milestones" || k == "total" || k == "t0" || k == "duration" || k == "step_size_up" ||
           k == "step_size_down";
}

inline HpFunction function_in(const json& j, const std::string& where, StepCount steps_per_iteration) {
    if (!j.is_object()) throw ConfigError(where + ": expected an object");
    if (!j.contains("family")) throw ConfigError(where + ": missing 'family'");
    HpFunction f;
    f.family = family_from_name(j.at("family").get<std::string>());
    for (const auto& [k, v] : j.items()) {
        if (k == "family") continue;
        const std::string at = where + "." + k;
        if (k == "inner") {
            f.inner = std::make_shared<HpFunction>(function_in(v, at, steps_per_iteration));
            continue;
        }
        const Rational unit(step_valued(k) ? steps_per_iteration : 1);
        const bool epochs = v.is_object() && v.contains("epochs");
        const json& body = epochs ? v.at("epochs") : v;
        const Rational scale = epochs ? unit : Rational(1);
        if (body.is_array()) {
            std::vector<Rational> vals;
            for (const auto& e : body) {
                const bool inner_epochs = e.is_object() && e.contains("epochs");
                vals.push_back(inner_epochs ? rational_in(e.at("epochs"), at) * unit : rational_in(e, at) * scale);
            }
            f.lists[k] = std::move(vals);
        } else {
            f.params[k] = rational_in(body, at) * scale;
        }
    }
    return f;
}

inline json desc_out(const CanonDesc& d) {
    json j;
    if (d.is_const) {
        j["kind"] = "const";
        j["value"] = rational_out(d.value);
    } else {
        j["kind"] = "atom";
        j["function"] = function_out(d.atom);
        j["local"] = d.local;
    }
    return j;
}

inline CanonDesc desc_in(const json& j) {
    CanonDesc d;
    d.is_const = j.at("kind") == "const";
    if (d.is_const) {
        d.value = rational_in(j.at("value"), "desc.value");
    } else {
        d.atom = function_in(j.at("function"), "desc.function", 1);
        d.local = j.at("local").get<StepCount>();
    }
    return d;
}

/// Trial config as used by the JSON command interface, the study spec and the tests:
/// {"total_steps": T, "hps": {"lr": [{"fn": {...}, "local_start": 0, "duration": T}, ...]}}
inline TrialConfig config_in(const json& j, StepCount steps_per_iteration = 1) {
    TrialConfig c;
    c.total_steps = j.at("total_steps").get<StepCount>();
    for (const auto& [name, segs] : j.at("hps").items()) {
        HpSequence s{name, {}};
        for (const auto& sj : segs) {
            Segment seg;
            seg.function = function_in(sj.at("fn"), name, steps_per_iteration);
            seg.local_start = sj.value("local_start", StepCount{0});
            seg.duration = sj.at("duration").get<StepCount>();
            s.segments.push_back(std::move(seg));
        }
        c.sequences.emplace(name, std::move(s));
    }
    return c;
}

inline json config_out(const TrialConfig& c) {
    json hps = json::object();
    for (const auto& [name, seq] : c.sequences) {
        json segs = json::array();
        for (const auto& s : seq.segments)
            segs.push_back({{"fn", function_out(s.function)}, {"local_start", s.local_start}, {"duration", s.duration}});
        hps[name] = std::move(segs);
    }
    return {{"total_steps", c.total_steps}, {"hps", std::move(hps)}};
}

}  // namespace stagemerge::codec
