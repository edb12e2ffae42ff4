// Study spec parsing, grid / random samplers and the merge-rate analysis.
#include "stagemerge/study.hpp"

#include <algorithm>

#include "json_codec.hpp"

namespace stagemerge {

using codec::json;

namespace {

std::uint64_t splitmix(std::uint64_t& s) {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

TrialConfig make_trial(const std::map<std::string, HpFunction>& fns, StepCount steps) {
    TrialConfig c;
    c.total_steps = steps;
    for (const auto& [name, f] : fns) c.sequences.emplace(name, make_sequence(name, f, steps));
    return c;
}

}  // namespace

StudySpec parse_study(const std::string& text) {
    const json j = json::parse(text);
    if (j.value("schema", 1) != 1) throw ConfigError("study spec: unsupported schema");
    StudySpec s;
    s.name = j.value("name", std::string("study"));
    s.steps_per_iteration = j.value("steps_per_iteration", StepCount{1});
    if (s.steps_per_iteration < 1) throw ConfigError("study spec: steps_per_iteration must be >= 1");
    const json& ms = j.at("max_steps");
    s.max_steps = ms.is_object() ? ms.at("epochs").get<StepCount>() * s.steps_per_iteration : ms.get<StepCount>();
    if (s.max_steps < 1) throw ConfigError("study spec: max_steps must be >= 1");
    s.eval_interval = j.value("eval_interval", StepCount{0}) * (j.value("eval_in_iterations", false) ? s.steps_per_iteration : 1);
    s.key.model = j.value("model", std::string("mlp"));
    s.key.dataset = j.value("dataset", std::string("synthetic"));

    std::map<std::string, std::vector<HpFunction>> space;
    if (j.contains("space"))
        for (const auto& [name, opts] : j.at("space").items()) {
            if (!opts.is_array() || opts.empty()) throw ConfigError("study spec: space." + name + " must be a non-empty list");
            for (std::size_t i = 0; i < opts.size(); ++i) {
                HpFunction f = codec::function_in(opts[i], "space." + name + "[" + std::to_string(i) + "]", s.steps_per_iteration);
                validate_function(f);
                space[name].push_back(std::move(f));
            }
        }
    for (const auto& kv : space) s.key.hp_set.push_back(kv.first);

    const json sampler = j.value("sampler", json{{"kind", "grid"}});
    const std::string kind = sampler.value("kind", std::string("grid"));
    if (!space.empty()) {
        std::vector<std::string> names;
        for (const auto& kv : space) names.push_back(kv.first);
        if (kind == "grid") {
            std::vector<std::size_t> idx(names.size(), 0);
            for (bool more = true; more;) {
                std::map<std::string, HpFunction> pick;
                for (std::size_t h = 0; h < names.size(); ++h) pick[names[h]] = space[names[h]][idx[h]];
                s.trials.push_back(make_trial(pick, s.max_steps));
                more = false;
                for (std::size_t h = names.size(); h-- > 0;) {
                    if (++idx[h] < space[names[h]].size()) {
                        more = true;
                        break;
                    }
                    idx[h] = 0;
                }
            }
        } else if (kind == "random") {
            std::uint64_t state = sampler.value("seed", std::uint64_t{0});
            const int n = sampler.at("trials").get<int>();
            for (int t = 0; t < n; ++t) {
                std::map<std::string, HpFunction> pick;
                for (const auto& name : names) pick[name] = space[name][splitmix(state) % space[name].size()];
                s.trials.push_back(make_trial(pick, s.max_steps));
            }
        } else {
            throw ConfigError("study spec: unknown sampler '" + kind + "'");
        }
    }
    if (j.contains("trials"))
        for (const auto& tj : j.at("trials")) {
            std::map<std::string, HpFunction> pick;
            for (const auto& [name, fj] : tj.at("hps").items())
                pick[name] = codec::function_in(fj, "trials.hps." + name, s.steps_per_iteration);
            if (s.key.hp_set.empty())
                for (const auto& kv : pick) s.key.hp_set.push_back(kv.first);
            s.trials.push_back(make_trial(pick, tj.value("steps", s.max_steps)));
        }
    if (s.trials.empty()) throw ConfigError("study spec: no trials");
    return s;
}

std::vector<TrialRequest> study_requests(const StudySpec& spec, StudyId study) {
    std::vector<TrialRequest> out;
    for (std::size_t i = 0; i < spec.trials.size(); ++i)
        out.push_back(TrialRequest{(static_cast<RequestId>(study) << 32) | static_cast<RequestId>(i), study,
                                   static_cast<TrialId>(i), spec.trials[i]});
    return out;
}

std::pair<StepCount, StepCount> merge_rate(const CompatKey& key, const std::vector<TrialConfig>& trials) {
    SearchPlan plan(key);
    StepCount total = 0;
    for (std::size_t i = 0; i < trials.size(); ++i) {
        plan.insert_trial(TrialRequest{static_cast<RequestId>(i), 0, static_cast<TrialId>(i), trials[i]});
        total += trials[i].total_steps;
    }
    StepCount unique = 0;
    for (const PlanNode& n : plan.nodes()) {
        StepCount hi = n.start_step;
        for (const auto& e : n.requests) hi = std::max(hi, e.end);
        for (NodeId c : n.children) hi = std::max(hi, plan.node(c).start_step);
        unique += hi - n.start_step;
    }
    return {total, unique};
}

}  // namespace stagemerge
