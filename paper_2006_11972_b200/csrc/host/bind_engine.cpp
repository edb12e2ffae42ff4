// pybind11 marshalling for the Engine and study helpers (see bind.cpp).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "json_codec.hpp"
#include "stagemerge/engine.hpp"
#include "stagemerge/study.hpp"
#include "stagemerge/tuner.hpp"

namespace py = pybind11;
using namespace stagemerge;
using codec::json;

namespace {

EngineOptions options_from(const json& o) {
    EngineOptions e;
    if (o.contains("devices")) e.devices = o.at("devices").get<std::vector<int>>();
    e.slots_per_gpu = o.value("slots_per_gpu", e.slots_per_gpu);
    e.ckpts_per_gpu = o.value("ckpts_per_gpu", e.ckpts_per_gpu);
    e.gemm_mode = o.value("gemm_mode", e.gemm_mode);
    e.max_steps = o.value("max_steps", e.max_steps);
    e.max_batch = o.value("max_batch", e.max_batch);
    e.n_train = o.value("n_train", e.n_train);
    e.n_val = o.value("n_val", e.n_val);
    e.seed = o.value("seed", e.seed);
    if (o.contains("eval_intervals")) e.eval_intervals = o.at("eval_intervals").get<std::vector<StepCount>>();
    e.trial_mode = o.value("trial_mode", false);
    e.use_graphs = o.value("use_graphs", true);
    e.hp_lr = o.value("hp_lr", e.hp_lr);
    e.hp_momentum = o.value("hp_momentum", e.hp_momentum);
    e.hp_wd = o.value("hp_wd", e.hp_wd);
    e.hp_bs = o.value("hp_bs", e.hp_bs);
    e.default_lr = o.value("default_lr", e.default_lr);
    e.default_momentum = o.value("default_momentum", e.default_momentum);
    e.default_wd = o.value("default_wd", e.default_wd);
    e.default_bs = o.value("default_bs", e.default_bs);
    e.rank = o.value("rank", 0);
    e.world = o.value("world", 1);
    if (o.contains("step_cost_us"))
        for (const auto& [k, v] : o.at("step_cost_us").items()) e.step_cost_us[std::stoi(k)] = v.get<double>();
    e.ckpt_gc = o.value("ckpt_gc", e.ckpt_gc);
    return e;
}

json stats_json(const EngineStats& s) {
    return {{"wall_s", s.wall_s},         {"locksteps", s.locksteps}, {"stage_steps", s.stage_steps},
            {"trial_steps", s.trial_steps}, {"saves", s.saves},       {"loads", s.loads},
            {"inits", s.inits},           {"peer_copies", s.peer_copies}, {"evals", s.evals},
            {"assignments", s.assignments}, {"spills", s.spills},     {"kernel_launches", s.kernel_launches},
            {"h2d_bytes", s.h2d_bytes},   {"d2h_bytes", s.d2h_bytes},   {"releases", s.releases},
            {"gc_frees", s.gc_frees},     {"model_busy_us", s.model_busy_us}, {"model_wall_us", s.model_wall_us}};
}

template <class F>
auto translate(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const ConfigError& e) {
        throw py::value_error(std::string("ConfigError: ") + e.what());
    } catch (const IntegrityError& e) {
        throw std::runtime_error(std::string("IntegrityError: ") + e.what());
    }
}

}  // namespace

void bind_engine(py::module_& m) {
    py::class_<Engine>(m, "Engine", py::module_local())
        .def(py::init([](const std::string& key_json, const std::string& opts_json) {
                 const json k = json::parse(key_json);
                 CompatKey key{k.at("model").get<std::string>(), k.at("dataset").get<std::string>(),
                               k.at("hp_set").get<std::vector<std::string>>()};
                 return translate([&] { return std::make_unique<Engine>(key, options_from(json::parse(opts_json))); });
             }),
             py::arg("key_json"), py::arg("options_json") = "{}")
        .def("submit_study",
             [](Engine& e, const std::string& spec_json, int study) {
                 return translate([&] {
                     const StudySpec spec = parse_study(spec_json);
                     int pending = 0;
                     for (const auto& r : study_requests(spec, study))
                         pending += e.submit(r).kind == InsertOutcome::Kind::kPending;
                     return pending;
                 });
             },
             py::arg("spec_json"), py::arg("study") = 0)
        .def("submit",
             [](Engine& e, const std::string& trial_json, long long id, int study, int trial) {
                 return translate([&] {
                     TrialRequest r{id, study, trial, codec::config_in(json::parse(trial_json))};
                     const InsertOutcome o = e.submit(r);
                     return std::make_tuple(o.kind == InsertOutcome::Kind::kPending, o.node, o.request_id);
                 });
             })
        .def("cancel", [](Engine& e, int study, int trial) { return e.cancel(TrialRef{study, trial}); })
        .def("run_tuned",
             [](Engine& e, const std::vector<std::string>& specs, int base) {
                 py::gil_scoped_release nogil;
                 return translate([&] {
                     json out = json::array();
                     for (const StudyOutcome& o : run_tuned_studies(e, specs, base)) {
                         json tt = json::object();
                         for (const auto& [t, s] : o.trained_to) tt[std::to_string(t)] = s;
                         out.push_back({{"study", o.study}, {"winners", o.winners}, {"actions", o.actions},
                                        {"trained_to", tt}, {"trial_steps", o.trial_steps}});
                     }
                     return out.dump();
                 });
             },
             py::arg("specs"), py::arg("base_study") = 0)
        .def("run",
             [](Engine& e) {
                 py::gil_scoped_release nogil;
                 translate([&] { e.run(); });
             })
        .def("reset", [](Engine& e) { translate([&] { e.reset(); }); })
        .def("trace",
             [](Engine& e) {
                 std::vector<std::tuple<long long, int, std::string, long long, long long, long long, std::string>> v;
                 for (const TraceEvent& t : e.trace()) v.emplace_back(t.time, t.worker, t.kind, t.node, t.start, t.end, t.detail);
                 return v;
             })
        .def("on_complete",
             [](Engine& e, py::object fn) {
                 if (fn.is_none()) {
                     e.on_complete(nullptr);
                     return;
                 }
                 // called from run() (GIL released there): take the GIL for the Python callback
                 e.on_complete([fn](Engine&, const CompletedRequest& c) {
                     py::gil_scoped_acquire gil;
                     std::vector<std::pair<int, int>> subs;
                     for (const TrialRef& t : c.subscribers) subs.emplace_back(t.study, t.trial);
                     fn(c.node, c.end, subs);
                 });
             })
        .def("collect_checkpoints", [](Engine& e) { return translate([&] { return e.collect_checkpoints(); }); })
        .def("calibrate",
             [](Engine& e, const std::vector<int>& bss) {
                 py::gil_scoped_release nogil;
                 translate([&] { e.calibrate(bss); });
             })
        .def("step_cost_us", [](Engine& e) { return e.options().step_cost_us; })
        .def("node_runtime", [](Engine& e, long long n) { return e.plan().node(n).runtime_sec_per_step; })
        .def("stats", [](Engine& e) { return stats_json(e.stats()).dump(); })
        .def("signature", [](Engine& e) { return e.plan().signature(); })
        .def("plan_json", [](Engine& e) { return e.plan().to_json(); })
        .def("node_count", [](Engine& e) { return e.plan().node_count(); })
        .def("has_pending", [](Engine& e) { return e.plan().has_pending(); })
        .def("trials",
             [](Engine& e) {
                 std::vector<std::pair<int, int>> v;
                 for (const auto& t : e.trials()) v.emplace_back(t.study, t.trial);
                 return v;
             })
        .def("trial_end", [](Engine& e, int s, int t) { return e.trial_end(TrialRef{s, t}); })
        .def("history",
             [](Engine& e, int s, int t) {
                 std::vector<std::tuple<long long, double, double>> v;
                 for (const auto& [step, rec] : e.history(TrialRef{s, t}))
                     v.emplace_back(step, rec.count("val_loss") ? rec.at("val_loss") : 0.0,
                                    rec.count("val_acc") ? rec.at("val_acc") : 0.0);
                 return v;
             })
        .def("owned_roots",
             [](Engine& e) {
                 const std::set<NodeId> own = e.owned_roots();
                 return std::vector<NodeId>(own.begin(), own.end());
             })
        .def("dataset_digest", [](Engine& e) { return e.dataset_digest(); })
        .def("context_ptrs",
             [](Engine& e) {
                 std::vector<std::uintptr_t> v;
                 for (auto* c : e.contexts()) v.push_back(reinterpret_cast<std::uintptr_t>(c));
                 return v;
             })
        .def("upload_dataset_ptrs",
             [](Engine& e, std::uintptr_t x, std::uintptr_t y, std::uintptr_t vx, std::uintptr_t vy) {
                 py::gil_scoped_release nogil;
                 e.upload_dataset(reinterpret_cast<const float*>(x), reinterpret_cast<const std::int32_t*>(y),
                                  reinterpret_cast<const float*>(vx), reinterpret_cast<const std::int32_t*>(vy));
             });

    // Pure tuner state machine (no engine): start() / on_result() -> action strings.
    struct PyTuner {
        std::unique_ptr<Tuner> t;
    };
    py::class_<PyTuner>(m, "Tuner", py::module_local())
        .def(py::init([](const std::string& spec_json) {
            return translate([&] {
                const StudySpec spec = parse_study(spec_json);
                const TunerParams p = parse_tuner(spec_json, spec);
                return PyTuner{make_tuner(p, static_cast<int>(spec.trials.size()), spec.max_steps)};
            });
        }))
        .def("start",
             [](PyTuner& t) {
                 std::vector<std::string> v;
                 for (const auto& a : translate([&] { return t.t->start(); })) v.push_back(a.to_string());
                 return v;
             })
        .def("on_result",
             [](PyTuner& t, int trial, long long end, const std::map<std::string, double>& metrics) {
                 std::vector<std::string> v;
                 for (const auto& a : translate([&] { return t.t->on_result(trial, end, metrics); }))
                     v.push_back(a.to_string());
                 return v;
             })
        .def("done", [](PyTuner& t) { return t.t->done(); })
        .def("winners", [](PyTuner& t) { return t.t->winners(); });
    m.def("sha_rungs", [](const std::string& spec_json) {
        return translate([&] {
            const StudySpec spec = parse_study(spec_json);
            const Rungs r = sha_rungs(parse_tuner(spec_json, spec), static_cast<int>(spec.trials.size()));
            return std::make_pair(r.ends, r.survivors);
        });
    });

    // merge rate p (one study) or q (several, SPEC.md analysis kwise_merge_rate) over one plan
    m.def("merge_rate_specs", [](const std::vector<std::string>& specs) {
        return translate([&] {
            std::vector<TrialConfig> all;
            CompatKey key;
            for (std::size_t i = 0; i < specs.size(); ++i) {
                const StudySpec s = parse_study(specs[i]);
                if (i == 0)
                    key = s.key;
                else if (!(s.key == key))
                    throw ConfigError("merge-rate: studies have different compatibility keys");
                all.insert(all.end(), s.trials.begin(), s.trials.end());
            }
            return merge_rate(key, all);
        });
    });

    m.def("expand_study", [](const std::string& spec_json) {
        return translate([&] {
            const StudySpec s = parse_study(spec_json);
            json out = {{"name", s.name},
                        {"key", {{"model", s.key.model}, {"dataset", s.key.dataset}, {"hp_set", s.key.hp_set}}},
                        {"max_steps", s.max_steps},
                        {"eval_interval", s.eval_interval}};
            json trials = json::array();
            for (const auto& t : s.trials) trials.push_back(codec::config_out(t));
            out["trials"] = trials;
            const auto [total, unique] = merge_rate(s.key, s.trials);
            out["total_steps"] = total;
            out["unique_steps"] = unique;
            return out.dump();
        });
    });
}
