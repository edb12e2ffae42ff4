// Tuners (grid, SHA, ASHA, median stopping) and the driver that runs them over the engine
// (reference SPEC.md [MODULE] tuners; see stagemerge/tuner.hpp).
#include "stagemerge/tuner.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <set>

#include "json_codec.hpp"
#include "stagemerge/engine.hpp"

namespace stagemerge {

using codec::json;

std::string TunerAction::to_string() const {
    switch (kind) {
        case Kind::kSubmit: return "SUBMIT " + std::to_string(trial) + " " + std::to_string(end);
        case Kind::kExtend: return "EXTEND " + std::to_string(trial) + " " + std::to_string(end);
        case Kind::kStop: return "STOP " + std::to_string(trial);
        case Kind::kDone: {
            std::string s = "DONE ";
            for (std::size_t i = 0; i < winners.size(); ++i) s += (i ? "," : "") + std::to_string(winners[i]);
            return s;
        }
    }
    return "?";
}

TunerParams parse_tuner(const std::string& spec_json, const StudySpec& spec) {
    TunerParams p;
    p.max_steps = spec.max_steps;
    const json j = json::parse(spec_json);
    if (!j.contains("tuner")) return p;
    const json& t = j.at("tuner");
    const StepCount spi = spec.steps_per_iteration;
    p.kind = t.value("kind", std::string("grid"));
    if (p.kind != "grid" && p.kind != "sha" && p.kind != "asha" && p.kind != "median")
        throw ConfigError("tuner: unknown kind '" + p.kind + "'");
    p.reduction = t.value("reduction", 4);
    if (p.reduction < 2) throw ConfigError("tuner: reduction must be >= 2");
    p.min_steps = t.value("min", StepCount{0}) * spi;
    p.max_steps = t.contains("max") ? t.at("max").get<StepCount>() * spi : spec.max_steps;
    p.interval = t.value("interval", StepCount{0}) * spi;
    p.parallelism = t.value("parallelism", 0);
    p.metric = t.value("metric", std::string("val_loss"));
    const std::string mode = t.value("mode", std::string("min"));
    if (mode != "min" && mode != "max") throw ConfigError("tuner: mode must be min or max");
    p.maximize = mode == "max";
    if (t.contains("milestones")) {
        StepCount prev = 0;
        int prev_n = 0;
        for (const auto& m : t.at("milestones")) {
            const StepCount s = m.at(0).get<StepCount>() * spi;
            const int n = m.at(1).get<int>();
            if (s <= prev) throw ConfigError("tuner: milestones must be strictly increasing");
            if (prev_n && n >= prev_n) throw ConfigError("tuner: milestone survivor counts must strictly decrease");
            p.milestones.emplace_back(s, n);
            prev = s;
            prev_n = n;
        }
        if (p.milestones.empty()) throw ConfigError("tuner: empty milestone schedule");
        p.max_steps = p.milestones.back().first;
    }
    if (p.max_steps > spec.max_steps) throw ConfigError("tuner: max exceeds the study's max_steps");
    if (p.kind == "sha" || p.kind == "asha") {
        if (p.milestones.empty() && (p.min_steps < 1 || p.min_steps > p.max_steps))
            throw ConfigError("tuner: need 1 <= min <= max");
    }
    if (p.kind == "median") {
        if (p.interval < 1) throw ConfigError("tuner: median stopping needs interval >= 1");
        if (p.min_steps < 1) p.min_steps = p.interval;
    }
    return p;
}

Rungs sha_rungs(const TunerParams& p, int n_trials) {
    Rungs r;
    if (!p.milestones.empty()) {
        for (std::size_t i = 0; i < p.milestones.size(); ++i) {
            r.ends.push_back(p.milestones[i].first);
            r.survivors.push_back(i == 0 ? n_trials : std::min(p.milestones[i].second, r.survivors.back()));
        }
        return r;
    }
    StepCount e = p.min_steps;
    int n = n_trials;
    for (;;) {
        const StepCount capped = std::min(e, p.max_steps);
        r.ends.push_back(capped);
        r.survivors.push_back(n);
        if (capped >= p.max_steps) break;
        e *= p.reduction;
        n = (n + p.reduction - 1) / p.reduction;
    }
    return r;
}

namespace {

using Kind = TunerAction::Kind;

TunerAction submit(TrialId t, StepCount end) { return {Kind::kSubmit, t, end, {}}; }
TunerAction extend(TrialId t, StepCount end) { return {Kind::kExtend, t, end, {}}; }
TunerAction stop(TrialId t) { return {Kind::kStop, t, 0, {}}; }

/// Metric value oriented so that smaller is better.
double score(const TunerParams& p, const MetricRecord& m) {
    const auto it = m.find(p.metric);
    if (it == m.end()) throw ConfigError("tuner: metric '" + p.metric + "' missing from a rung result");
    return p.maximize ? -it->second : it->second;
}

/// Trials ordered best first (score, then smaller id).
std::vector<TrialId> ranked(const std::map<TrialId, double>& res) {
    std::vector<std::pair<double, TrialId>> v;
    for (const auto& [t, s] : res) v.emplace_back(s, t);
    std::sort(v.begin(), v.end());
    std::vector<TrialId> out;
    for (const auto& e : v) out.push_back(e.second);
    return out;
}

class GridTuner final : public Tuner {
public:
    GridTuner(TunerParams p, int n) : p_(std::move(p)), n_(n) {}
    std::vector<TunerAction> start() override {
        std::vector<TunerAction> a;
        for (TrialId t = 0; t < n_; ++t) a.push_back(submit(t, p_.max_steps));
        return a;
    }
    std::vector<TunerAction> on_result(TrialId t, StepCount end, const MetricRecord& m) override {
        if (done_ || end != p_.max_steps) return {};
        res_[t] = score(p_, m);
        if (static_cast<int>(res_.size()) < n_) return {};
        done_ = true;
        winners_ = {ranked(res_).front()};
        return {TunerAction{Kind::kDone, 0, 0, winners_}};
    }

private:
    TunerParams p_;
    int n_;
    std::map<TrialId, double> res_;
};

// Synchronous successive halving: wait for every participant of a rung, promote the top
// n_{i+1}, STOP the rest (SPEC.md sha_step).
class ShaTuner final : public Tuner {
public:
    ShaTuner(TunerParams p, int n) : p_(std::move(p)), rungs_(sha_rungs(p_, n)) {
        for (TrialId t = 0; t < n; ++t) part_.insert(t);
    }
    std::vector<TunerAction> start() override {
        std::vector<TunerAction> a;
        for (TrialId t : part_) a.push_back(submit(t, rungs_.ends[0]));
        return a;
    }
    std::vector<TunerAction> on_result(TrialId t, StepCount end, const MetricRecord& m) override {
        if (done_ || end != rungs_.ends[rung_] || !part_.count(t)) return {};
        res_[t] = score(p_, m);
        if (res_.size() < part_.size()) return {};
        const std::vector<TrialId> order = ranked(res_);
        std::vector<TunerAction> a;
        if (rung_ + 1 < rungs_.ends.size()) {
            const int keep = rungs_.survivors[rung_ + 1];
            part_.clear();
            for (int i = 0; i < static_cast<int>(order.size()); ++i) {
                if (i < keep) {
                    part_.insert(order[static_cast<std::size_t>(i)]);
                    a.push_back(extend(order[static_cast<std::size_t>(i)], rungs_.ends[rung_ + 1]));
                } else {
                    a.push_back(stop(order[static_cast<std::size_t>(i)]));
                }
            }
            ++rung_;
            res_.clear();
            return a;
        }
        const int keep = p_.milestones.empty()
                             ? (static_cast<int>(order.size()) + p_.reduction - 1) / p_.reduction
                             : static_cast<int>(order.size());
        winners_.assign(order.begin(), order.begin() + keep);
        done_ = true;
        a.push_back(TunerAction{Kind::kDone, 0, 0, winners_});
        return a;
    }

private:
    TunerParams p_;
    Rungs rungs_;
    std::size_t rung_ = 0;
    std::set<TrialId> part_;
    std::map<TrialId, double> res_;
};

// Asynchronous successive halving (SPEC.md asha_step): a finishing trial is promoted iff it
// ranks in the top ceil(count/eta) of the results recorded so far at its rung and that rung still
// has an unused promotion; otherwise it stops and the next unstarted trial begins.
class AshaTuner final : public Tuner {
public:
    AshaTuner(TunerParams p, int n) : p_(std::move(p)), n_(n), rungs_(sha_rungs(p_, n)) {
        res_.resize(rungs_.ends.size());
        promoted_.assign(rungs_.ends.size(), 0);
        par_ = p_.parallelism > 0 ? std::min(p_.parallelism, n_) : n_;
    }
    std::vector<TunerAction> start() override {
        std::vector<TunerAction> a;
        while (next_ < par_) a.push_back(launch());
        return a;
    }
    std::vector<TunerAction> on_result(TrialId t, StepCount end, const MetricRecord& m) override {
        auto cur = at_.find(t);
        if (done_ || cur == at_.end() || rungs_.ends[cur->second] != end) return {};
        const std::size_t k = cur->second;
        res_[k][t] = score(p_, m);
        --in_flight_;
        std::vector<TunerAction> a;
        bool promoted = false;
        if (k + 1 < rungs_.ends.size()) {
            const int quota = (static_cast<int>(res_[k].size()) + p_.reduction - 1) / p_.reduction;
            const std::vector<TrialId> order = ranked(res_[k]);
            const int rank = static_cast<int>(std::find(order.begin(), order.end(), t) - order.begin());
            if (rank < quota && promoted_[k] < quota) {
                promoted_[k] += 1;
                cur->second = k + 1;
                ++in_flight_;
                a.push_back(extend(t, rungs_.ends[k + 1]));
                promoted = true;
            }
        }
        if (!promoted) {
            at_.erase(cur);
            if (k + 1 < rungs_.ends.size()) a.push_back(stop(t));
            if (next_ < n_) a.push_back(launch());
        }
        if (in_flight_ == 0 && next_ >= n_) {
            for (std::size_t r = res_.size(); r-- > 0;)
                if (!res_[r].empty()) {
                    winners_ = {ranked(res_[r]).front()};
                    break;
                }
            done_ = true;
            a.push_back(TunerAction{Kind::kDone, 0, 0, winners_});
        }
        return a;
    }

private:
    TunerAction launch() {
        const TrialId t = next_++;
        at_[t] = 0;
        ++in_flight_;
        return submit(t, rungs_.ends[0]);
    }
    TunerParams p_;
    int n_, par_ = 0;
    Rungs rungs_;
    std::vector<std::map<TrialId, double>> res_;
    std::vector<int> promoted_;
    std::map<TrialId, std::size_t> at_;  // trial -> rung it is training towards
    TrialId next_ = 0;
    int in_flight_ = 0;
};

// Median stopping (SPEC.md median_stop): trials report at milestones min, min+interval, ...;
// a trial whose best score so far is strictly worse than the median of the other trials'
// running averages at the same milestone stops.
class MedianTuner final : public Tuner {
public:
    MedianTuner(TunerParams p, int n) : p_(std::move(p)), n_(n) {
        par_ = p_.parallelism > 0 ? std::min(p_.parallelism, n_) : n_;
        for (StepCount s = p_.min_steps; s < p_.max_steps; s += p_.interval) marks_.push_back(s);
        marks_.push_back(p_.max_steps);
    }
    std::vector<TunerAction> start() override {
        std::vector<TunerAction> a;
        while (next_ < par_) a.push_back(launch());
        return a;
    }
    std::vector<TunerAction> on_result(TrialId t, StepCount end, const MetricRecord& m) override {
        auto cur = at_.find(t);
        if (done_ || cur == at_.end() || marks_[cur->second] != end) return {};
        const std::size_t j = cur->second;
        const double s = score(p_, m);
        auto& h = hist_[t];
        h.push_back(s);
        // others' running averages over their reports up to this milestone
        std::vector<double> avgs;
        for (const auto& [o, oh] : hist_) {
            if (o == t || oh.size() <= j) continue;
            double sum = 0;
            for (std::size_t i = 0; i <= j; ++i) sum += oh[i];
            avgs.push_back(sum / static_cast<double>(j + 1));
        }
        bool stop_it = false;
        if (!avgs.empty()) {
            std::sort(avgs.begin(), avgs.end());
            const std::size_t k = avgs.size();
            const double med = k % 2 ? avgs[k / 2] : 0.5 * (avgs[k / 2 - 1] + avgs[k / 2]);
            const double best = *std::min_element(h.begin(), h.end());
            stop_it = best > med;
        }
        std::vector<TunerAction> a;
        --in_flight_;
        if (!stop_it && j + 1 < marks_.size()) {
            cur->second = j + 1;
            ++in_flight_;
            a.push_back(extend(t, marks_[j + 1]));
        } else {
            if (j + 1 >= marks_.size()) final_[t] = s;
            if (stop_it) a.push_back(stop(t));
            at_.erase(cur);
            if (next_ < n_) a.push_back(launch());
        }
        if (in_flight_ == 0 && next_ >= n_) {
            if (!final_.empty()) winners_ = {ranked(final_).front()};
            done_ = true;
            a.push_back(TunerAction{Kind::kDone, 0, 0, winners_});
        }
        return a;
    }

private:
    TunerAction launch() {
        const TrialId t = next_++;
        at_[t] = 0;
        ++in_flight_;
        return submit(t, marks_[0]);
    }
    TunerParams p_;
    int n_, par_ = 0;
    std::vector<StepCount> marks_;
    std::map<TrialId, std::vector<double>> hist_;
    std::map<TrialId, std::size_t> at_;
    std::map<TrialId, double> final_;
    TrialId next_ = 0;
    int in_flight_ = 0;
};

}  // namespace

std::unique_ptr<Tuner> make_tuner(const TunerParams& p, int n_trials, StepCount max_steps) {
    TunerParams q = p;
    if (q.max_steps <= 0) q.max_steps = max_steps;
    if (n_trials < 1) throw ConfigError("tuner: study has no trials");
    if (q.kind == "grid") return std::make_unique<GridTuner>(q, n_trials);
    if (q.kind == "sha") return std::make_unique<ShaTuner>(q, n_trials);
    if (q.kind == "asha") return std::make_unique<AshaTuner>(q, n_trials);
    if (q.kind == "median") return std::make_unique<MedianTuner>(q, n_trials);
    throw ConfigError("tuner: unknown kind '" + q.kind + "'");
}

std::vector<StudyOutcome> run_tuned_studies(Engine& engine, const std::vector<std::string>& spec_jsons,
                                            StudyId base_study) {
    struct Run {
        StudySpec spec;
        std::unique_ptr<Tuner> tuner;
        StudyOutcome out;
        std::int64_t seq = 0;
    };
    std::vector<Run> runs(spec_jsons.size());
    for (std::size_t i = 0; i < spec_jsons.size(); ++i) {
        Run& r = runs[i];
        r.spec = parse_study(spec_jsons[i]);
        const TunerParams p = parse_tuner(spec_jsons[i], r.spec);
        r.tuner = make_tuner(p, static_cast<int>(r.spec.trials.size()), r.spec.max_steps);
        r.out.study = base_study + static_cast<StudyId>(i);
    }
    auto run_of = [&](StudyId s) -> Run& {
        const auto i = static_cast<std::size_t>(s - base_study);
        if (s < base_study || i >= runs.size()) throw IntegrityError("completion for an unknown study");
        return runs[i];
    };

    // results delivered synchronously by the plan (kImmediate) are queued, not re-entered
    std::deque<std::tuple<StudyId, TrialId, StepCount, MetricRecord>> ready;
    auto apply = [&](Run& r, const std::vector<TunerAction>& acts) {
        for (const TunerAction& a : acts) {
            r.out.actions.push_back(a.to_string());
            const TrialRef ref{r.out.study, a.trial};
            switch (a.kind) {
                case Kind::kSubmit:
                case Kind::kExtend: {
                    const TrialConfig& full = r.spec.trials.at(static_cast<std::size_t>(a.trial));
                    TrialRequest req{(static_cast<RequestId>(r.out.study) << 32) | r.seq++, r.out.study, a.trial,
                                     truncate_config(full, a.end)};
                    const InsertOutcome o = engine.submit(req);
                    if (o.kind == InsertOutcome::Kind::kImmediate) ready.emplace_back(r.out.study, a.trial, a.end, o.metrics);
                    break;
                }
                case Kind::kStop: engine.cancel(ref); break;
                case Kind::kDone: r.out.winners = a.winners; break;
            }
        }
    };
    auto deliver = [&](StudyId s, TrialId t, StepCount end, const MetricRecord& m) {
        Run& r = run_of(s);
        auto& reached = r.out.trained_to[t];
        reached = std::max(reached, end);
        apply(r, r.tuner->on_result(t, end, m));
    };
    auto drain = [&] {
        while (!ready.empty()) {
            auto [s, t, e, m] = ready.front();
            ready.pop_front();
            deliver(s, t, e, m);
        }
    };

    auto previous = engine.completion_callback();
    engine.on_complete([&](Engine&, const CompletedRequest& c) {
        for (const TrialRef& t : c.subscribers) deliver(t.study, t.trial, c.end, c.metrics);
        drain();
    });
    try {
        for (Run& r : runs) apply(r, r.tuner->start());
        drain();
        engine.run();
    } catch (...) {
        engine.on_complete(previous);
        throw;
    }
    engine.on_complete(previous);

    std::vector<StudyOutcome> out;
    for (Run& r : runs) {
        if (!r.tuner->done()) throw IntegrityError("study '" + r.spec.name + "' ended before its tuner was DONE");
        for (const auto& [t, e] : r.out.trained_to) r.out.trial_steps += e;
        out.push_back(std::move(r.out));
    }
    return out;
}

}  // namespace stagemerge
