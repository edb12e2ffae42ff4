"""Tuner state machines (C++ host library) against the reference SPEC's examples and independent
Python restatements (SPEC.md [MODULE] tuners: sha_step, asha_step, median_stop, grid).

Metric tables are fixed, so every decision sequence is a pure function of (spec, metrics); the
simulation feeds results back first-in first-out.  No GPU: the engine-driven runs are in
test_tuner_gpu.py.
"""
import json
import math
import random

import pytest

from paper_2006_11972_b200 import host


def spec(n_trials, tuner, max_steps=120, spi=1):
    """A study of n distinct constant-lr trials (the configs do not matter to the tuner)."""
    return json.dumps({
        "schema": 1, "name": "t", "max_steps": max_steps, "steps_per_iteration": spi,
        "trials": [{"hps": {"lr": {"family": "constant", "value": f"0.{i + 1:04d}"}}} for i in range(n_trials)],
        "tuner": tuner})


def simulate(spec_json, metric):
    """Drive a tuner FIFO: metric(trial, end) -> val_loss.  Returns (actions, winners)."""
    t = host.Tuner(spec_json)
    log, queue = [], []

    def take(acts):
        for a in acts:
            log.append(a)
            parts = a.split()
            if parts[0] in ("SUBMIT", "EXTEND"):
                queue.append((int(parts[1]), int(parts[2])))

    take(t.start())
    while queue:
        tr, end = queue.pop(0)
        take(t.on_result(tr, end, {"val_loss": metric(tr, end), "val_acc": 0.5}))
    assert t.done()
    return log, t.winners()


# ---------------------------------------------------------------- independent restatements

def sha_oracle(n, rungs, eta, metric, milestone_mode=False, survivors=None):
    part = list(range(n))
    acts = [f"SUBMIT {t} {rungs[0]}" for t in part]
    for i, end in enumerate(rungs):
        order = sorted(part, key=lambda t: (metric(t, end), t))
        if i + 1 < len(rungs):
            keep = survivors[i + 1] if survivors else math.ceil(len(part) / eta)
            for j, t in enumerate(order):
                acts.append(f"EXTEND {t} {rungs[i + 1]}" if j < keep else f"STOP {t}")
            part = order[:keep]
        else:
            keep = len(order) if milestone_mode else math.ceil(len(order) / eta)
            win = order[:keep]
            acts.append("DONE " + ",".join(map(str, win)))
            return acts, win


def asha_oracle(n, rungs, eta, par, metric):
    acts, queue, res, promoted = [], [], [dict() for _ in rungs], [0] * len(rungs)
    nxt = 0

    def launch():
        nonlocal nxt
        acts.append(f"SUBMIT {nxt} {rungs[0]}")
        queue.append((nxt, 0))
        nxt += 1

    while nxt < min(par, n):
        launch()
    while queue:
        t, k = queue.pop(0)
        res[k][t] = metric(t, rungs[k])
        if k + 1 < len(rungs):
            quota = math.ceil(len(res[k]) / eta)
            order = sorted(res[k], key=lambda x: (res[k][x], x))
            if order.index(t) < quota and promoted[k] < quota:
                promoted[k] += 1
                acts.append(f"EXTEND {t} {rungs[k + 1]}")
                queue.append((t, k + 1))
                continue
            acts.append(f"STOP {t}")
        if nxt < n:
            launch()
    best = next(r for r in reversed(res) if r)
    win = min(best, key=lambda x: (best[x], x))
    acts.append(f"DONE {win}")
    return acts, [win]


# ---------------------------------------------------------------- SHA

def test_sha_rungs_table1():
    s = host.study_spec("c4_sha")
    ends, surv = host.sha_rungs(s)
    assert ends == [150, 600, 1200]          # 15 / 60 / 120 iterations x 10 steps
    assert surv == [448, 112, 28]


def test_sha_table1_survivor_counts():
    """448 trials, eta 4: 448 -> 112 -> 28 -> 7 (SPEC.md sha_step example)."""
    s = spec(448, {"kind": "sha", "reduction": 4, "min": 15, "max": 120}, max_steps=120)
    rnd = random.Random(7)
    table = {(t, e): rnd.random() for t in range(448) for e in (15, 60, 120)}
    acts, win = simulate(s, lambda t, e: table[(t, e)])
    ext = [a for a in acts if a.startswith("EXTEND")]
    assert sum(a.endswith(" 60") for a in ext) == 112
    assert sum(a.endswith(" 120") for a in ext) == 28
    assert sum(a.startswith("STOP") for a in acts) == 448 - 112 + 112 - 28
    assert len(win) == 7
    want, wwin = sha_oracle(448, [15, 60, 120], 4, lambda t, e: table[(t, e)])
    assert acts == want and win == wwin


def test_sha_fig10_milestones():
    """Schedule.from_milestones((5, 8), (10, 4)): 8 trials to step 5, STOP 4, 4 more to 10."""
    s = spec(8, {"kind": "sha", "milestones": [[5, 8], [10, 4]]}, max_steps=10)
    acts, win = simulate(s, lambda t, e: (t * 37 % 8) + e * 0.01)
    assert [a for a in acts if a.startswith("SUBMIT")] == [f"SUBMIT {t} 5" for t in range(8)]
    assert sum(a.startswith("STOP") for a in acts) == 4
    assert sum(a.startswith("EXTEND") for a in acts) == 4
    assert len(win) == 4
    want, _ = sha_oracle(8, [5, 10], 2, lambda t, e: (t * 37 % 8) + e * 0.01, milestone_mode=True,
                         survivors=[8, 4])
    assert acts == want


def test_sha_single_trial_trains_to_max():
    s = spec(1, {"kind": "sha", "reduction": 4, "min": 15, "max": 120})
    acts, win = simulate(s, lambda t, e: 1.0)
    assert acts == ["SUBMIT 0 15", "EXTEND 0 60", "EXTEND 0 120", "DONE 0"] and win == [0]


def test_sha_ties_smaller_id_survives():
    s = spec(4, {"kind": "sha", "reduction": 4, "min": 10, "max": 20}, max_steps=20)
    acts, win = simulate(s, lambda t, e: 0.5)
    assert "EXTEND 0 20" in acts and win == [0]


def test_sha_randomised_vs_oracle():
    rnd = random.Random(3)
    for _ in range(20):
        n = rnd.randint(1, 60)
        eta = rnd.choice([2, 3, 4])
        mn = rnd.randint(1, 10)
        mx = mn * eta ** rnd.randint(0, 3) + rnd.randint(0, 3)
        s = spec(n, {"kind": "sha", "reduction": eta, "min": mn, "max": mx}, max_steps=mx)
        ends, _ = host.sha_rungs(s)
        table = {}
        f = lambda t, e: table.setdefault((t, e), round(rnd.random(), 2))  # ties happen
        acts, win = simulate(s, f)
        want, wwin = sha_oracle(n, ends, eta, lambda t, e: table[(t, e)])
        assert acts == want and win == wwin


def test_metric_mode_max_and_missing_metric():
    s = json.loads(spec(4, {"kind": "sha", "reduction": 4, "min": 10, "max": 20, "metric": "val_acc",
                            "mode": "max"}, max_steps=20))
    t = host.Tuner(json.dumps(s))
    t.start()
    for i in range(4):
        acts = t.on_result(i, 10, {"val_acc": i / 10, "val_loss": 0.0})
    assert "EXTEND 3 20" in acts                                  # highest accuracy survives
    t2 = host.Tuner(json.dumps(s))
    t2.start()
    with pytest.raises(ValueError, match="metric"):
        t2.on_result(0, 10, {"val_loss": 1.0})


def test_bad_tuner_specs():
    for bad in ({"kind": "pbt"}, {"kind": "sha", "reduction": 1, "min": 1, "max": 4},
                {"kind": "sha", "min": 0, "max": 4}, {"kind": "sha", "milestones": [[5, 8], [4, 2]]},
                {"kind": "sha", "milestones": [[5, 8], [10, 8]]}, {"kind": "median"},
                {"kind": "sha", "min": 10, "max": 1000}):
        with pytest.raises(ValueError):
            host.Tuner(spec(4, bad))


# ---------------------------------------------------------------- ASHA

def test_asha_first_trial_promoted_and_low_rank_not():
    s = spec(8, {"kind": "asha", "reduction": 4, "min": 10, "max": 40, "parallelism": 2}, max_steps=40)
    t = host.Tuner(s)
    assert t.start() == ["SUBMIT 0 10", "SUBMIT 1 10"]
    assert t.on_result(0, 10, {"val_loss": 0.5}) == ["EXTEND 0 40"]      # top-1 of 1
    assert t.on_result(1, 10, {"val_loss": 0.9}) == ["STOP 1", "SUBMIT 2 10"]  # below the 1/4 quantile


def test_asha_randomised_vs_oracle():
    rnd = random.Random(11)
    for _ in range(20):
        n = rnd.randint(1, 80)
        eta = rnd.choice([2, 3, 4])
        par = rnd.randint(1, 16)
        s = spec(n, {"kind": "asha", "reduction": eta, "min": 5, "max": 5 * eta * eta, "parallelism": par},
                 max_steps=5 * eta * eta)
        ends, _ = host.sha_rungs(s)
        table = {(t, e): round(rnd.random(), 2) for t in range(n) for e in ends}
        acts, win = simulate(s, lambda t, e: table[(t, e)])
        want, wwin = asha_oracle(n, ends, eta, par, lambda t, e: table[(t, e)])
        assert acts == want and win == wwin


def test_asha_table1_spec_runs_to_done():
    s = host.study_spec("c4_asha")
    rnd = random.Random(5)
    acts, win = simulate(s, lambda t, e: rnd.random())
    assert acts[-1].startswith("DONE") and len(win) == 1
    assert sum(a.startswith("SUBMIT") for a in acts) == 448


# ---------------------------------------------------------------- median stopping / grid

def test_median_stopping_examples():
    s = spec(3, {"kind": "median", "interval": 10, "min": 10, "parallelism": 3}, max_steps=30)
    t = host.Tuner(s)
    assert t.start() == ["SUBMIT 0 10", "SUBMIT 1 10", "SUBMIT 2 10"]
    assert t.on_result(0, 10, {"val_loss": 0.5}) == ["EXTEND 0 20"]      # nobody else reported yet
    assert t.on_result(1, 10, {"val_loss": 0.5}) == ["EXTEND 1 20"]      # at the median: continues
    assert t.on_result(2, 10, {"val_loss": 9.0}) == ["STOP 2"]           # diverged: stops
    single = host.Tuner(spec(1, {"kind": "median", "interval": 10}, max_steps=20))
    single.start()
    assert single.on_result(0, 10, {"val_loss": 5.0}) == ["EXTEND 0 20"]
    assert single.on_result(0, 20, {"val_loss": 5.0}) == ["DONE 0"]


def test_grid_tuner_done_with_best():
    s = spec(5, {"kind": "grid"}, max_steps=50)
    acts, win = simulate(s, lambda t, e: abs(t - 3))
    assert acts[:5] == [f"SUBMIT {t} 50" for t in range(5)] and win == [3]


# ---------------------------------------------------------------- acceptance 7

def simulate_seeded(spec_json, metric, rng):
    """Like simulate(), but the next completion is a seeded random pick among in-flight jobs."""
    t = host.Tuner(spec_json)
    log, inflight = [], []

    def take(acts):
        for a in acts:
            log.append(a)
            parts = a.split()
            if parts[0] in ("SUBMIT", "EXTEND"):
                inflight.append((int(parts[1]), int(parts[2])))

    take(t.start())
    while inflight:
        tr, end = inflight.pop(rng.randrange(len(inflight)))
        take(t.on_result(tr, end, {"val_loss": metric(tr, end), "val_acc": 0.5}))
    assert t.done()
    return log, t.winners()


def asha_sequential_reference(n, rungs, eta, par, metric, rng):
    """The published ASHA rule (Li et al. 2020, Alg. 2) run sequentially: a finishing job is
    promoted iff it ranks in the top ceil(|rung| / eta) of its rung and the rung still has a
    promotion left; otherwise the next fresh trial starts.  Completion order drawn from `rng`
    exactly as simulate_seeded draws it."""
    acts, inflight, res, promoted = [], [], [dict() for _ in rungs], [0] * len(rungs)
    nxt = 0

    def launch():
        nonlocal nxt
        acts.append(f"SUBMIT {nxt} {rungs[0]}")
        inflight.append((nxt, rungs[0]))
        nxt += 1

    while nxt < min(par, n):
        launch()
    while inflight:
        t, end = inflight.pop(rng.randrange(len(inflight)))
        k = rungs.index(end)
        res[k][t] = metric(t, end)
        if k + 1 < len(rungs):
            quota = math.ceil(len(res[k]) / eta)
            order = sorted(res[k], key=lambda x: (res[k][x], x))
            if order.index(t) < quota and promoted[k] < quota:
                promoted[k] += 1
                acts.append(f"EXTEND {t} {rungs[k + 1]}")
                inflight.append((t, rungs[k + 1]))
                continue
            acts.append(f"STOP {t}")
        if nxt < n:
            launch()
    best = next(r for r in reversed(res) if r)
    win = min(best, key=lambda x: (best[x], x))
    acts.append(f"DONE {win}")
    return acts, [win]


RECORDED = random.Random(2020)
ASHA_TABLE = {(t, e): round(RECORDED.random(), 3) for t in range(20) for e in (5, 15, 45)}


@pytest.mark.parametrize("seed", range(200))
def test_asha_200_completion_orders(seed):
    """SPEC acceptance 7: a fixed recorded metric table (20 trials, 3 rungs 5 / 15 / 45), 200
    seeded completion orders: the tuner's asynchronous promotion sequence equals the sequential
    reference of the ASHA rule for every order."""
    s = spec(20, {"kind": "asha", "reduction": 3, "min": 5, "max": 45, "parallelism": 6}, max_steps=45)
    assert host.sha_rungs(s)[0] == [5, 15, 45]
    acts, win = simulate_seeded(s, lambda t, e: ASHA_TABLE[(t, e)], random.Random(seed))
    want, wwin = asha_sequential_reference(20, [5, 15, 45], 3, 6, lambda t, e: ASHA_TABLE[(t, e)],
                                           random.Random(seed))
    assert acts == want and win == wwin
