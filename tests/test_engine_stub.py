"""The C++ engine (plan + stage trees + scheduler + lockstep event loop + checkpoint pool) on a
host-only executor stub (tests/native/smx_stub.cpp), so scheduling properties are checked on
CPU at scale.  The stub's "model state" is a digest of the hp rows a slot trained on, so equal
metrics <=> equal hp prefix, and a wrong LOAD / missing hp upload shows up as a conflict.

SPEC acceptance 8: with at least as many workers as leaves the makespan equals the
critical path, and with one worker it equals the unique stage-steps (NewCheckpoint unlocks
children).  Plus STAGE == TRIAL metric histories (acceptance 5)
and the savings law on random studies."""
import json
import random
import sys
from pathlib import Path

import pytest

from hostgen import rand_config, shared_space

sys.path.insert(0, str(Path(__file__).resolve().parent / "native"))
stub = pytest.importorskip("_stagemerge_stub")

KEY = {"model": "mlp", "dataset": "synthetic", "hp_set": ["lr", "momentum"]}
STUDIES = Path(__file__).resolve().parent.parent / "paper_2006_11972_b200" / "studies"


def engine(key=KEY, **opts):
    opts.setdefault("ckpts_per_gpu", 4096)
    return stub.Engine(json.dumps(key), json.dumps(opts))


def random_trials(rng):
    hps = tuple(KEY["hp_set"])
    pool = shared_space(rng, hps, n_choices=rng.randint(1, 3), total=rng.choice([100, 200, 300]))
    out = []
    for _ in range(rng.randint(1, 24)):
        if rng.random() < 0.75:
            cfg = json.loads(json.dumps(rng.choice(pool)))
            if rng.random() < 0.3:
                t = rng.randint(1, cfg["total_steps"])
                for h, segs in cfg["hps"].items():
                    acc, new = 0, []
                    for s in segs:
                        if acc >= t:
                            break
                        new.append({**s, "duration": min(s["duration"], t - acc)})
                        acc += s["duration"]
                    cfg["hps"][h] = new
                cfg["total_steps"] = t
        else:
            cfg = rand_config(rng, hps)
        out.append(cfg)
    return out


def plan_shape(plan):
    """(unique stage-steps, leaves, critical path in steps) of a fresh plan."""
    nodes = {n["id"]: n for n in plan["nodes"]}
    kids = {i: [] for i in nodes}
    for n in nodes.values():
        if n["parent"] is not None:
            kids[n["parent"]].append(n["boundary"])
    unique = leaves = crit = 0
    for i, n in nodes.items():
        ends = [r["end"] for r in n["requests"]]
        hi = max(ends + kids[i])
        unique += hi - n["boundary"]
        leaves += hi > max(kids[i], default=-1)
        crit = max(crit, max(ends, default=0))
    return unique, leaves, crit


def submit_all(e, trials):
    for i, cfg in enumerate(trials):
        e.submit(json.dumps(cfg), i, 0, i)


def run(trials, **opts):
    e = engine(**opts)
    submit_all(e, trials)
    shape = plan_shape(json.loads(e.plan_json()))
    e.run()
    return e, shape, json.loads(e.stats())


@pytest.mark.parametrize("seed", range(200))
def test_makespan_acceptance8(seed):
    rng = random.Random(seed)
    trials = random_trials(rng)
    ev = [rng.choice([0, 0, 25, 40])]
    # workers >= leaves: every leaf starts as soon as its branch checkpoint exists
    probe = engine(slots_per_gpu=1)
    submit_all(probe, trials)
    unique, leaves, crit = plan_shape(json.loads(probe.plan_json()))
    e, _, st = run(trials, slots_per_gpu=max(1, leaves), eval_intervals=ev)
    assert st["locksteps"] == crit, (st, unique, leaves, crit)
    assert st["stage_steps"] == unique
    assert not e.has_pending()
    # one worker: the makespan is the unique stage-steps (no re-execution, no idle locksteps)
    e1, _, st1 = run(trials, slots_per_gpu=1, eval_intervals=ev)
    assert st1["locksteps"] == unique and st1["stage_steps"] == unique
    # and the metric histories do not depend on the worker count
    assert {t: e.history(*t) for t in e.trials()} == {t: e1.history(*t) for t in e1.trials()}


@pytest.mark.parametrize("seed", range(60))
def test_stage_equals_trial_stub(seed):
    rng = random.Random(1000 + seed)
    trials = random_trials(rng)
    w = rng.choice([1, 3, 8])
    es, _, sst = run(trials, slots_per_gpu=w)
    et, _, tst = run(trials, slots_per_gpu=w, trial_mode=True)
    hs = {t: dict((r[0], r[1:]) for r in es.history(*t)) for t in es.trials()}
    ht = {t: dict((r[0], r[1:]) for r in et.history(*t)) for t in et.trials()}
    assert hs.keys() == ht.keys()
    for t, h in ht.items():
        # STAGE additionally holds the evals of other requests sharing the path; on every step
        # TRIAL mode evaluated, the merged run recorded bitwise the same metrics
        assert h and {s: hs[t][s] for s in h} == h, t
    # TRIAL mode trains every trial's own steps; STAGE the merged plan's unique steps
    assert tst["stage_steps"] == sum(c["total_steps"] for c in trials)
    assert sst["trial_steps"] == tst["trial_steps"] == sum(c["total_steps"] for c in trials)


def test_c2_grid_makespan_is_critical_path():
    # BASELINE configs[1]: 64 trials x 1,200 steps; 41,000 unique stage-steps; with 64 workers
    # the study takes exactly its 1,200-step critical path (acceptance 8)
    spec = (STUDIES / "c2_grid.json").read_text()
    info = json.loads(stub.expand_study(spec))
    e = stub.Engine(json.dumps(info["key"]), json.dumps({"slots_per_gpu": 64, "ckpts_per_gpu": 1024,
                                                          "eval_intervals": [info["eval_interval"]]}))
    e.submit_study(spec, 0)
    e.run()
    st = json.loads(e.stats())
    assert st["stage_steps"] == info["unique_steps"] == 41000
    assert st["trial_steps"] == info["total_steps"] == 76800
    assert st["locksteps"] == 1200, st
