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


def lr_trial(lr, steps):
    return {"total_steps": steps, "hps": {"lr": [{"fn": {"family": "constant", "value": lr}, "local_start": 0,
                                                  "duration": steps}]}}


KEY_LR = {"model": "mlp", "dataset": "synthetic", "hp_set": ["lr"]}


def test_stop_releases_in_flight_slot():
    """STOP of a trial whose only pending request is in flight frees that worker's slot
    (smx_release_slot); the shared prefix it served for another trial was already trained."""
    e = engine(KEY_LR, slots_per_gpu=4)
    for i, (lr, T) in enumerate([("0.1", 20), ("0.1", 300), ("0.01", 300)]):
        e.submit(json.dumps(lr_trial(lr, T)), i, 0, i)
    stops = []

    def on_done(node, end, subs):
        if (0, 0) in [tuple(s) for s in subs]:
            stops.append(e.cancel(0, 1))

    e.on_complete(on_done)
    e.run()
    st = json.loads(e.stats())
    assert stops == [True] and st["releases"] == 1
    assert st["stage_steps"] == 20 + 300 and st["locksteps"] == 300
    assert not e.has_pending()
    assert [s for s, _, _ in e.history(0, 1)] == [20] and len(e.history(0, 2)) == 1  # never reached 300
    idle = [ev for ev in e.trace() if ev[2] == "IDLE" and ev[6] == "released"]
    assert len(idle) == 1 and idle[0][0] == 20


def test_stop_keeps_shared_stages_running():
    """STOP of one of two trials sharing an in-flight path: the other still needs it -> no release."""
    e = engine(KEY_LR, slots_per_gpu=4)
    for i, (lr, T) in enumerate([("0.1", 20), ("0.1", 300), ("0.1", 200)]):
        e.submit(json.dumps(lr_trial(lr, T)), i, 0, i)
    e.on_complete(lambda node, end, subs: e.cancel(0, 1) if [0, 0] in [list(s) for s in subs] else None)
    e.run()
    st = json.loads(e.stats())
    assert st["releases"] == 0 and st["stage_steps"] == 200 and [s for s, _, _ in e.history(0, 2)] == [20, 200]


@pytest.mark.parametrize("seed", range(20))
def test_checkpoint_gc_frees_instead_of_spilling(seed):
    rng = random.Random(500 + seed)
    trials = random_trials(rng)
    runs = {}
    for gc in (False, True):
        e, _, st = run(trials, slots_per_gpu=2, ckpts_per_gpu=3, ckpt_gc=gc)
        runs[gc] = (st, {t: e.history(*t) for t in e.trials()})
    (s0, h0), (s1, h1) = runs[False], runs[True]
    assert h0 == h1                       # GC never changes results
    assert s1["spills"] <= s0["spills"]   # dead entries are freed, not spilled
    assert s0["gc_frees"] == 0
    if s0["spills"]:
        assert s1["gc_frees"] > 0 or s1["spills"] == s0["spills"]


def test_collect_checkpoints_keeps_what_live_trials_need():
    e = engine(KEY_LR, slots_per_gpu=2, ckpts_per_gpu=64, eval_intervals=[40])
    for i, (lr, T) in enumerate([("0.1", 100), ("0.1", 200), ("0.01", 150)]):
        e.submit(json.dumps(lr_trial(lr, T)), i, 0, i)
    e.run()
    saves = json.loads(e.stats())["saves"]
    freed = e.collect_checkpoints()
    # the eval-mark checkpoints (40, 80, 120, 160) go; each live trial's end checkpoint stays
    assert saves == 10 and freed == 7
    # an EXTEND of trial 1 resumes from its kept end checkpoint: no retraining of [0, 200)
    e.submit(json.dumps(lr_trial("0.1", 260)), 10, 0, 1)
    before = json.loads(e.stats())["stage_steps"]
    e.run()
    assert json.loads(e.stats())["stage_steps"] - before == 60


def test_set_runtime_fed_from_profile_table():
    key = {"model": "mlp", "dataset": "synthetic", "hp_set": ["batch_size", "lr"]}
    cfg = lambda lr, bs: {"total_steps": 100, "hps": {
        "lr": [{"fn": {"family": "constant", "value": lr}, "local_start": 0, "duration": 100}],
        "batch_size": [{"fn": {"family": "constant", "value": bs}, "local_start": 0, "duration": 100}]}}
    e = engine(key, slots_per_gpu=2, step_cost_us={"128": 51.5, "256": 97.25})
    e.submit(json.dumps(cfg("0.1", 128)), 0, 0, 0)
    e.submit(json.dumps(cfg("0.1", 256)), 1, 0, 1)
    e.run()
    plan = json.loads(e.plan_json())
    rt = sorted(n["runtime_sec_per_step"] for n in plan["nodes"])
    assert rt == pytest.approx([51.5e-6, 97.25e-6], rel=1e-12)


def test_trace_determinism_and_accounting():
    rng = random.Random(77)
    trials = random_trials(rng)
    tr = []
    for _ in range(2):
        e, shape, st = run(trials, slots_per_gpu=3, eval_intervals=[40])
        tr.append(e.trace())
    assert tr[0] == tr[1]  # acceptance 10: byte-identical traces
    ev = tr[0]
    kinds = {k for _, _, k, *_ in ev}
    assert kinds <= {"LOAD", "TRAIN", "SAVE", "EVAL", "IDLE"}
    # TRAIN durations sum to the executed stage-steps; per worker they never overlap
    assert sum(end - start for _, _, k, _, start, end, _ in ev if k == "TRAIN") == st["stage_steps"]
    per = {}
    for t, w, k, _, start, end, _ in ev:
        if k == "TRAIN":
            per.setdefault(w, []).append((t, t + end - start))
    for spans in per.values():
        spans.sort()
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
    # every trial is reported exactly once, at its end step, by an EVAL event
    seen = {}
    for _, _, k, _, start, end, d in ev:
        if k == "EVAL" and "trials=" in d:
            for s in d.split("trials=")[1].split(","):
                seen.setdefault(s, []).append(end)
    assert sorted(seen) == sorted(f"0:{i}" for i in range(len(trials)))
    assert all(seen[f"0:{i}"] == [c["total_steps"]] for i, c in enumerate(trials))


# ---------------------------------------------------------------- in-process multi-GPU (§8e)

def dominant_root_trials(n=16, total=300, momentum=True):
    """One root (lr 0.1 for the first 100 steps) carries every trial; they branch at 100 / 200."""
    out = []
    for i in range(n):
        segs = [{"fn": {"family": "constant", "value": "0.1"}, "local_start": 0, "duration": 100},
                {"fn": {"family": "constant", "value": ["0.05", "0.02", "0.01", "0.005"][i % 4]}, "local_start": 0,
                 "duration": 100},
                {"fn": {"family": "constant", "value": ["0.003", "0.002", "0.001", "0.0005"][i // 4]},
                 "local_start": 0, "duration": total - 200}]
        hps = {"lr": segs}
        if momentum:
            hps["momentum"] = [{"fn": {"family": "constant", "value": "0.9"}, "local_start": 0, "duration": total}]
        out.append({"total_steps": total, "hps": hps})
    return out


def test_placement_splits_a_dominant_root():
    from paper_2006_11972_b200 import host
    trials = dominant_root_trials(momentum=False)
    acts = [{"kind": "insert", "id": i, "study": 0, "trial": i, "config": c} for i, c in enumerate(trials)]
    for G in (1, 2, 4, 8):
        r = host.call({"op": "plan", "key": KEY_LR, "actions": acts, "placement": G})
        place = {int(k): v for k, v in r["placement"].items()}
        plan = json.loads(r["json"])
        assert set(place) == {n["id"] for n in plan["nodes"]} and set(place.values()) <= set(range(G))
        if G == 1:
            assert set(place.values()) == {0}
        else:  # the single root's subtree is split at its branch points over every device
            assert len(set(place.values())) == G
        # deterministic: same plan -> same placement
        assert host.call({"op": "plan", "key": KEY_LR, "actions": acts, "placement": G})["placement"] == r["placement"]


@pytest.mark.parametrize("seed", range(30))
def test_multi_device_engine_equals_single_device(seed):
    """Engine(devices=[0, 0]) (two contexts): paths placed by subtree, split-off subtrees LOAD
    through peer copies; every trial's metrics equal the single-device run's, no step re-run."""
    rng = random.Random(900 + seed)
    trials = dominant_root_trials() if seed % 3 == 0 else random_trials(rng)
    one, _, s1 = run(trials, slots_per_gpu=4)
    two, _, s2 = run(trials, slots_per_gpu=4, devices=[0, 0])
    four, _, s4 = run(trials, slots_per_gpu=2, devices=[0, 0, 0, 0])
    h1 = {t: one.history(*t) for t in one.trials()}
    assert {t: two.history(*t) for t in two.trials()} == h1
    assert {t: four.history(*t) for t in four.trials()} == h1
    assert s1["stage_steps"] == s2["stage_steps"] == s4["stage_steps"]
    if seed % 3 == 0:
        assert s2["peer_copies"] > 0 and s4["peer_copies"] > 0


def test_dominant_root_speeds_up_with_devices():
    """Four GPUs x 2 slots vs one GPU x 2 slots on the dominant-root study: the makespan (max over
    GPUs of their locksteps is bounded by the sum) drops; the work is spread over all devices."""
    trials = dominant_root_trials()
    e1, _, s1 = run(trials, slots_per_gpu=2)
    e4, _, s4 = run(trials, slots_per_gpu=2, devices=[0, 0, 0, 0])
    assert s4["peer_copies"] > 0
    assert s4["model_wall_us"] < s1["model_wall_us"]
