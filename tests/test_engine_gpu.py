"""End-to-end parity of the study engine on the GPU (exact mode):

* the plan the engine builds is the reference's plan (signature pinned in
  test_host_vs_reference; here: node count / checkpoints / completions);
* STAGE (merged) and TRIAL (unmerged) metric histories are byte-equal (SPEC.md:421,
  acceptance 5) and unique-step counts give the merge-rate savings (acceptance 4);
* every trial's metrics equal the CPU oracle trained on that trial's own hp sequence;
* spilling the checkpoint pool to host memory changes nothing.
"""
import json

import numpy as np
import pytest

from oracle_lib import Slot
from paper_2006_11972_b200 import host

pytestmark = pytest.mark.gpu

HP_COLS = ("lr", "momentum", "weight_decay", "batch_size")
DEFAULTS = {"lr": 0.1, "momentum": 0.9, "weight_decay": 0.0, "batch_size": 128}


def hp_table(cfg: dict) -> np.ndarray:
    """Per-step hp rows of one trial config, computed by the host library (value_at)."""
    r = host.call({"op": "sequence", "config": cfg})
    T = cfg["total_steps"]
    rows = np.zeros((T, 4), np.float32)
    for c, name in enumerate(HP_COLS):
        rows[:, c] = r["hps"][name]["values"] if name in r["hps"] else DEFAULTS[name]
    return rows


def oracle_history(cfg: dict, marks):
    s = Slot(max_steps=cfg["total_steps"] + 1)
    hp = hp_table(cfg)
    out, done = {}, 0
    for m in sorted(marks):
        s.train(hp, m - done)
        done = m
        out[m] = s.eval()
    return out


def run(spec, **opts):
    e = host.Engine.for_study(spec, **opts)
    e.submit_study(spec)
    e.run()
    return e


def test_fig1_stage_vs_trial_and_oracle():
    spec = host.study_spec("c1_fig1")
    st = run(spec, slots_per_gpu=4)
    tr = run(spec, slots_per_gpu=4, trial_mode=True)
    s1, s2 = st.stats(), tr.stats()
    assert s1["stage_steps"] == 600 and s2["stage_steps"] == 800       # p = 4/3 (acceptance 4)
    assert s1["trial_steps"] == s2["trial_steps"] == 800
    assert st.plan_json()["nodes"].__len__() == 5
    assert not json.loads(st._e.plan_json())["nodes"][0]["requests"]
    h1, h2 = st.histories(), tr.histories()
    assert h1 == h2 and len(h1) == 4                                     # byte-equal metrics
    info = host.expand_study(spec)
    for (study, trial), hist in h1.items():
        cfg = info["trials"][trial]
        want = oracle_history(cfg, [200])
        assert [(s, l, a) for s, l, a in hist] == [(200, *want[200])]
    # checkpoints were saved at stage ends: the branch point n0@100 is shared
    nodes = st.plan_json()["nodes"]
    assert "100" in nodes[0]["ckpt"]


def test_random_study_with_eval_marks_bs_changes_and_spill():
    spec = json.dumps({
        "schema": 1, "name": "mini", "max_steps": 120, "eval_interval": 40,
        "space": {"lr": [{"family": "step", "initial": "0.1", "gamma": "0.1", "milestones": [60]},
                         {"family": "exponential", "initial": "0.1", "gamma": "0.99"},
                         {"family": "warmup", "duration": 10, "target": "0.1",
                          "inner": {"family": "constant", "value": "0.05"}}],
                  "batch_size": [{"family": "constant", "value": 64},
                                 {"family": "step", "values": [64, 200], "milestones": [50]}],
                  "momentum": [{"family": "constant", "value": "0.9"},
                               {"family": "step", "values": ["0.5", "0.9"], "milestones": [80]}]},
        "sampler": {"kind": "random", "trials": 16, "seed": 3}})
    st = run(spec, slots_per_gpu=8)
    tr = run(spec, slots_per_gpu=8, trial_mode=True)
    sp = run(spec, slots_per_gpu=3, ckpts_per_gpu=4)  # forces LRU spills to host memory
    assert sp.stats()["spills"] > 0
    h = st.histories()
    assert h == tr.histories() == sp.histories()
    assert all([s for s, _, _ in v] == [40, 80, 120] for v in h.values())
    assert st.stats()["stage_steps"] < tr.stats()["stage_steps"]
    info = host.expand_study(spec)
    for trial in (0, 5):
        want = oracle_history(info["trials"][trial], [40, 80, 120])
        assert [(s, l, a) for s, l, a in h[(0, trial)]] == [(m, *want[m]) for m in (40, 80, 120)]


def test_engine_reset_and_determinism():
    spec = host.study_spec("c1_fig1")
    e = host.Engine.for_study(spec, slots_per_gpu=2)
    e.submit_study(spec)
    e.run()
    first = (e.plan_json(), e.histories())
    e.reset()
    e.submit_study(spec)
    e.run()
    assert (e.plan_json(), e.histories()) == first  # byte-identical plan files (acceptance 10)


def test_partitioned_ranks_cover_all_roots():
    spec = host.study_spec("c1_fig1")
    owned, hist = [], {}
    for rank in range(2):
        e = host.Engine.for_study(spec, slots_per_gpu=4, rank=rank, world=2)
        e.submit_study(spec)
        e.run()
        owned.append(set(e.owned_roots()))
        for t, v in e.histories().items():
            if v:
                hist[t] = v
    assert owned[0].isdisjoint(owned[1]) and owned[0] | owned[1] == {0, 3}
    ref = run(spec, slots_per_gpu=4).histories()
    assert hist == ref


def dominant_root_spec(n=16, total=120):
    """16 trials on one root (lr 0.1 for 40 steps) branching at 40 and 80: one subtree holds all
    the work, so the multi-GPU placement splits it and the split-off subtrees LOAD by peer copy."""
    trials = []
    for i in range(n):
        trials.append({"hps": {"lr": {"family": "step", "values": ["0.1", ["0.05", "0.02", "0.01", "0.005"][i % 4],
                                                                  ["0.003", "0.002", "0.001", "0.0005"][i // 4]],
                                      "milestones": [40, 80]}}})
    return json.dumps({"schema": 1, "name": "dominant", "model": "mlp", "max_steps": total, "eval_interval": 40,
                       "trials": trials})


@pytest.mark.parametrize("spec_name", ["c1_fig1", "dominant"])
def test_two_contexts_equal_one_device(spec_name):
    """Engine(devices=[0, 0]): two executor contexts on the one B200, paths placed by subtree
    (place_nodes / schedule_placed); split-off subtrees LOAD through smx_ckpt_peer_copy (K7).
    Every trial's history is bitwise the single-context run's and no step is re-executed."""
    spec = host.study_spec("c1_fig1") if spec_name == "c1_fig1" else dominant_root_spec()
    one = run(spec, slots_per_gpu=4)
    two = run(spec, slots_per_gpu=4, devices=[0, 0])
    assert two.histories() == one.histories()
    s1, s2 = one.stats(), two.stats()
    assert s1["stage_steps"] == s2["stage_steps"] and s1["trial_steps"] == s2["trial_steps"]
    if spec_name == "dominant":
        assert s2["peer_copies"] > 0
    # tensor-core mode too (grouping invariance across contexts)
    one_tc = run(spec, slots_per_gpu=4, gemm_mode=1)
    two_tc = run(spec, slots_per_gpu=4, gemm_mode=1, devices=[0, 0])
    assert two_tc.histories() == one_tc.histories()
