"""Tuned studies through the engine on the GPU (exact mode):

* SHA decisions and step totals are identical in STAGE and TRIAL mode (SPEC.md tuners
  invariant: "total training steps across a SHA study are identical between STAGE and TRIAL
  modes"), while STAGE executes fewer unique stage-steps;
* the trials SHA promotes are the ones the CPU oracle ranks best at the rung (the metrics the
  tuner sees are the oracle's, bit for bit);
* ASHA and median stopping run to DONE; several tuned studies share one merged plan.
"""
import json

import numpy as np
import pytest

from oracle_lib import Slot
from paper_2006_11972_b200 import host
from test_engine_gpu import hp_table

pytestmark = pytest.mark.gpu


def sha_spec(tuner, n=12, seed=1):
    return json.dumps({
        "schema": 1, "name": "sha_mini", "max_steps": 80,
        "space": {"lr": [{"family": "step", "initial": "0.1", "gamma": "0.1", "milestones": [30]},
                         {"family": "constant", "value": "0.05"},
                         {"family": "exponential", "initial": "0.2", "gamma": "0.98"},
                         {"family": "constant", "value": "0.01"}],
                  "momentum": [{"family": "constant", "value": "0.9"},
                               {"family": "step", "values": ["0.5", "0.9"], "milestones": [10]},
                               {"family": "constant", "value": "0.0"}],
                  "batch_size": [{"family": "constant", "value": 32},
                                 {"family": "step", "values": [32, 64], "milestones": [25]}]},
        "sampler": {"kind": "random", "trials": n, "seed": seed},
        "tuner": tuner})


def run_tuned(specs, **opts):
    e = host.Engine.for_study(specs[0], max_batch=64, **opts)
    out = e.run_tuned(specs)
    return e, out


def test_sha_stage_equals_trial_and_oracle_ranking():
    spec = sha_spec({"kind": "sha", "reduction": 4, "min": 20, "max": 80})
    st, o1 = run_tuned([spec], slots_per_gpu=8)
    tr, o2 = run_tuned([spec], slots_per_gpu=8, trial_mode=True)
    assert o1 == o2                                            # same actions, winners, steps
    a = o1[0]
    assert a["actions"][-1].startswith("DONE") and len(a["winners"]) == 1
    assert st.stats()["trial_steps"] == tr.stats()["trial_steps"] == a["trial_steps"]
    assert st.stats()["stage_steps"] < tr.stats()["stage_steps"]
    # rung 0 ranking by the CPU oracle's val_loss at step 20
    info = host.expand_study(spec)
    losses = []
    for t, cfg in enumerate(info["trials"]):
        s = Slot(max_steps=81)
        s.train(hp_table(cfg), 20)
        losses.append((s.eval()[0], t))
    promoted = sorted(int(x.split()[1]) for x in a["actions"] if x.startswith("EXTEND"))
    assert promoted == sorted(t for _, t in sorted(losses)[:3])   # ceil(12 / 4) survivors


def test_asha_and_median_run_to_done_on_one_plan():
    s1 = sha_spec({"kind": "asha", "reduction": 2, "min": 20, "max": 80, "parallelism": 4}, seed=2)
    s2 = sha_spec({"kind": "median", "interval": 20, "parallelism": 6}, seed=3)
    e, out = run_tuned([s1, s2], slots_per_gpu=6)
    assert [o["study"] for o in out] == [0, 1]
    for o in out:
        assert o["actions"][-1].startswith("DONE")
        assert sum(a.startswith("SUBMIT") for a in o["actions"]) == 12
    assert e.stats()["trial_steps"] == sum(o["trial_steps"] for o in out)
    # deterministic: a second engine makes the same decisions
    _, again = run_tuned([s1, s2], slots_per_gpu=6)
    assert again == out
