"""Differential tests: the product host library (paper_2006_11972_b200/_stagemerge) against the
*compiled reference* (oracle/_ref/libstagemerge_ref.so = reference hpseq.cpp + plan.cpp).

Both expose the same JSON command interface; every answer — values, canonical forms, digests,
plan signatures, to_json bytes, DOT, pending lists, error kinds and messages — must be equal.
Also pins the SPEC known answers and the Fig. 1 plan
(SURVEY Appendix A)."""
import json
import random

import pytest

from hostgen import rand_config, rand_fn, rand_script
from oracle_lib import REF_SO, ref_call
from paper_2006_11972_b200 import host

pytestmark = pytest.mark.skipif(not REF_SO.exists(), reason="reference oracle not built (needs /root/reference)")


def both(cmd):
    a = ref_call(cmd)
    b = host.call(cmd)
    assert b == a, json.dumps(cmd)[:2000]
    return b


def test_spec_value_at_known_answers():
    r = both({"op": "value_at", "fn": {"family": "exponential", "initial": "0.1", "gamma": "0.95"}, "steps": [0, 2]})
    assert r["values"] == [0.1, 0.09025]
    r = both({"op": "value_at", "fn": {"family": "step", "values": [128, 256], "milestones": [70]}, "steps": [69, 70]})
    assert r["values"] == [128, 256]
    r = both({"op": "value_at", "fn": {"family": "constant", "value": "0.1"}, "steps": [57]})
    assert r["values"] == [0.1]
    r = both({"op": "value_at", "fn": {"family": "cosine_restarts", "initial": "0.1", "t0": 200, "t_mult": 2},
              "steps": [1, 100, 200]})
    assert r["values"][1] == pytest.approx(0.05) and r["values"][2] == 0.1


def test_spec_canonicalize_and_split_known_answers():
    cfg = {"total_steps": 180, "hps": {"lr": [{"fn": {"family": "step", "initial": "0.1", "gamma": "0.1",
                                                      "milestones": [90, 135]}, "duration": 180}]}}
    r = both({"op": "sequence", "config": cfg, "digest_steps": [0, 90, 180]})
    assert r["hps"]["lr"]["canon"] == [["constant(value=0.1)@0", 0, 90], ["constant(value=0.01)@0", 90, 45],
                                       ["constant(value=0.001)@0", 135, 45]]
    exp = {"total_steps": 60, "hps": {"lr": [{"fn": {"family": "exponential", "initial": "0.1", "gamma": "0.95"},
                                              "duration": 60}]}}
    r = both({"op": "sequence", "config": exp, "split": 20})
    assert r["hps"]["lr"]["split_left"] + r["hps"]["lr"]["split_right"] == r["hps"]["lr"]["values"]
    warm = {"total_steps": 20, "hps": {"lr": [{"fn": {"family": "warmup", "duration": 5, "target": "0.1",
                                                      "inner": {"family": "exponential", "initial": "0.1", "gamma": "0.95"}},
                                               "duration": 20}]}}
    r = both({"op": "sequence", "config": warm})
    assert [c[0] for c in r["hps"]["lr"]["canon"]] == ["warmup(duration=5,target=0.1)@0",
                                                      "exponential(gamma=0.95,initial=0.1)@0"]
    assert r["hps"]["lr"]["values"][:8] == pytest.approx([0.02, 0.04, 0.06, 0.08, 0.1, 0.1, 0.095, 0.09025])


def test_cross_family_merge_via_exact_rationals():
    a = {"total_steps": 200, "hps": {"lr": [{"fn": {"family": "step", "initial": "0.1", "gamma": "0.1",
                                                    "milestones": [100]}, "duration": 200}]}}
    b = {"total_steps": 200, "hps": {"lr": [{"fn": {"family": "constant", "value": "0.1"}, "duration": 100},
                                            {"fn": {"family": "constant", "value": "0.01"}, "duration": 100}]}}
    assert both({"op": "common_prefix", "a": a, "b": b})["n"] == 200


FIG1 = {"A": ("0.1", "0.01"), "B": ("0.1", "0.001"), "C": ("0.01", "0.001"), "D": ("0.01", "0.01")}


def fig1_cfg(first, second):
    return {"total_steps": 200, "hps": {"lr": [{"fn": {"family": "constant", "value": first}, "duration": 100},
                                               {"fn": {"family": "constant", "value": second}, "duration": 100}]}}


def test_fig1_plan_signature_and_digest():
    actions = [{"kind": "insert", "id": i, "study": 0, "trial": i, "config": fig1_cfg(*FIG1[k])}
               for i, k in enumerate("ABCD")]
    actions.append({"kind": "digest_at", "node": 0, "step": 100})
    r = both({"op": "plan", "key": {"model": "mlp", "dataset": "synthetic", "hp_set": ["lr"]}, "actions": actions})
    assert r["node_count"] == 5
    assert r["results"][-1]["digest"] == "8b1723e0a18b2b46"
    assert r["signature"] == (
        "mlp|synthetic|lr{@0 lr=constant(value=0.01)@0 ck:[] mx:[] rq:[200(0:3 ),] {@100 lr=constant(value=0.001)@0 "
        "ck:[] mx:[] rq:[200(0:2 ),] }}{@0 lr=constant(value=0.1)@0 ck:[] mx:[] rq:[] {@100 "
        "lr=constant(value=0.001)@0 ck:[] mx:[] rq:[200(0:1 ),] }{@100 lr=constant(value=0.01)@0 ck:[] mx:[] "
        "rq:[200(0:0 ),] }}")
    assert r["file_name"] == "mlp_synthetic_lr-08a83c7c2cf32643.json"


def test_rationals():
    texts = ["0.1", "-0.5", "1/3", "5e-5", "0.095", "-3", "+2.50", "1e3", "6/4", "0.0001", "-1/8", "abc", "", "1.2.3",
             "1/0", "1e+3", "123456789012345678901234567890"]
    for t in texts:
        both({"op": "rational", "texts": [t]})


@pytest.mark.parametrize("seed", range(40))
def test_random_functions_values(seed):
    rng = random.Random(seed)
    for _ in range(10):
        both({"op": "value_at", "fn": rand_fn(rng), "steps": [0, 1, 7, 50, 99, 100, 151, 299]})


@pytest.mark.parametrize("seed", range(60))
def test_random_sequences(seed):
    rng = random.Random(1000 + seed)
    cfg = rand_config(rng, ("lr", "momentum"))
    cmd = {"op": "sequence", "config": cfg, "digest_steps": sorted({0, 1, cfg["total_steps"] // 2, cfg["total_steps"]})}
    if cfg["total_steps"] > 1:
        cmd["split"] = rng.randint(1, cfg["total_steps"] - 1)
    both(cmd)
    other = rand_config(rng, ("lr", "momentum"))
    both({"op": "common_prefix", "a": cfg, "b": other})
    both({"op": "common_prefix", "a": cfg, "b": cfg})


@pytest.mark.parametrize("seed", range(150))
def test_random_plan_scripts(seed):
    rng = random.Random(seed)
    r = both(rand_script(rng, n_trials=rng.randint(1, 16)))
    assert r.get("roundtrip_signature", r["signature"]) == r["signature"]


def test_insertion_order_invariance_of_signature():
    rng = random.Random(7)
    script = rand_script(rng, n_trials=14)
    inserts = [a for a in script["actions"] if a["kind"] == "insert"]
    s1 = host.call({**script, "actions": inserts})
    shuffled = inserts[:]
    rng.shuffle(shuffled)
    s2 = host.call({**script, "actions": shuffled})
    # ids differ but structure must not (subscriber sets of re-submissions may differ; drop them)
    if not any(i["id"] < j for j, i in enumerate(inserts) if i["id"] != j):
        assert s1["signature"] == s2["signature"]
