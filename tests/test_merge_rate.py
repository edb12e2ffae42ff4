"""SPEC acceptance 3: for 500 randomised search spaces (<= 50 trials, <= 2,000
steps, mixed function families) the plan-based merge rate against brute-force per-step
value-prefix deduplication (a trie over per-step value tuples, values from the compiled
reference's hpseq, oracle/_ref -- no canonical forms involved).

Finding (checked here): the reference's plan merges by canonical atoms (hpseq.cpp: constant runs
merge across families, any other family only with an identical descriptor), so a pointwise
coincidence between *different* non-constant functions -- e.g. exponential(0.01, 0.99) and
constant 0.01 agree at step 0 only -- is not merged by the reference.  The SPEC's "exact
equality" therefore holds for spaces whose families are piecewise constant (constant / step),
and for mixed spaces the reference plan is sound (never merges unequal prefixes: unique_plan >=
unique_bruteforce).  The product plan must equal the reference plan exactly in both cases (the
north_star's bit-exact plan requirement)."""
import random
from fractions import Fraction

import pytest

import oracle_lib as ol
from hostgen import rand_fn
from paper_2006_11972_b200 import host

pytestmark = pytest.mark.skipif(not ol.REF_SO.exists(), reason="oracle/_ref not built")

HPS = ("lr", "momentum")


def rand_space(rng, piecewise_constant=False):
    """A space whose trials share prefixes often: per-hp pools of 1-3 segment sequences over a
    common horizon, trials truncated at random ends."""
    total = rng.randint(1, 2000)
    pools = {}
    for h in HPS:
        pools[h] = []
        for _ in range(rng.randint(1, 3)):
            n = rng.randint(1, 3) if total >= 3 else 1
            cuts = sorted(rng.sample(range(1, total), n - 1)) if n > 1 else []
            bounds = [0] + cuts + [total]
            segs = []
            for a, b in zip(bounds, bounds[1:]):
                fn = rand_fn(rng, allow_warmup=False)
                while piecewise_constant and fn["family"] not in ("constant", "step"):
                    fn = rand_fn(rng, allow_warmup=False)
                segs.append({"fn": fn, "local_start": rng.choice([0, 0, 3]), "duration": b - a})
            pools[h].append(segs)
    trials = []
    for _ in range(rng.randint(1, 50)):
        t = total if rng.random() < 0.6 else rng.randint(1, total)
        cfg = {"total_steps": t, "hps": {}}
        for h in HPS:
            acc, new = 0, []
            for s in rng.choice(pools[h]):
                if acc >= t:
                    break
                new.append({**s, "duration": min(s["duration"], t - acc)})
                acc += s["duration"]
            cfg["hps"][h] = new
        trials.append(cfg)
    return trials


@pytest.mark.parametrize("seed", range(500))
def test_merge_rate_vs_bruteforce_prefix_dedup(seed):
    rng = random.Random(seed)
    pwc = seed % 2 == 0  # even seeds: piecewise-constant families only (exact equality)
    trials = rand_space(rng, piecewise_constant=pwc)
    key = {"model": "mlp", "dataset": "synthetic", "hp_set": list(HPS)}
    acts = [{"kind": "insert", "id": i, "study": 0, "trial": i, "config": c} for i, c in enumerate(trials)]
    r = host.call({"op": "plan", "key": key, "actions": acts})
    if any("error" in x for x in r["results"]):  # an invalid random function: both sides reject it
        ref = ol.ref_call({"op": "plan", "key": key, "actions": acts})
        assert [("error" in x) for x in r["results"]] == [("error" in x) for x in ref["results"]]
        pytest.skip("invalid random space")
    import json

    def unique_of(plan_json):
        plan = json.loads(plan_json)
        kids = {n["id"]: [] for n in plan["nodes"]}
        for n in plan["nodes"]:
            if n["parent"] is not None:
                kids[n["parent"]].append(n["boundary"])
        return sum(max([q["end"] for q in n["requests"]] + kids[n["id"]] + [n["boundary"]]) - n["boundary"]
                   for n in plan["nodes"])

    unique_plan = unique_of(r["json"])
    assert unique_plan == unique_of(ol.ref_call({"op": "plan", "key": key, "actions": acts})["json"])
    total = sum(c["total_steps"] for c in trials)
    # brute force: a trie over per-step value tuples (values from the compiled reference)
    root, unique_bf = {}, 0
    for c in trials:
        vals = {h: ol.ref_call({"op": "sequence", "config": {"total_steps": c["total_steps"],
                                                            "hps": {h: c["hps"][h]}}})["hps"][h]["values"]
                for h in HPS}
        node = root
        for s in range(c["total_steps"]):
            step_key = tuple(vals[h][s] for h in HPS)
            if step_key not in node:
                node[step_key] = {}
                unique_bf += 1
            node = node[step_key]
    if pwc:
        assert Fraction(total, unique_plan) == Fraction(total, unique_bf), (unique_plan, unique_bf)
    else:
        assert unique_plan >= unique_bf  # sound: never merges unequal value prefixes
