"""Stage trees (paper Alg. 1 / Fig. 7; SPEC acceptance 1, 2, 8) and the critical-path scheduler.

The reference declares this API without implementing it, so the checks are the SPEC's: the
Fig. 6 -> Fig. 7 reconstruction, equivalence of per-request training intervals with an
independent non-memoised backward-walk oracle on random plans, memo transparency, exact cover
/ no duplication invariants, and critical-path / scheduling examples."""
import random

import pytest

from hostgen import rand_script
from paper_2006_11972_b200 import host

KEY = {"model": "mlp", "dataset": "synthetic", "hp_set": ["lr"]}
EXP = {"family": "exponential", "initial": "0.1", "gamma": "0.95"}
LIN = {"family": "linear", "initial": "0.1", "total": 100}
C05 = {"family": "constant", "value": "0.05"}
C02 = {"family": "constant", "value": "0.02"}


def seq(*parts):
    segs, local = [], {}
    for fn, d in parts:
        key = str(fn)
        segs.append({"fn": fn, "local_start": local.get(key, 0), "duration": d})
        local[key] = local.get(key, 0) + d
    return {"total_steps": sum(d for _, d in parts), "hps": {"lr": segs}}


def fig6_actions():
    trials = [seq((EXP, 15)),                          # H1 request 15
              seq((EXP, 10), (LIN, 15)),               # H2 at 10, request 25
              seq((EXP, 20), (C05, 15)),               # H3 at 20, request 35
              seq((EXP, 20), (C05, 20), (C02, 10))]    # H4 at 40 under H3, request 50
    acts = [{"kind": "insert", "id": i, "study": 0, "trial": i, "config": c} for i, c in enumerate(trials)]
    acts += [{"kind": "ckpt", "node": 0, "step": 10, "handle": "h1@10"},
             {"kind": "ckpt", "node": 0, "step": 20, "handle": "h1@20"},
             {"kind": "ckpt", "node": 1, "step": 20, "handle": "h2@20"}]
    return acts


def run_tree(actions, **tree):
    r = host.call({"op": "plan", "key": KEY, "actions": actions, "tree": tree})
    assert "error" not in r, r
    return r


def test_fig6_to_fig7():
    r = run_tree(fig6_actions())
    nodes = {n["id"]: n for n in __import__("json").loads(r["json"])["nodes"]}
    assert [nodes[i]["boundary"] for i in range(4)] == [0, 10, 20, 40]
    st = {(s["node"], s["start"], s["end"]): s for s in r["tree"]["stages"]}
    assert set(st) == {(0, 10, 15), (1, 20, 25), (2, 20, 35), (2, 35, 40), (3, 40, 50)}
    assert st[(0, 10, 15)]["resume"] == [0, 10]
    assert st[(1, 20, 25)]["resume"] == [1, 20]      # "resuming from H2's checkpoint at 20"
    assert st[(2, 20, 35)]["resume"] == [0, 20]      # "[20,35) on H3 resuming from H1@20"
    assert st[(2, 35, 40)]["parent"] == st[(2, 20, 35)]["id"]
    assert st[(3, 40, 50)]["parent"] == st[(2, 35, 40)]["id"]
    assert st[(2, 20, 35)]["eval_at_end"] and not st[(2, 35, 40)]["eval_at_end"]
    assert r["tree"]["leaf_count"] == 3
    assert r["tree"]["intervals"]["3"] == [[2, 20, 40], [3, 40, 50]]


def test_empty_tree_and_eval_only_stage():
    acts = [{"kind": "insert", "id": 0, "study": 0, "trial": 0, "config": seq((EXP, 30))},
            {"kind": "ckpt", "node": 0, "step": 30, "handle": "x"}]
    r = run_tree(acts)
    assert [(s["start"], s["end"], s["resume"]) for s in r["tree"]["stages"]] == [(30, 30, [0, 30])]
    acts.append({"kind": "metrics", "node": 0, "step": 30, "record": {"acc": 1.0}})
    assert run_tree(acts)["tree"]["stages"] == []


def test_running_blocks_and_scratch():
    acts = [{"kind": "insert", "id": i, "study": 0, "trial": i, "config": c}
            for i, c in enumerate([seq((EXP, 100), (C05, 100)), seq((EXP, 100), (C02, 100))])]
    r = run_tree(acts)
    roots = [r["tree"]["stages"][i] for i in r["tree"]["roots"]]
    assert [(s["node"], s["start"], s["end"], s["resume"]) for s in roots] == [(0, 0, 100, None)]
    assert run_tree(acts, running=[0])["tree"]["stages"] == []
    acts.append({"kind": "ckpt", "node": 0, "step": 100, "handle": "b"})
    r = run_tree(acts, running=[1])
    assert [(s["node"], s["start"], s["end"]) for s in r["tree"]["stages"]] == [(2, 100, 200)]
    # acceptance 8: node 0 still running, but its checkpoint at the branch
    # step exists -- both children resolve to it instead of staying blocked
    r = run_tree(acts, running=[0])
    assert sorted((s["node"], s["start"], s["end"], tuple(s["resume"])) for s in r["tree"]["stages"]) == [
        (1, 100, 200, (0, 100)), (2, 100, 200, (0, 100))]
    # ... while a step the running worker has not saved yet stays blocked
    acts2 = acts[:2] + [{"kind": "ckpt", "node": 0, "step": 50, "handle": "c"}]
    assert run_tree(acts2, running=[0])["tree"]["stages"] == []


def test_eval_interval_splits():
    acts = [{"kind": "insert", "id": 0, "study": 0, "trial": 0, "config": seq((EXP, 100))}]
    r = run_tree(acts, eval_intervals=[30])
    assert [(s["start"], s["end"], s["eval_at_end"]) for s in r["tree"]["stages"]] == [
        (0, 30, True), (30, 60, True), (60, 90, True), (90, 100, True)]


def test_critical_path_and_schedule():
    # Fig. 1 plan: paths n0->n1 and n0->n2 (200 steps), n3->n4 (200) and n3 alone (request 200)
    cfg = lambda a, b: seq(({"family": "constant", "value": a}, 100), ({"family": "constant", "value": b}, 100))
    trials = [cfg("0.1", "0.01"), cfg("0.1", "0.001"), cfg("0.01", "0.001"), cfg("0.01", "0.01")]
    acts = [{"kind": "insert", "id": i, "study": 0, "trial": i, "config": c} for i, c in enumerate(trials)]
    r = run_tree(acts, workers=[3, 1, 2])
    st = r["tree"]["stages"]
    path = [(st[i]["node"], st[i]["start"], st[i]["end"]) for i in r["tree"]["critical_path"]]
    assert path == [(0, 0, 100), (1, 100, 200)]  # equal lengths: smaller node id wins
    assert r["tree"]["critical_us"] == 200
    got = [(a["worker"], [(st[i]["node"], st[i]["start"]) for i in a["stages"]]) for a in r["tree"]["assignments"]]
    # n3's path n3[0,100) -> n3[100,200) ... the tree splits n3 at 100 (n4's boundary)
    assert got[0] == (1, [(0, 0), (1, 100)])
    assert got[1][0] == 2 and got[1][1][0] == (3, 0)
    assert len(got) == 2  # children of scheduled roots wait for their checkpoint
    # per-node step cost changes the choice
    r = run_tree(acts, step_us={"3": 5})
    assert r["tree"]["stages"][r["tree"]["critical_path"][0]]["node"] == 3


# ---- acceptance 2: random plans vs an independent backward-walk oracle ----------------------

def oracle_intervals(plan, running):
    nodes = {n["id"]: n for n in plan["nodes"]}
    out = {}
    for n in nodes.values():
        for req in n["requests"]:
            pieces, cur, hi, blocked = [], n["id"], req["end"], False
            while True:
                nd = nodes[cur]
                if cur in running:
                    # acceptance 8: a running node unlocks a request only through a checkpoint
                    # it already holds at exactly the step asked for
                    if str(hi) in (nd["ckpt"] or {}) and hi > nd["boundary"]:
                        pieces.append((cur, hi, hi))
                    else:
                        blocked = True
                    break
                cks = [int(s) for s in (nd["ckpt"] or {}) if nd["boundary"] < int(s) <= hi]
                if cks:
                    pieces.append((cur, max(cks), hi))
                    break
                pieces.append((cur, nd["boundary"], hi))
                if nd["parent"] is None:
                    break
                hi, cur = nd["boundary"], nd["parent"]
            if blocked:
                continue
            pieces = pieces[::-1]
            keep = [p for p in pieces if p[1] < p[2]] or [pieces[-1]]
            out[str(req["id"])] = [list(p) for p in keep]
    return out


@pytest.mark.parametrize("seed", range(1000))  # 1,000 random plans
def test_random_plans_match_backward_walk_oracle(seed):
    import json
    rng = random.Random(seed)
    script = rand_script(rng, n_trials=rng.randint(1, 12), hps=("lr",))
    script["actions"] = [a for a in script["actions"] if a["kind"] in ("insert", "ckpt", "metrics", "cancel")]
    base = host.call({**script, "key": KEY})
    plan = json.loads(base["json"])
    n = base["node_count"]
    # extra random (valid and invalid) checkpoints
    for _ in range(rng.randint(0, 8)):
        script["actions"].append({"kind": "ckpt", "node": rng.randrange(n), "step": rng.randint(1, 300),
                                  "handle": "h"})
    running = sorted(rng.sample(range(n), rng.randint(0, min(3, n)))) if rng.random() < 0.5 else []
    r1 = host.call({**script, "key": KEY, "tree": {"running": running, "eval_intervals": [rng.choice([0, 25, 40])]}})
    r2 = host.call({**script, "key": KEY, "tree": {"running": running, "use_memo": False}})
    plan = json.loads(r1["json"])
    assert r1["tree"]["intervals"] == oracle_intervals(plan, set(running))
    assert r1["tree"]["intervals"] == r2["tree"]["intervals"]  # memoisation is transparent
    # invariants: no two stages of one node overlap; parents end where children start
    st = r1["tree"]["stages"]
    by_node = {}
    for s in st:
        for o in by_node.get(s["node"], []):
            assert s["end"] <= o["start"] or o["end"] <= s["start"] or (s["start"] == s["end"] == o["start"] == o["end"])
        by_node.setdefault(s["node"], []).append(s)
        if s["parent"] is not None:
            assert st[s["parent"]]["end"] == s["start"] and s["resume"] is None
        elif s["resume"] is None:
            assert s["start"] == 0
    # statelessness
    assert host.call({**script, "key": KEY, "tree": {"running": running, "eval_intervals": [0]}})["tree"]["intervals"] == \
        r1["tree"]["intervals"]
