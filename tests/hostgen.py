"""Random generators for hp functions, trial configs and plan action scripts (test helpers)."""
from __future__ import annotations

import random

DEC = ["0.1", "0.01", "0.05", "0.001", "1/3", "0.2", "0.5", "0.9", "0.95"]


def rand_fn(rng: random.Random, depth: int = 0, allow_warmup: bool = True) -> dict:
    fams = ["constant", "constant", "step", "step", "exponential", "linear", "cosine_restarts", "cyclic"]
    if allow_warmup and depth == 0:
        fams.append("warmup")
    fam = rng.choice(fams)
    if fam == "constant":
        return {"family": "constant", "value": rng.choice(DEC[:4])}
    if fam == "step":
        ms = sorted(rng.sample(range(1, 200), rng.randint(1, 3)))
        if rng.random() < 0.5:
            return {"family": "step", "initial": rng.choice(DEC[:3]), "gamma": rng.choice(["0.1", "0.5"]), "milestones": ms}
        return {"family": "step", "values": [rng.choice(DEC[:4]) for _ in range(len(ms) + 1)], "milestones": ms}
    if fam == "exponential":
        return {"family": "exponential", "initial": rng.choice(DEC[:2]), "gamma": rng.choice(["0.95", "0.99"])}
    if fam == "linear":
        f = {"family": "linear", "initial": "0.1", "total": rng.choice([50, 100, 150])}
        if rng.random() < 0.5:
            f["final"] = "0.01"
        return f
    if fam == "cosine_restarts":
        f = {"family": "cosine_restarts", "initial": "0.1", "t0": rng.choice([20, 50])}
        if rng.random() < 0.5:
            f["t_mult"] = 2
        if rng.random() < 0.3:
            f["eta_min"] = "0.001"
        return f
    if fam == "cyclic":
        f = {"family": "cyclic", "base": "0.01", "max": "0.1", "step_size_up": rng.choice([10, 25])}
        if rng.random() < 0.5:
            f["step_size_down"] = 15
        return f
    f = {"family": "warmup", "duration": rng.choice([5, 10]), "target": "0.1"}
    if rng.random() < 0.8:
        f["inner"] = rand_fn(rng, depth + 1)
    return f


def rand_seq(rng: random.Random, total: int) -> list:
    n = rng.randint(1, 3) if total >= 3 else 1
    cuts = sorted(rng.sample(range(1, total), n - 1)) if n > 1 else []
    bounds = [0] + cuts + [total]
    segs = []
    for a, b in zip(bounds, bounds[1:]):
        fn = rand_fn(rng)
        local = rng.choice([0, 0, 0, 5, 20]) if fn["family"] != "warmup" or "inner" in fn else 0
        if fn["family"] == "warmup" and "inner" not in fn:
            fn["duration"] = max(fn["duration"], b - a + local)
        segs.append({"fn": fn, "local_start": local, "duration": b - a})
    return segs


def rand_config(rng: random.Random, hps=("lr",), max_total: int = 300) -> dict:
    total = rng.choice([100, 200, 200, 300, rng.randint(1, max_total)])
    return {"total_steps": total, "hps": {h: rand_seq(rng, total) for h in hps}}


def shared_space(rng: random.Random, hps=("lr", "momentum"), n_choices: int = 3, total: int = 200) -> list:
    """A small space of per-hp sequences so random trials merge often."""
    space = {h: [rand_seq(rng, total) for _ in range(n_choices)] for h in hps}
    return [{"total_steps": total, "hps": {h: rng.choice(space[h]) for h in hps}} for _ in range(8)]


def rand_script(rng: random.Random, n_trials: int = 12, hps=("lr", "momentum")) -> dict:
    key = {"model": "mlp", "dataset": "synthetic", "hp_set": sorted(hps)}
    pool = shared_space(rng, hps, n_choices=rng.randint(1, 3), total=rng.choice([100, 200]))
    actions = []
    rid = 0
    for _ in range(n_trials):
        if rng.random() < 0.8:
            cfg = rng.choice(pool)
            if rng.random() < 0.3:  # a truncated variant (shorter request on the same path)
                t = rng.randint(1, cfg["total_steps"])
                cfg = truncate(cfg, t)
        else:
            cfg = rand_config(rng, hps)
        actions.append({"kind": "insert", "id": rid, "study": rng.randint(0, 2), "trial": rid, "config": cfg})
        rid += 1
        if rng.random() < 0.15:  # re-submission of a known id
            actions.append({"kind": "insert", "id": rng.randint(0, rid - 1), "study": 0, "trial": 0, "config": cfg})
        for _ in range(rng.randint(0, 3)):
            node, step = rng.randint(0, 2 * n_trials), rng.randint(0, 320)
            kind = rng.choice(["ckpt", "ckpt", "metrics", "value_at", "digest_at", "cancel"])
            if kind == "ckpt":
                actions.append({"kind": "ckpt", "node": node, "step": step, "handle": rng.choice(["a", "b"])})
            elif kind == "metrics":
                actions.append({"kind": "metrics", "node": node, "step": step,
                                "record": {"acc": rng.choice([0.5, 0.25])}})
            elif kind == "value_at":
                actions.append({"kind": "value_at", "node": node, "hp": rng.choice(list(hps) + ["bs"]), "step": step})
            elif kind == "digest_at":
                actions.append({"kind": "digest_at", "node": node, "step": step})
            else:
                actions.append({"kind": "cancel", "study": rng.randint(0, 2), "trial": rng.randint(0, rid)})
    return {"op": "plan", "key": key, "actions": actions, "kwise": [0, 1], "roundtrip": True}


def truncate(cfg: dict, t: int) -> dict:
    out = {"total_steps": t, "hps": {}}
    for h, segs in cfg["hps"].items():
        acc, new = 0, []
        for s in segs:
            if acc >= t:
                break
            new.append({**s, "duration": min(s["duration"], t - acc)})
            acc += s["duration"]
        out["hps"][h] = new
    return out
