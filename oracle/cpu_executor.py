"""TEST INFRASTRUCTURE / TIMED CPU BASELINE ONLY -- never imported by the product package.

The reference-side CPU executor: the stage executor's semantics run on the CPU oracle
(liboracle: the builder's fp32 restatement of the training arithmetic, DESIGN.md §3/§3b) over
the merged search plan the *reference itself* builds (oracle/_ref/libstagemerge_ref.so: the
reference's SearchPlan::insert_trial and SearchPlan::value_at, plan.cpp:53-151 / :278-288,
compiled from /root/reference by oracle/Makefile).  Nothing here touches paper_2006_11972_b200.

Semantics (the reference's worker_execute; Alg. 1 resume):
every plan node's step range [start, hi) is trained exactly once, from the parent's state at the
node boundary (the fork: a copy of w | m | step | data offset) or from the
shared seeded init for roots (prefix_digest(cfg, 0) is config independent); EVAL runs at every
request end and at every multiple of the study's eval interval inside a node's range -- the
same (node, step) set the engine's stage trees evaluate.  Independent subtrees run concurrently
on all host cores; every step is additionally split over OpenMP threads by independent outputs
(orc_*_train_mt), which is bitwise the single-thread result.

Used by bench.py --impl reference (timed, bounded wall budget, fraction executed reported) and
by the -m gpu study parity tests (per-trial metric histories vs the GPU engine)."""
from __future__ import annotations

import ctypes
import itertools
import json
import os
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from functools import lru_cache
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libstagemerge_ref.so"
SEED = 2006_11972
_FP = ctypes.POINTER(ctypes.c_float)
_I64P = ctypes.POINTER(ctypes.c_int64)

# executor defaults for hps a study does not tune (EngineOptions defaults, engine.hpp)
DEFAULTS = {"lr": 0.1, "momentum": 0.9, "weight_decay": 0.0, "batch_size": 128.0}
HP_COLS = ("lr", "momentum", "weight_decay", "batch_size")


def host_has_avx512() -> bool:
    try:
        flags = next(l for l in open("/proc/cpuinfo") if l.startswith("flags")).split()
    except (OSError, StopIteration):
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512cd"))


@lru_cache(None)
def oracle_lib(isa: str = "auto") -> ctypes.CDLL:
    """liboracle_v4.so (AVX-512) when the host supports it, else liboracle.so (x86-64-v3)."""
    os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")  # idle teams must not spin on shared cores
    use_v4 = (isa == "v4") or (isa == "auto" and host_has_avx512() and (HERE / "liboracle_v4.so").exists())
    lib = ctypes.CDLL(str(HERE / ("liboracle_v4.so" if use_v4 else "liboracle.so")))
    lib.isa = "x86-64-v4 (AVX-512)" if use_v4 else "x86-64-v3 (AVX2+FMA)"
    train_args = [_FP, _FP, _I64P, _I64P, _FP, ctypes.c_int64, ctypes.c_int, _FP, ctypes.c_void_p, ctypes.c_int, _FP,
                  ctypes.c_int]
    for pre in ("orc_", "orc_cnn_"):
        getattr(lib, pre + "train_mt").argtypes = train_args
        getattr(lib, pre + "train_mt").restype = ctypes.c_int
        getattr(lib, pre + "eval_mt").argtypes = [_FP, _FP, ctypes.c_void_p, ctypes.c_int,
                                                  ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        getattr(lib, pre + "init").argtypes = [ctypes.c_uint64, _FP, _FP]
        getattr(lib, pre + "gen_dataset").argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _FP,
                                                      ctypes.c_void_p, _FP, ctypes.c_void_p]
    lib.orc_layout.argtypes = [_I64P, _I64P, _I64P]
    lib.orc_cnn_layout.argtypes = [_I64P, _I64P, _I64P]
    return lib


@lru_cache(None)
def ref_lib() -> ctypes.CDLL:
    if not REF_SO.exists():
        raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, in the dev container)")
    lib = ctypes.CDLL(str(REF_SO))
    lib.ref_call.argtypes = [ctypes.c_char_p]
    lib.ref_call.restype = ctypes.c_char_p
    return lib


def ref_call(cmd: dict) -> dict:
    out = json.loads(ref_lib().ref_call(json.dumps(cmd).encode()))
    if "error" in out:
        raise RuntimeError(f"reference: {out['error']}: {out.get('what')}")
    return out


# ---- study specs (the bundled schema-1 specs) --------------------------------

def _splitmix(state: int):
    state = (state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return state, z ^ (z >> 31)


def expand_study(spec: str | dict) -> dict:
    """Trial configs of a study spec (grid: hp names sorted, last varies fastest; random: one
    splitmix64 draw per hp in name order; explicit `trials`), in the JSON form the reference shim
    parses.  The configs reach the reference's insert_trial unchanged."""
    j = json.loads(spec) if isinstance(spec, str) else spec
    spi = int(j.get("steps_per_iteration", 1))
    ms = j["max_steps"]
    max_steps = ms["epochs"] * spi if isinstance(ms, dict) else int(ms)
    ev = int(j.get("eval_interval", 0)) * (spi if j.get("eval_in_iterations") else 1)
    space = {k: v for k, v in sorted(j.get("space", {}).items())}
    names = list(space)

    def config(pick: dict, steps: int) -> dict:
        return {"total_steps": steps,
                "hps": {n: [{"fn": f, "local_start": 0, "duration": steps, "spi": spi}] for n, f in sorted(pick.items())}}

    trials = []
    sampler = j.get("sampler", {"kind": "grid"})
    if names:
        if sampler.get("kind", "grid") == "grid":
            for combo in itertools.product(*(space[n] for n in names)):
                trials.append(config(dict(zip(names, combo)), max_steps))
        elif sampler["kind"] == "random":
            state = int(sampler.get("seed", 0))
            for _ in range(int(sampler["trials"])):
                pick = {}
                for n in names:
                    state, r = _splitmix(state)
                    pick[n] = space[n][r % len(space[n])]
                trials.append(config(pick, max_steps))
        else:
            raise ValueError(f"unknown sampler {sampler['kind']}")
    hp_set = list(names)
    for t in j.get("trials", []):
        if not hp_set:
            hp_set = sorted(t["hps"])
        trials.append(config(t["hps"], int(t.get("steps", max_steps))))
    key = {"model": j.get("model", "mlp"), "dataset": j.get("dataset", "synthetic"), "hp_set": sorted(hp_set)}
    return {"key": key, "trials": trials, "max_steps": max_steps, "eval_interval": ev, "name": j.get("name", "study")}


def reference_plan(key: dict, trials: list, study: int = 0) -> dict:
    """The merged plan built by the reference (insert_trial in trial order) plus per-node hp values
    (value_at) over each node's range."""
    acts = [{"kind": "insert", "id": (study << 32) | i, "study": study, "trial": i, "config": c}
            for i, c in enumerate(trials)]
    out = ref_call({"op": "plan", "key": key, "actions": acts, "values": True, "indent": -1})
    for i, r in enumerate(out["results"]):
        if "error" in r:
            raise RuntimeError(f"reference rejected trial {i}: {r}")
    return out


# ---- models ----------------------------------------------------------------------------------

class Model:
    """The oracle's model of a study key: 'mlp' (784-256-256-10) or 'cnn'."""

    def __init__(self, name: str, lib: ctypes.CDLL, n_train: int = 65536, max_batch: int = 256, n_val: int = 4096,
                 seed: int = SEED):
        self.name, self.lib, self.seed = name, lib, seed
        pre = "orc_cnn_" if name == "cnn" else "orc_"
        self._train = getattr(lib, pre + "train_mt")
        self._eval = getattr(lib, pre + "eval_mt")
        self._init = getattr(lib, pre + "init")
        pa, pl = ctypes.c_int64(), ctypes.c_int64()
        off = (ctypes.c_int64 * 9)()
        (lib.orc_cnn_layout if name == "cnn" else lib.orc_layout)(ctypes.byref(pa), ctypes.byref(pl), off)
        self.p_algo, self.p_alloc = pa.value, pl.value
        self.d_in = 32 * 32 * 4 if name == "cnn" else 784
        self.n_train, self.max_batch, self.n_val = n_train, max_batch, n_val
        self.x = np.empty((n_train + max_batch, self.d_in), np.float32)
        self.y = np.empty(n_train + max_batch, np.int32)
        self.vx = np.empty((n_val, self.d_in), np.float32)
        self.vy = np.empty(n_val, np.int32)
        getattr(lib, pre + "gen_dataset")(seed, n_train, max_batch, n_val, self.x.ctypes.data_as(_FP),
                                          self.y.ctypes.data, self.vx.ctypes.data_as(_FP), self.vy.ctypes.data)

    def init_state(self):
        w = np.empty(self.p_alloc, np.float32)
        m = np.empty(self.p_alloc, np.float32)
        self._init(self.seed, w.ctypes.data_as(_FP), m.ctypes.data_as(_FP))
        return [w, m, ctypes.c_int64(0), ctypes.c_int64(0)]

    def train(self, st, hp: np.ndarray, n: int, threads: int) -> None:
        w, m, step, off = st
        rc = self._train(w.ctypes.data_as(_FP), m.ctypes.data_as(_FP), ctypes.byref(step), ctypes.byref(off),
                         hp.ctypes.data_as(_FP), hp.shape[0], n, self.x.ctypes.data_as(_FP), self.y.ctypes.data,
                         self.n_train, None, threads)
        if rc:
            raise RuntimeError(f"oracle train failed ({rc})")

    def eval(self, st, threads: int):
        out = (ctypes.c_double * 2)()
        self._eval(st[0].ctypes.data_as(_FP), self.vx.ctypes.data_as(_FP), self.vy.ctypes.data, self.n_val, out,
                   threads)
        return {"val_loss": out[0], "val_acc": out[1]}


def _fork(st):
    return [st[0].copy(), st[1].copy(), ctypes.c_int64(st[2].value), ctypes.c_int64(st[3].value)]


# ---- the executor --------------------------------------------------------------------------------

def run_plan(plan: dict, model: Model, eval_interval: int = 0, threads: int | None = None,
             budget_s: float | None = None, chunk: int | None = None) -> dict:
    """Executes every node of `plan` (reference_plan output) once; returns metrics per
    (node, step), executed stage-steps, wall seconds and whether the plan completed.  Training
    runs in chunks of `chunk` steps (the thread split is re-balanced and the budget checked
    between chunks)."""
    nodes = {n["id"]: n for n in plan["node_values"]}
    chunk = chunk or (2 if model.name == "cnn" else 16)
    threads = threads or os.cpu_count() or 1
    # critical path below each node (steps to its deepest request): schedule the longest first
    depth = {}
    for nid in sorted(nodes, reverse=True):  # children have larger ids than parents
        n = nodes[nid]
        depth[nid] = max([n["hi"]] + [depth[c] for c in n["children"]]) - n["start"]
    unique = sum(n["hi"] - n["start"] for n in nodes.values())
    metrics, lock = {}, threading.Lock()
    state = {"running": 0, "executed": 0, "stopped": False}
    t0 = time.perf_counter()
    pool = ThreadPoolExecutor(max_workers=threads)
    pending = []

    def table(n):
        hi, lo = n["hi"], n["start"]
        hp = np.zeros((max(hi, 1), 4), np.float32)
        for c, name in enumerate(HP_COLS):
            vals = n["hps"].get(name)
            hp[lo:hi, c] = np.float32(vals) if vals is not None else np.float32(DEFAULTS[name])
        return hp

    def submit(nid, st):
        pending.append(pool.submit(run_node, nid, st))

    def run_node(nid, st):
        n = nodes[nid]
        lo, hi = n["start"], n["hi"]
        hp = table(n)
        kids = {}
        for c in n["children"]:
            kids.setdefault(nodes[c]["start"], []).append(c)
        evals = {r["end"] for r in n["requests"]}
        if eval_interval > 0:
            evals |= set(range((lo // eval_interval + 1) * eval_interval, hi + 1, eval_interval))
        cuts = sorted({c for c in list(kids) + list(evals) if lo < c <= hi} | {hi})
        with lock:
            state["running"] += 1
        try:
            cur = lo
            for cut in cuts:
                while cur < cut:
                    with lock:
                        if budget_s is not None and time.perf_counter() - t0 > budget_s:
                            state["stopped"] = True
                        if state["stopped"]:
                            return
                        inner = max(1, threads // max(1, state["running"]))
                    k = min(chunk, cut - cur)
                    model.train(st, hp, k, inner)
                    cur += k
                    with lock:
                        state["executed"] += k
                if cut in evals:
                    with lock:
                        inner = max(1, threads // max(1, state["running"]))
                    rec = model.eval(st, inner)
                    with lock:
                        metrics[(nid, cut)] = rec
                for c in sorted(kids.get(cut, []), key=lambda c: -depth[c]):
                    submit(c, _fork(st))
        finally:
            with lock:
                state["running"] -= 1

    roots = sorted((nid for nid, n in nodes.items() if n["parent"] is None), key=lambda r: -depth[r])
    for r in roots:
        submit(r, model.init_state())
    # drain: tasks submit their children before finishing, so wait until no future is left
    done_i = 0
    while done_i < len(pending):
        pending[done_i].result()
        done_i += 1
    pool.shutdown(wait=True)
    wall = time.perf_counter() - t0
    return {"metrics": metrics, "executed": state["executed"], "unique": unique, "wall_s": wall,
            "complete": state["executed"] == unique and not state["stopped"], "threads": threads}


def trial_histories(plan: dict, metrics: dict) -> dict:
    """Per trial (study, trial): {step: record} along its plan path (the engine's history():
    metrics on each path node at steps in (start, next node's start], the last up to the end)."""
    nodes = {n["id"]: n for n in plan["node_values"]}
    out = {}
    for n in nodes.values():
        for r in n["requests"]:
            path, cur = [], n["id"]
            while cur is not None:
                path.append(cur)
                cur = nodes[cur]["parent"]
            path.reverse()
            h = {}
            for i, pid in enumerate(path):
                pn = nodes[pid]
                top = nodes[path[i + 1]]["start"] if i + 1 < len(path) else r["end"]
                for (mid, s), rec in metrics.items():
                    if mid == pid and pn["start"] < s <= top:
                        h[s] = rec
            for st, tr in r["subscribers"]:
                out[(st, tr)] = h
    return out


def total_trial_steps(plan: dict) -> int:
    return sum(r["end"] * len(r["subscribers"]) for n in plan["node_values"] for r in n["requests"])
