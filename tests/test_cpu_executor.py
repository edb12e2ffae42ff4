"""The reference-side CPU executor (oracle/cpu_executor.py): plans built by the compiled
reference (oracle/_ref), training by the CPU oracle.  Checked here on CPU:

* its study expansion yields the same plan (signature) as the product engine's parser;
* the multi-threaded oracle entry points and the AVX-512 build are bitwise the single-thread
  x86-64-v3 oracle (so the timed baseline computes exactly what the checker computes);
* executing a merged plan gives every trial bitwise the metrics of training it alone (STAGE ==
  TRIAL), each unique stage-step exactly once."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as ol

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests" / "native"))
import cpu_executor as cx  # noqa: E402

STUDIES = ROOT / "paper_2006_11972_b200" / "studies"
pytestmark = pytest.mark.skipif(not cx.REF_SO.exists(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name", ["c1_fig1", "c2_grid", "c3_random", "c4_sha", "c5_space"])
def test_expansion_matches_product_parser(name):
    stub = pytest.importorskip("_stagemerge_stub")
    spec = (STUDIES / f"{name}.json").read_text()
    info = cx.expand_study(spec)
    mine = json.loads(stub.expand_study(spec))
    assert info["key"] == mine["key"] and info["max_steps"] == mine["max_steps"]
    assert info["eval_interval"] == mine["eval_interval"] and len(info["trials"]) == len(mine["trials"])
    plan = cx.reference_plan(info["key"], info["trials"])
    e = stub.Engine(json.dumps(info["key"]), json.dumps({"slots_per_gpu": 1, "max_steps": 8192}))
    e.submit_study(spec, 0)
    assert plan["signature"] == e.signature()
    unique = sum(n["hi"] - n["start"] for n in plan["node_values"])
    assert unique == mine["unique_steps"]
    assert cx.total_trial_steps(plan) == mine["total_steps"]


def _slot_state(lib, cnn):
    pa, pl = ctypes_layout(lib, cnn)
    w = np.empty(pl, np.float32)
    m = np.empty(pl, np.float32)
    (lib.orc_cnn_init if cnn else lib.orc_init)(cx.SEED, w.ctypes.data_as(cx._FP), m.ctypes.data_as(cx._FP))
    return w, m


def ctypes_layout(lib, cnn):
    import ctypes
    pa, pl = ctypes.c_int64(), ctypes.c_int64()
    off = (ctypes.c_int64 * 9)()
    (lib.orc_cnn_layout if cnn else lib.orc_layout)(ctypes.byref(pa), ctypes.byref(pl), off)
    return pa.value, pl.value


@pytest.mark.parametrize("cnn", [False, True])
def test_multithreaded_and_avx512_builds_are_bitwise_the_oracle(cnn):
    name = "cnn" if cnn else "mlp"
    v3 = cx.oracle_lib("v3")
    m3 = cx.Model(name, v3, n_train=4096, max_batch=64, n_val=256)
    hp = np.tile(np.float32([0.05, 0.9, 5e-4, 64]), (3, 1))
    hp[1, 3] = 48
    outs = []
    libs = [(v3, 1), (v3, 7)]
    if cx.host_has_avx512() and (cx.HERE / "liboracle_v4.so").exists():
        libs.append((cx.oracle_lib("v4"), 5))
    for lib, th in libs:
        mdl = m3 if lib is v3 else cx.Model(name, lib, n_train=4096, max_batch=64, n_val=256)
        st = mdl.init_state()
        mdl.train(st, hp, 3, th)
        outs.append((st[0].copy(), st[1].copy(), st[3].value, mdl.eval(st, th)))
    # and the single-thread path the GPU tests check against (tests/oracle_lib, orc_*_train)
    if cnn:
        o = ol.CnnSlot(ol.cnn_dataset(4096, 256, 64), max_steps=4)
    else:
        d = ol.Dataset(n_train=4096, max_batch=64, n_val=256)
        o = ol.Slot(max_steps=4)
    o.train(hp, 3) if cnn else o.train(hp, 3, ds=d)
    for w, m, off, ev in outs:
        assert np.array_equal(w, outs[0][0]) and np.array_equal(m, outs[0][1]) and off == outs[0][2]
        assert ev == outs[0][3]
    assert np.array_equal(outs[0][0], o.w) and np.array_equal(outs[0][1], o.m)


def test_merged_plan_execution_equals_trial_by_trial():
    spec = {"schema": 1, "name": "fig1_short", "model": "mlp", "max_steps": 24, "eval_interval": 8,
            "trials": [{"hps": {"lr": {"family": "step", "values": ["0.1", "0.01"], "milestones": [12]}}},
                       {"hps": {"lr": {"family": "step", "values": ["0.1", "0.001"], "milestones": [12]}}},
                       {"hps": {"lr": {"family": "step", "values": ["0.01", "0.001"], "milestones": [12]}}},
                       {"hps": {"lr": {"family": "constant", "value": "0.01"}}, "steps": 20}]}
    info = cx.expand_study(json.dumps(spec))
    plan = cx.reference_plan(info["key"], info["trials"])
    model = cx.Model("mlp", cx.oracle_lib(), n_train=4096, max_batch=128, n_val=256)
    res = cx.run_plan(plan, model, eval_interval=8, threads=4, chunk=5)
    assert res["complete"] and res["executed"] == res["unique"] == 12 + 12 + 12 + 20 + 12
    hist = cx.trial_histories(plan, res["metrics"])
    for t, cfg in enumerate(info["trials"]):
        T = cfg["total_steps"]
        # trial alone: its hp table from the reference's value_at, trained from init
        one = cx.reference_plan(info["key"], [cfg])
        st = model.init_state()
        hp = np.zeros((T, 4), np.float32)
        for node in one["node_values"]:  # a single trial's plan is one chain of nodes
            for c, hname in enumerate(cx.HP_COLS):
                hp[node["start"]:node["hi"], c] = node["hps"].get(hname, [cx.DEFAULTS[hname]] * (node["hi"] - node["start"]))
        expect = {}
        for s in range(1, T + 1):
            model.train(st, hp, 1, 1)
            if s % 8 == 0 or s == T:
                expect[s] = model.eval(st, 1)
        assert hist[(0, t)] == expect, t
