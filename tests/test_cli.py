"""The command-line entry point (reference SPEC.md [MODULE] cli): merge-rate, dump-plan,
dump-tree, report and their exit codes on CPU; `run` (STAGE and TRIAL, then `report`) on the GPU."""
import json
import subprocess
import sys

import pytest

from oracle_lib import ROOT
from paper_2006_11972_b200 import cli, host


def run_cli(*args):
    p = subprocess.run([sys.executable, "-m", "paper_2006_11972_b200", *args], cwd=ROOT, capture_output=True,
                       text=True)
    return p.returncode, p.stdout, p.stderr


def test_merge_rate_p_and_q():
    rc, out, _ = run_cli("merge-rate", "c1_fig1")
    assert rc == 0 and out.strip() == "p = 800/600 = 1.333333"       # PAPER Fig. 1 / SPEC acceptance 4
    rc, out, _ = run_cli("merge-rate", "c1_fig1", "c1_fig1")
    assert rc == 0 and out.startswith("q = 1600/600")                # identical studies: q = K total / unique


def test_dump_plan_and_tree_fig1():
    rc, out, _ = run_cli("dump-plan", "c1_fig1")
    plan = json.loads(out)
    assert rc == 0 and len(plan["nodes"]) == 5
    rc, out, _ = run_cli("dump-plan", "c1_fig1", "--dot")
    assert rc == 0 and out.startswith("digraph")
    rc, out, _ = run_cli("dump-tree", "c1_fig1")
    tree = json.loads(out)
    assert rc == 0 and tree["leaf_count"] == 4 and len(tree["stages"]) == 6   # 2 roots, 4 leaves


def test_config_errors_exit_1(tmp_path):
    assert run_cli("merge-rate", str(tmp_path / "missing.json"))[0] == 1
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"schema": 1, "max_steps": 10, "space": {"lr": []}}))
    assert run_cli("merge-rate", str(bad))[0] == 1
    other = tmp_path / "other.json"
    other.write_text(json.dumps({"schema": 1, "model": "cnn", "max_steps": 10,
                                 "space": {"lr": [{"family": "constant", "value": "0.1"}]}}))
    assert run_cli("merge-rate", "c1_fig1", str(other))[0] == 1      # different compatibility keys


def summary(mode, gpu_hours, stage_steps, metrics, digest="d", seed=1):
    return {"mode": mode, "spec_digest": digest, "seed": seed, "gemm": "tc", "executed_merge_rate": 1.5,
            "gpu_hours": gpu_hours, "stats": {"stage_steps": stage_steps, "trial_steps": 900},
            "final_metrics": metrics}


def test_report(tmp_path):
    s, t = tmp_path / "s.json", tmp_path / "t.json"
    s.write_text(json.dumps(summary("stage", 2.0, 600, {"0:0": [200, 1.0, 0.5]})))
    t.write_text(json.dumps(summary("trial", 3.0, 800, {"0:0": [200, 1.0, 0.5]})))
    rc, out, _ = run_cli("report", "--stage-summary", str(s), "--trial-summary", str(t))
    r = json.loads(out)
    assert rc == 0 and r["gpu_hours_ratio"] == 1.5 and abs(r["stage_steps_ratio"] - 4 / 3) < 1e-12
    t.write_text(json.dumps(summary("trial", 3.0, 800, {"0:0": [200, 1.0, 0.5]}, digest="other")))
    assert run_cli("report", "--stage-summary", str(s), "--trial-summary", str(t))[0] == 1
    t.write_text(json.dumps(summary("trial", 3.0, 800, {"0:0": [200, 1.0, 0.25]})))
    assert run_cli("report", "--stage-summary", str(s), "--trial-summary", str(t))[0] == 2


def write_trace(path, mode, rows, seed=1, digest="d"):
    with open(path, "w") as f:
        f.write(f"# smx trace v1 mode={mode} seed={seed} spec_digest={digest} (time_us = ...)\n")
        f.write("time_us,worker,kind,node,start,end,detail\n")
        for r in rows:
            f.write(",".join(map(str, r)) + "\n")


def test_report_on_traces(tmp_path):
    s, t = tmp_path / "s.csv", tmp_path / "t.csv"
    ev = "val_acc=0.5;val_loss=1.25;trials=0:0"
    write_trace(s, "stage", [(0, 0, "LOAD", 0, 0, 0, "init"), (0, 0, "TRAIN", 0, 0, 100, ""),
                             (100, 0, "EVAL", 0, 100, 100, ev)])
    write_trace(t, "trial", [(0, 0, "LOAD", 0, 0, 0, "init"), (0, 0, "TRAIN", 0, 0, 150, ""),
                             (150, 0, "EVAL", 0, 100, 100, ev)])
    rc, out, err = run_cli("report", "--stage-trace", str(s), "--trial-trace", str(t))
    assert rc == 0, err
    assert json.loads(out)["gpu_steps_ratio"] == 1.5
    write_trace(t, "trial", [(0, 0, "EVAL", 0, 100, 100, ev)], seed=2)
    assert run_cli("report", "--stage-trace", str(s), "--trial-trace", str(t))[0] == 1   # mismatched seeds
    write_trace(t, "trial", [(0, 0, "EVAL", 0, 100, 100, ev.replace("1.25", "1.5"))])
    assert run_cli("report", "--stage-trace", str(s), "--trial-trace", str(t))[0] == 2   # metrics differ


@pytest.mark.gpu
def test_run_stage_trial_report_deterministic(tmp_path):
    outs = {}
    for mode, tag in (("stage", "a"), ("stage", "b"), ("trial", "c")):
        path = tmp_path / f"{tag}.json"
        trace = tmp_path / f"{tag}.csv"
        rc, out, err = run_cli("run", "c1_fig1", "--mode", mode, "--gemm", "exact", "--slots", "4",
                               "--summary", str(path), "--trace", str(trace))
        assert rc == 0, err
        outs[tag] = (path.read_text(), trace.read_text())
    assert outs["a"] == outs["b"]                      # acceptance 10: byte-identical summary + trace
    summ = json.loads(outs["a"][0])
    assert set(summ["best_metric"]) == {"0:0", "0:1", "0:2", "0:3"} and summ["gpu_hours"] > 0
    rc, out, _ = run_cli("report", "--stage-summary", str(tmp_path / "a.json"), "--trial-summary",
                         str(tmp_path / "c.json"))
    r = json.loads(out)
    assert rc == 0 and abs(r["stage_steps_ratio"] - 4 / 3) < 1e-12 and r["trial_steps"] == 800
    assert abs(r["gpu_hours_ratio"] - 4 / 3) < 1e-12                # savings law (acceptance 4)
    rc, out, _ = run_cli("report", "--stage-trace", str(tmp_path / "a.csv"), "--trial-trace", str(tmp_path / "c.csv"))
    r = json.loads(out)
    assert rc == 0 and abs(r["gpu_steps_ratio"] - 4 / 3) < 1e-12 and r["trials"] == 4
