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


def summary(mode, wall, stage_steps, metrics, digest="d", seed=1):
    return {"mode": mode, "spec_digest": digest, "seed": seed, "gemm": "tc", "executed_merge_rate": 1.5,
            "stats": {"wall_s": wall, "stage_steps": stage_steps, "trial_steps": 900},
            "final_metrics": metrics}


def test_report(tmp_path):
    s, t = tmp_path / "s.json", tmp_path / "t.json"
    s.write_text(json.dumps(summary("stage", 2.0, 600, {"0:0": [200, 1.0, 0.5]})))
    t.write_text(json.dumps(summary("trial", 3.0, 800, {"0:0": [200, 1.0, 0.5]})))
    rc, out, _ = run_cli("report", "--stage-summary", str(s), "--trial-summary", str(t))
    r = json.loads(out)
    assert rc == 0 and r["gpu_seconds_ratio"] == 1.5 and abs(r["stage_steps_ratio"] - 4 / 3) < 1e-12
    t.write_text(json.dumps(summary("trial", 3.0, 800, {"0:0": [200, 1.0, 0.5]}, digest="other")))
    assert run_cli("report", "--stage-summary", str(s), "--trial-summary", str(t))[0] == 1
    t.write_text(json.dumps(summary("trial", 3.0, 800, {"0:0": [200, 1.0, 0.25]})))
    assert run_cli("report", "--stage-summary", str(s), "--trial-summary", str(t))[0] == 2


@pytest.mark.gpu
def test_run_stage_trial_report_deterministic(tmp_path):
    outs = {}
    for mode, tag in (("stage", "a"), ("stage", "b"), ("trial", "c")):
        path = tmp_path / f"{tag}.json"
        trace = tmp_path / f"{tag}.csv"
        rc, out, err = run_cli("run", "c1_fig1", "--mode", mode, "--gemm", "exact", "--slots", "4",
                               "--summary", str(path), "--trace", str(trace))
        assert rc == 0, err
        outs[tag] = json.loads(path.read_text())
        assert trace.read_text().count("\n") == 1 + 4                 # header + one eval per trial
    a, b = dict(outs["a"]), dict(outs["b"])
    a["stats"], b["stats"] = {k: v for k, v in a["stats"].items() if k != "wall_s"}, \
        {k: v for k, v in b["stats"].items() if k != "wall_s"}
    assert a == b                                                     # deterministic summaries
    rc, out, _ = run_cli("report", "--stage-summary", str(tmp_path / "a.json"), "--trial-summary",
                         str(tmp_path / "c.json"))
    r = json.loads(out)
    assert rc == 0 and abs(r["stage_steps_ratio"] - 4 / 3) < 1e-12 and r["trial_steps"] == 800
