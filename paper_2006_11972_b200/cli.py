"""Command-line entry point (reference SPEC.md [MODULE] cli).

    python -m paper_2006_11972_b200 run SPEC [SPEC ...] [--mode stage|trial] [--summary PATH]
                                        [--trace PATH] [--gemm tc|exact] [--slots N] [--device D]
                                        [--seed S] [--step-cost TABLE] [--timing PATH]
    python -m paper_2006_11972_b200 merge-rate SPEC [SPEC ...]
    python -m paper_2006_11972_b200 report --stage-trace A --trial-trace B   (or --stage-summary / --trial-summary)
    python -m paper_2006_11972_b200 dump-plan SPEC [SPEC ...] [--dot]
    python -m paper_2006_11972_b200 dump-tree SPEC [SPEC ...]

Exit codes follow the reference (types.hpp:31-43): 0 ok, 1 configuration error,
2 integrity error.  `run` executes on the B200 executor (it needs a GPU; there is no CPU
fallback); the other subcommands are host-only.  Specs are the JSON study files (schema 1) of
`studies/`; a spec with a "tuner" object runs under that tuner, otherwise every trial is
submitted at once.  Trace (SPEC.md:436 columns; time = the logical lockstep clock) and summary
(gpu_hours / end_to_end_s from the cost model over the executed schedule, per-trial best_metric)
are byte-identical for a fixed spec and seed (acceptance 10); measured time goes to --timing.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import json
import sys

from . import host


class CliError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _read(path: str) -> str:
    try:
        return host.study_spec(path)
    except OSError as e:
        raise CliError(1, f"cannot read spec {path}: {e}")


def _specs(paths):
    return [_read(p) for p in paths]


def _digest(specs) -> str:
    h = hashlib.sha256()
    for s in specs:
        h.update(json.dumps(json.loads(s), sort_keys=True).encode())
    return h.hexdigest()[:16]


def _inserts(specs):
    """Plan insert actions for every trial of every spec (study ids 0..)."""
    acts, key = [], None
    for study, spec in enumerate(specs):
        info = host.expand_study(spec)
        if key is None:
            key = info["key"]
        elif info["key"] != key:
            raise CliError(1, "studies have different compatibility keys")
        for t, cfg in enumerate(info["trials"]):
            acts.append({"kind": "insert", "id": (study << 32) | t, "study": study, "trial": t, "config": cfg})
    return key, acts


def cmd_merge_rate(a) -> dict:
    specs = _specs(a.spec)
    total, unique = host._native.merge_rate_specs(specs)
    out = {"total_steps": total, "unique_steps": unique, "merge_rate": total / unique,
           "studies": len(specs), "name": "q" if len(specs) > 1 else "p"}
    print(f"{out['name']} = {total}/{unique} = {total / unique:.6f}")
    return out


def cmd_dump_plan(a) -> dict:
    key, acts = _inserts(_specs(a.spec))
    r = host.call({"op": "plan", "key": key, "actions": acts})
    if "error" in r:
        raise CliError(1 if r["error"] == "ConfigError" else 2, r["what"])
    print(r["dot"] if a.dot else r["json"])
    return r


def cmd_dump_tree(a) -> dict:
    key, acts = _inserts(_specs(a.spec))
    r = host.call({"op": "plan", "key": key, "actions": acts, "tree": {}})
    if "error" in r:
        raise CliError(1 if r["error"] == "ConfigError" else 2, r["what"])
    print(json.dumps(r["tree"], indent=1))
    return r["tree"]


TRACE_COLUMNS = ["time_us", "worker", "kind", "node", "start", "end", "detail"]


def _best(hist):
    if not hist:
        return None
    return {"val_acc": max(v for _, _, v in hist), "val_loss": min(v for _, v, _ in hist)}


def cmd_run(a) -> dict:
    specs = _specs(a.spec)
    from . import executor as ex

    tuned = any("tuner" in json.loads(s) for s in specs)
    info = host.expand_study(specs[0])
    opts = dict(devices=[a.device], slots_per_gpu=a.slots, gemm_mode=ex.GEMM_TC if a.gemm == "tc" else ex.GEMM_EXACT,
                trial_mode=a.mode == "trial", max_batch=a.max_batch)
    if a.seed is not None:
        opts["seed"] = a.seed
    if a.step_cost:
        try:
            opts["step_cost_us"] = {str(k): float(v) for k, v in json.load(open(a.step_cost)).items()}
        except (OSError, ValueError) as e:
            raise CliError(1, f"cannot read step-cost table {a.step_cost}: {e}")
    eng = host.Engine.for_study(specs[0], **opts)
    outcomes = None
    if tuned:
        outcomes = eng.run_tuned(specs)
    else:
        for i, s in enumerate(specs):
            eng.submit_study(s, i)
        eng.run()
    st = eng.stats()
    hist = eng.histories()
    digest = _digest(specs)
    seed = opts.get("seed", 2006_11972)
    # deterministic summary (acceptance 10): GPU-hours / end-to-end from the cost model over the
    # executed schedule (SPEC.md:436 keys); measured device time goes to --timing / stdout
    summary = {
        "mode": a.mode, "specs": [json.loads(s).get("name", "") for s in specs], "spec_digest": digest,
        "seed": seed, "model": info["key"]["model"], "gemm": a.gemm,
        "gpu_hours": st["model_busy_us"] / 3.6e9, "end_to_end_s": st["model_wall_us"] / 1e6,
        "cost_model": "step_cost_us table" if a.step_cost else "bs-proportional (1 us per sample per step)",
        "merge_rate_executed": st["trial_steps"] / max(1, st["stage_steps"]),
        "executed_merge_rate": st["trial_steps"] / max(1, st["stage_steps"]),
        "stats": {k: v for k, v in st.items() if k not in ("wall_s",)},
        "signature_digest": hashlib.sha256(eng.signature().encode()).hexdigest()[:16],
        "tuners": outcomes,
        "best_metric": {f"{s}:{t}": _best(v) for (s, t), v in sorted(hist.items())},
        "final_metrics": {f"{s}:{t}": (v[-1] if v else None) for (s, t), v in sorted(hist.items())},
    }
    if a.trace:
        with open(a.trace, "w", newline="") as f:
            f.write(f"# smx trace v1 mode={a.mode} seed={seed} spec_digest={digest} "
                    f"(time_us = the engine's logical lockstep clock in training steps)\n")
            w = csv.writer(f, lineterminator="\n")
            w.writerow(TRACE_COLUMNS)
            for ev in eng.trace():
                w.writerow(ev)
    if a.summary:
        with open(a.summary, "w") as f:
            json.dump(summary, f, indent=1, sort_keys=True)
    timing = {"wall_s": st["wall_s"], "kernel_launches": st["kernel_launches"], "mode": a.mode}
    if a.timing:
        with open(a.timing, "w") as f:
            json.dump(timing, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("mode", "specs", "executed_merge_rate", "gpu_hours")} |
                     {"stats": st}))
    return summary


def _read_trace(path: str) -> dict:
    try:
        lines = open(path).read().splitlines()
    except OSError as e:
        raise CliError(1, f"cannot read trace {path}: {e}")
    if not lines or not lines[0].startswith("# smx trace v1"):
        raise CliError(1, f"{path}: not an smx trace")
    meta = dict(kv.split("=", 1) for kv in lines[0][2:].split() if "=" in kv)
    rows = list(csv.reader(lines[1:]))
    if not rows or rows[0] != TRACE_COLUMNS:
        raise CliError(1, f"{path}: bad trace header")
    busy, counts, metrics = 0, {}, {}
    for r in rows[1:]:
        t, _, kind, _, start, end, detail = r
        counts[kind] = counts.get(kind, 0) + 1
        if kind == "TRAIN":
            busy += int(end) - int(start)
        if kind == "EVAL" and "trials=" in detail:
            vals = dict(kv.split("=", 1) for kv in detail.split(";"))
            for tr in vals["trials"].split(","):
                metrics[tr] = (int(end), vals["val_loss"], vals["val_acc"])
    return {"meta": meta, "busy_steps": busy, "counts": counts, "metrics": metrics}


def cmd_report(a) -> dict:
    if a.stage_trace or a.trial_trace:
        if not (a.stage_trace and a.trial_trace):
            raise CliError(1, "report needs both --stage-trace and --trial-trace")
        st, tr = _read_trace(a.stage_trace), _read_trace(a.trial_trace)
        if st["meta"].get("mode") != "stage" or tr["meta"].get("mode") != "trial":
            raise CliError(1, "report needs one stage-mode and one trial-mode trace")
        for k in ("seed", "spec_digest"):
            if st["meta"].get(k) != tr["meta"].get(k):
                raise CliError(1, f"traces differ in {k}: {st['meta'].get(k)} vs {tr['meta'].get(k)}")
        if st["metrics"] != tr["metrics"]:
            raise CliError(2, "STAGE and TRIAL metrics differ (SPEC.md:421 metric equivalence violated)")
        out = {"gpu_steps_ratio": tr["busy_steps"] / max(1, st["busy_steps"]),
               "stage_busy_steps": st["busy_steps"], "trial_busy_steps": tr["busy_steps"],
               "trials": len(st["metrics"]), "stage_events": st["counts"], "trial_events": tr["counts"]}
        print(json.dumps(out))
        return out
    if not (a.stage_summary and a.trial_summary):
        raise CliError(1, "report needs --stage-trace/--trial-trace or --stage-summary/--trial-summary")
    try:
        stage = json.load(open(a.stage_summary))
        trial = json.load(open(a.trial_summary))
    except (OSError, ValueError) as e:
        raise CliError(1, f"cannot read summaries: {e}")
    if stage.get("mode") != "stage" or trial.get("mode") != "trial":
        raise CliError(1, "report needs one stage-mode and one trial-mode summary")
    for k in ("spec_digest", "seed", "gemm"):
        if stage.get(k) != trial.get(k):
            raise CliError(1, f"summaries differ in {k}: {stage.get(k)} vs {trial.get(k)}")
    if stage["final_metrics"] != trial["final_metrics"]:
        raise CliError(2, "STAGE and TRIAL metrics differ (SPEC.md:421 metric equivalence violated)")
    out = {"gpu_hours_ratio": trial.get("gpu_hours", 0) / stage["gpu_hours"] if stage.get("gpu_hours") else None,
           "stage_steps_ratio": trial["stats"]["stage_steps"] / stage["stats"]["stage_steps"],
           "executed_merge_rate": stage["executed_merge_rate"],
           "trial_steps": stage["stats"]["trial_steps"]}
    print(json.dumps(out))
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2006_11972_b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("spec", nargs="+")
    r.add_argument("--mode", default="stage", choices=["stage", "trial"])
    r.add_argument("--summary")
    r.add_argument("--trace")
    r.add_argument("--gemm", default="tc", choices=["tc", "exact"])
    r.add_argument("--slots", type=int, default=64)
    r.add_argument("--device", type=int, default=0)
    r.add_argument("--max-batch", type=int, default=256)
    r.add_argument("--seed", type=int)
    r.add_argument("--step-cost", help="JSON {batch_size: us per stage-step} profile table (set_runtime feed)")
    r.add_argument("--timing", help="write measured device/wall time here (kept out of the deterministic summary)")
    m = sub.add_parser("merge-rate")
    m.add_argument("spec", nargs="+")
    rep = sub.add_parser("report")
    rep.add_argument("--stage-trace")
    rep.add_argument("--trial-trace")
    rep.add_argument("--stage-summary")
    rep.add_argument("--trial-summary")
    d = sub.add_parser("dump-plan")
    d.add_argument("spec", nargs="+")
    d.add_argument("--dot", action="store_true")
    t = sub.add_parser("dump-tree")
    t.add_argument("spec", nargs="+")
    a = ap.parse_args(argv)
    fn = {"run": cmd_run, "merge-rate": cmd_merge_rate, "report": cmd_report, "dump-plan": cmd_dump_plan,
          "dump-tree": cmd_dump_tree}[a.cmd]
    try:
        fn(a)
    except CliError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.code
    except ValueError as e:  # ConfigError from the host library
        print(f"error: {e}", file=sys.stderr)
        return 1
    except RuntimeError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2 if "IntegrityError" in str(e) else 3
    return 0
