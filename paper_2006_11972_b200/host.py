"""Python face of the C++ host library (`_stagemerge`): the JSON command interface and the
study engine.  Fails loudly if the native module is not built."""
from __future__ import annotations

import json

try:
    from . import _stagemerge as _native
except ImportError as e:  # pragma: no cover - build problem, not a fallback
    raise ImportError("paper_2006_11972_b200/_stagemerge is not built; run "
                      "`python -m paper_2006_11972_b200.build`") from e


def call(cmd: dict) -> dict:
    """Run one JSON command (same schema as oracle/ref_shim.cpp) through the C++ host library."""
    return json.loads(_native.call(json.dumps(cmd)))


STUDIES = __import__("pathlib").Path(__file__).resolve().parent / "studies"


def study_spec(name_or_path) -> str:
    """Text of a bundled study spec (studies/<name>.json) or of a spec file path."""
    from pathlib import Path

    p = Path(name_or_path)
    if not p.exists():
        p = STUDIES / f"{name_or_path}.json"
    return p.read_text()


def expand_study(spec: str) -> dict:
    return json.loads(_native.expand_study(spec))


class Tuner:
    """A tuner state machine on its own (no engine): start() / on_result() return the actions
    ("SUBMIT t end", "EXTEND t end", "STOP t", "DONE a,b") the C++ tuner issues."""

    def __init__(self, spec: str):
        self._t = _native.Tuner(spec)

    def start(self) -> list:
        return self._t.start()

    def on_result(self, trial: int, end: int, metrics: dict) -> list:
        return self._t.on_result(trial, end, metrics)

    def done(self) -> bool:
        return self._t.done()

    def winners(self) -> list:
        return self._t.winners()


def sha_rungs(spec: str):
    return _native.sha_rungs(spec)


class Engine:
    """The study engine: plan + stage trees + scheduler (C++) driving the B200 executor."""

    def __init__(self, key: dict, **options):
        self._e = _native.Engine(json.dumps(key), json.dumps(options))
        self.key, self.options = key, options

    @classmethod
    def for_study(cls, spec: str, **options) -> "Engine":
        info = expand_study(spec)
        if info["eval_interval"] and "eval_intervals" not in options:
            options["eval_intervals"] = [info["eval_interval"]]
        options.setdefault("max_steps", max(4096, info["max_steps"]))
        return cls(info["key"], **options)

    def submit_study(self, spec: str, study: int = 0) -> int:
        return self._e.submit_study(spec, study)

    def submit(self, config: dict, request_id: int, study: int = 0, trial: int = 0):
        return self._e.submit(json.dumps(config), request_id, study, trial)

    def cancel(self, study: int, trial: int) -> bool:
        return self._e.cancel(study, trial)

    def run_tuned(self, specs, base_study: int = 0) -> list:
        """Runs every study spec under its own tuner (spec key "tuner") until each is DONE;
        returns per study {study, winners, actions, trained_to, trial_steps}."""
        if isinstance(specs, str):
            specs = [specs]
        return json.loads(self._e.run_tuned(list(specs), base_study))

    def run(self) -> None:
        self._e.run()

    def reset(self) -> None:
        self._e.reset()

    def stats(self) -> dict:
        return json.loads(self._e.stats())

    def trace(self) -> list:
        """Execution events (time, worker, kind, node, start, end, detail); time = the logical
        lockstep clock in steps (deterministic)."""
        return self._e.trace()

    def collect_checkpoints(self) -> int:
        return self._e.collect_checkpoints()

    def calibrate(self, batch_sizes) -> dict:
        """Profile us per stage-step for each batch size into the engine's step-cost table."""
        self._e.calibrate(list(batch_sizes))
        return self._e.step_cost_us()

    def on_complete(self, fn) -> None:
        """fn(node, end, [(study, trial), ...]) on every completed request (may call cancel)."""
        self._e.on_complete(fn)

    def signature(self) -> str:
        return self._e.signature()

    def plan_json(self) -> dict:
        return json.loads(self._e.plan_json())

    def trials(self):
        return self._e.trials()

    def history(self, study: int, trial: int):
        return self._e.history(study, trial)

    def histories(self) -> dict:
        return {t: self._e.history(*t) for t in self._e.trials()}

    def dataset_digest(self) -> int:
        return self._e.dataset_digest()

    def owned_roots(self):
        return self._e.owned_roots()

    def context_ptrs(self):
        return self._e.context_ptrs()

    def upload_dataset(self, x, y, vx, vy) -> None:
        """Host->device copy of a dataset (numpy arrays; pinned buffers give DMA-speed copies)."""
        self._e.upload_dataset_ptrs(x.ctypes.data, y.ctypes.data, vx.ctypes.data, vy.ctypes.data)
