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
