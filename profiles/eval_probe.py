"""Eval cost probe (CNN, tensor-core mode, 64-slot context, 4,096 validation samples): wall time of
smx_eval for k slots (synchronous call: forward in max_batch chunks + the fixed-order reduction),
next to the 64-slot lockstep time.  A probe, not a bench number."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11972_b200 import executor as ex  # noqa: E402

e = ex.Executor(n_slots=64, n_ckpts=4, max_steps=64, gemm_mode=ex.GEMM_TC, model=ex.MODEL_CNN, max_batch=128)
hp = np.tile(np.float32([0.01, 0.9, 5e-4, 128]), (64, 1))
for s in range(64):
    e.slot_init(s)
    e.hp_upload(s, 0, hp)
e.train(list(range(64)), 2)
e.sync()
for k in (1, 2, 4, 8, 16, 64):
    e.eval(list(range(k)))
    t0 = time.perf_counter()
    for _ in range(3):
        e.eval(list(range(k)))
    dt = (time.perf_counter() - t0) / 3 * 1e3
    print(json.dumps({"eval_slots": k, "ms": round(dt, 3), "ms_per_slot": round(dt / k, 3)}), flush=True)
t0 = time.perf_counter()
e.train(list(range(64)), 10)
e.sync()
print(json.dumps({"lockstep_ms_64": round((time.perf_counter() - t0) / 10 * 1e3, 3)}))
