"""Lockstep time vs active-slot count (CNN, tensor-core mode, bs 128, graphs on = the engine path).

C2's 41,000 stage-steps run in 1,200 locksteps at 34 active slots on average, so the per-slot cost
at low occupancy sets the study time as much as the 64-slot lockstep does.  Wall-clock over a
synchronised block of locksteps (a probe, not a bench number).

    python profiles/occupancy_sweep.py [--steps 40] [--counts 1,4,8,16,24,32,48,64]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11972_b200 import executor as ex  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--counts", default="1,2,4,8,12,16,20,24,32,40,48,56,64")
ap.add_argument("--bs", type=int, default=128)
a = ap.parse_args()
counts = [int(x) for x in a.counts.split(",")]
S = max(counts)
e = ex.Executor(n_slots=S, n_ckpts=4, max_steps=4 * a.steps + 16, gemm_mode=ex.GEMM_TC, model=ex.MODEL_CNN,
                max_batch=128)
hp = np.tile(np.float32([0.01, 0.9, 5e-4, a.bs]), (4 * a.steps + 16, 1))
for s in range(S):
    e.slot_init(s)
    e.hp_upload(s, 0, hp)
out = []
for n in counts:
    slots = list(range(n))
    e.train(slots, 3)
    e.sync()
    best = 1e9
    for _ in range(2):
        t0 = time.perf_counter()
        e.train(slots, a.steps)
        e.sync()
        best = min(best, (time.perf_counter() - t0) / a.steps * 1e3)
    for s in range(S):  # keep every slot's step counter inside its hp table
        e.slot_init(s)
    out.append({"slots": n, "ms_per_lockstep": round(best, 4), "us_per_stage_step": round(best * 1e3 / n, 2)})
    print(json.dumps(out[-1]), flush=True)
