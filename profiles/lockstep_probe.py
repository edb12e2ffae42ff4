"""Profiling probe: a fixed number of grouped training locksteps on a typical active set
(64 slots, bs 128, MLP or CNN) so ncu can capture every kernel of a lockstep.

    python profiles/lockstep_probe.py [--gemm tc|exact] [--slots 64] [--steps 3] [--warmup 2]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11972_b200 import executor as ex  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gemm", default="tc")
ap.add_argument("--slots", type=int, default=64)
ap.add_argument("--bs", type=int, default=128)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--model", default="mlp", choices=["mlp", "cnn"])
ap.add_argument("--max-batch", type=int, default=0, help="0: the executor default")
a = ap.parse_args()
e = ex.Executor(n_slots=a.slots, n_ckpts=4, max_steps=64, gemm_mode=ex.GEMM_TC if a.gemm == "tc" else ex.GEMM_EXACT,
                model=ex.MODEL_CNN if a.model == "cnn" else ex.MODEL_MLP, **({"max_batch": a.max_batch} if a.max_batch else {}))
e.set_graphs(False)
hp = np.tile(np.float32([0.05, 0.9, 1e-4, a.bs]), (64, 1))
for s in range(a.slots):
    e.slot_init(s)
    e.hp_upload(s, 0, hp)
slots = list(range(a.slots))
e.train(slots, a.warmup)
e.sync()
e.set_timing(True)
e.reset_stats()
e.train(slots, a.steps)
st = e.stats()
print({k: st[k] for k in ("lockstep_ms", "update_ms", "gemm_ms", "locksteps")},
      "ms/lockstep", st["lockstep_ms"] / a.steps)
