"""Run-to-run determinism stress of the tensor-core CNN path: R fresh contexts train the same 64
slots for S steps; every slot's weights must be bitwise equal across runs.  Prints the slots and
parameter ranges (per layer) that differ, if any."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from paper_2006_11972_b200 import executor as ex  # noqa: E402
import oracle_lib as ol  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = 64
_, _, off = ol.cnn_layout()
names = ["W1", "b1", "W2", "b2", "W3", "b3", "W4", "b4"]
ref = None
bad = 0
for r in range(R):
    e = ex.Executor(n_slots=n, n_ckpts=2, max_steps=16, gemm_mode=ex.GEMM_TC, max_batch=128, model=ex.MODEL_CNN,
                    n_train=8192, n_val=256)
    for s in range(n):
        e.slot_init(s)
        hp = np.tile(np.float32([0.05, 0.9, 1e-4, 128 if s % 2 == 0 else 64]), (16, 1))
        e.hp_upload(s, 0, hp)
    e.train(list(range(n)), S)
    ws = [e.slot_read(s)[1 if S == 1 else 0].copy() for s in range(n)]  # 1 step: the gradient (momentum)
    e.close()
    if ref is None:
        ref = ws
        continue
    for s in range(n):
        if not np.array_equal(ws[s], ref[s]):
            bad += 1
            diff = [names[i] for i in range(8) if not np.array_equal(ws[s][off[i]:off[i + 1]], ref[s][off[i]:off[i + 1]])]
            print(f"run {r} slot {s}: differs in {diff}", flush=True)
print("runs", R, "steps", S, "mismatching slot-runs", bad)
