"""A/B of the conv1 kernels (64 slots, bs 128, tensor-core mode): standalone CUDA-event times of
kinds 8 (conv1 weight gradient + reduce) and 9 (conv1 forward) and a 10-lockstep time, under the
current environment (SMX_CONV1_WGRAD_LANE=1 selects the FFMA2 weight-gradient kernel)."""
import os
import sys
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else ".")
import numpy as np
from paper_2006_11972_b200 import executor as ex
e = ex.Executor(n_slots=64, n_ckpts=4, max_steps=64, gemm_mode=ex.GEMM_TC, model=ex.MODEL_CNN, max_batch=128)
for s in range(64):
    e.slot_init(s)
    e.hp_upload(s, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 128]), (64, 1)))
e.train(list(range(64)), 2)
e.sync()
r = {k: round(e.bench_kernel(k, 64, 20) * 1e3, 1) for k in (8, 9, 2, 3, 4, 5, 6, 7)}
e.set_timing(True)
e.reset_stats()
e.train(list(range(64)), 10)
st = e.stats()
print("lane" if os.environ.get("SMX_CONV1_WGRAD_LANE") else "tc", "kernel us", r, "lockstep us",
      round(st["lockstep_ms"] / 10 * 1e3, 1), flush=True)
