"""A/B probe: standalone CUDA-event times of the MLP layer-1 GEMMs and a full lockstep, for the
package found at sys.argv[1] (a worktree of another revision or this tree)."""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_2006_11972_b200 import executor as ex
for model in (ex.MODEL_MLP, ex.MODEL_CNN):
    e = ex.Executor(n_slots=64, n_ckpts=4, max_steps=64, gemm_mode=ex.GEMM_TC, model=model,
                    max_batch=256 if model == ex.MODEL_MLP else 128)
    for s in range(64):
        e.slot_init(s)
        e.hp_upload(s, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 128]), (64, 1)))
    e.train(list(range(64)), 2)
    e.sync()
    ks = (2, 3) if model == ex.MODEL_MLP else (2, 3, 4, 5, 6, 7)
    r = {k: round(e.bench_kernel(k, 64, 30) * 1e3, 1) for k in ks}
    e.set_timing(True)
    e.reset_stats()
    e.train(list(range(64)), 10)
    st = e.stats()
    print(sys.argv[1], "mlp" if model == ex.MODEL_MLP else "cnn", "kernel us", r, "lockstep us", round(st["lockstep_ms"] / 10 * 1e3, 1))
    e.close()
