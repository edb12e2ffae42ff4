"""CUDA-event timing of the CNN tensor-core kernels through smx_bench_kernel (warm, 64 slots, bs
128): A/B comparison of library builds on the same box.

    python profiles/debug/kbench.py lib_a.so [lib_b.so ...]
"""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
    import numpy as np
    from paper_2006_11972_b200 import executor as ex
    n = 64
    e = ex.Executor(n_slots=n, n_ckpts=4, max_steps=64, gemm_mode=ex.GEMM_TC, max_batch=128, model=ex.MODEL_CNN)
    for s in range(n):
        e.slot_init(s)
        e.hp_upload(s, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 128]), (64, 1)))
    e.train(list(range(n)), 2)
    e.sync()
    names = {2: "Fwd2", 3: "Wgrad2", 4: "Dgrad2", 5: "Dgrad3", 6: "Fwd3", 7: "Wgrad3+red"}
    out = {names[k]: round(e.bench_kernel(k, n, 20) * 1e3, 1) for k in names}
    print(json.dumps(out))
    sys.exit(0)

for lib in sys.argv[1:]:
    env = dict(os.environ, SMX_LIB_PATH=os.path.abspath(lib))
    r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr[-500:])
