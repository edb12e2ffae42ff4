"""Diagnose the tensor-core weight gradients against the oracle: one step (lr 1, mu 0 -> m = g)
at a small batch; per-layer / per-output-channel / per-(tap, ci) error structure."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
import numpy as np
import oracle_lib as ol
from paper_2006_11972_b200 import executor as ex

bs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ds = ol.cnn_dataset(4096, 256, 64)
hp = np.tile(np.float32([1.0, 0.0, 0.0, bs]), (4, 1))
with ex.Executor(n_slots=2, n_ckpts=1, gemm_mode=ex.GEMM_TC, max_steps=4, max_batch=64, n_train=4096, n_val=256,
                 model=ex.MODEL_CNN) as e:
    e.slot_init(0)
    e.hp_upload(0, 0, hp)
    e.train([0], 1)
    _, m = e.slot_read(0)
o = ol.CnnSlot(ds, max_steps=4)
o.train(hp, 1)
_, _, off = ol.cnn_layout()
names = ["W1", "b1", "W2", "b2", "W3", "b3", "W4", "b4"]
cout = (32, 32, 64, 64, 128, 128, 16, 16)
for i, (a, b) in enumerate(zip(off[:8], off[1:9])):
    g, r = m[a:b].astype(np.float64), o.m[a:b].astype(np.float64)
    rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
    print(f"{names[i]}: rel {rel:.3e}")
    if rel > 1e-4 and names[i] in ("W2", "W3"):
        C = cout[i]
        k = (b - a) // C
        G, R = g.reshape(C, k), r.reshape(C, k)
        rowerr = np.linalg.norm(G - R, axis=1) / np.maximum(np.linalg.norm(R, axis=1), 1e-30)
        colerr = np.linalg.norm(G - R, axis=0) / np.maximum(np.linalg.norm(R, axis=0), 1e-30)
        print("  per co:", np.array2string(rowerr, precision=2, max_line_width=200))
        print("  per k (first 64):", np.array2string(colerr[:64], precision=2, max_line_width=200))
        # is G a permutation of R along co?  best matching row for each co
        match = [int(np.argmin(np.linalg.norm(R - G[c], axis=1))) for c in range(C)]
        print("  best-matching oracle co for each co:", match)
