"""Diagnostic: per-tensor and per-tap relative error of the tensor-core CNN gradient vs float64."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as ol  # noqa: E402
from paper_2006_11972_b200 import executor as ex  # noqa: E402
from test_cnn_oracle import grad_vector, torch_loss, unpack  # noqa: E402

ds = ol.cnn_dataset(4096, 256, 64)
_, _, off = ol.cnn_layout()
for bs in (16, 64):
    hp = np.tile(np.float32([1.0, 0.0, 0.0, bs]), (4, 1))
    res = {}
    for mode in (ex.GEMM_TC, ex.GEMM_EXACT):
        with ex.Executor(n_slots=2, n_ckpts=1, gemm_mode=mode, max_steps=8, max_batch=64, n_train=4096, n_val=256,
                         model=ex.MODEL_CNN) as e:
            e.slot_init(0)
            e.hp_upload(0, 0, hp)
            e.train([0], 1)
            res[mode] = e.slot_read(0)[1]
    o = ol.CnnSlot(ds)
    params = unpack(o.w)
    tl, _ = torch_loss(params, ds.x[:bs], ds.y[:bs])
    tl.backward()
    g = grad_vector(params, o.w)
    names = ["W1", "b1", "W2", "b2", "W3", "b3", "W4", "b4"]
    for i, (a, b) in enumerate(zip(off[:8], off[1:9])):
        errs = [np.linalg.norm(res[m][a:b] - g[a:b]) / np.linalg.norm(g[a:b]) for m in (ex.GEMM_TC, ex.GEMM_EXACT)]
        print(bs, names[i], "tc %.3e exact %.3e" % tuple(errs))
    d = (res[ex.GEMM_TC][:1152] - g[:1152]).reshape(32, 9, 4)
    gg = g[:1152].reshape(32, 9, 4)
    print("per tap rel", [float("%.2e" % (np.linalg.norm(d[:, t]) / np.linalg.norm(gg[:, t]))) for t in range(9)])
    print("per ci rel", [float("%.2e" % (np.linalg.norm(d[:, :, c]) / (np.linalg.norm(gg[:, :, c]) + 1e-30))) for c in range(4)])
    print("per co rel", [float("%.1e" % (np.linalg.norm(d[c]) / np.linalg.norm(gg[c]))) for c in range(32)])
