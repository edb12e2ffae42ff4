"""Per-chunk timeline of one CTA of a conv_ws kernel (profiling variant built with
-DSMX_DBG_TIMELINE: profiles/debug/var/libsmx_TIMELINE.so, loaded through SMX_LIB_PATH).

    SMX_LIB_PATH=profiles/debug/var/libsmx_TIMELINE.so python profiles/debug/timeline.py [kind ...]

kind 2 = conv2 forward, 3 = conv2 weight gradient (smx_bench_kernel kinds, 64 slots at bs 128).
Prints, per producer chunk, the cycles spent waiting for its own A copies, in the gather/refill,
waiting for the stage (MMA of the previous use), and in the TMEM/smem stores; per MMA chunk the
wait for `full` and the issue time; per epilogue unit the wait for `acc_full`.
"""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2006_11972_b200 import executor as ex  # noqa: E402

kinds = [int(k) for k in sys.argv[1:]] or [2, 3]
n = 64
e = ex.Executor(n_slots=n, n_ckpts=4, max_steps=64, gemm_mode=ex.GEMM_TC, max_batch=128, model=ex.MODEL_CNN)
for s in range(n):
    e.slot_init(s)
    e.hp_upload(s, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 128]), (64, 1)))
e.train(list(range(n)), 1)
e.sync()
lib = e._lib
lib.smx_dbg_timeline.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 4096)()
for kind in kinds:
    assert lib.smx_dbg_timeline(1, buf, 4096) == 0
    e.bench_kernel(kind, n, 1)
    assert lib.smx_dbg_timeline(0, buf, 4096) == 0
    t = np.array(buf[:], dtype=np.int64)
    t0 = t[4095]
    if t0 == 0:
        print("kind", kind, "no timeline recorded")
        continue
    rel = lambda v: (v - t0) if v else -1  # noqa: E731
    P8 = t[:1024].reshape(128, 8)
    P = P8[:, :5]
    M = t[1024:1536].reshape(128, 4)[:, :3]
    E = t[2048:3072].reshape(256, 4)[:, :2]
    T = t[3072:3584].reshape(256, 2)
    nch = int((P[:, 0] > 0).sum())
    if nch > 64:
        nch = 64
    print(f"== kind {kind}: CTA cycles {t[4094] - t0}, chunks {nch}")
    print(" g   start  | own-A wait | LDS | refill | stage wait | stores | st-wait | -> MMA full-wait  issue")
    for g in range(nch):
        p = P8[g]
        m = M[g]
        print(f"{g:3d} {rel(p[0]):7d} | {p[1] - p[0]:6d} | {p[5] - p[1]:5d} | {p[2] - p[5]:5d} | {p[3] - p[2]:6d} |"
              f" {p[6] - p[3]:6d} | {p[4] - p[6]:5d} | mma@{rel(m[0]):7d} wait {m[1] - m[0]:6d} issue {m[2] - m[1]:5d}")
    tot = lambda a, b: int(sum(P[g][b] - P[g][a] for g in range(nch)))  # noqa: E731
    print("producer totals (sum over both groups): own-A wait", tot(0, 1), "gather", tot(1, 2), "stage wait",
          tot(2, 3), "stores", tot(3, 4))
    mw = int(sum(M[g][1] - M[g][0] for g in range(nch)))
    mi = int(sum(M[g][2] - M[g][1] for g in range(nch)))
    print("MMA: full-wait", mw, "issue", mi)
    nu = int((E[:, 0] > 0).sum())
    ew = int(sum(E[u][1] - E[u][0] for u in range(nu)))
    print("epilogue: units", nu, "acc_full wait", ew, " tiles",
          [(rel(T[i][0]), int(T[i][1] - T[i][0]) if T[i][1] else -1) for i in range(int((T[:, 0] > 0).sum()))][:12])
e.close()
