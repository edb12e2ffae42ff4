"""Back-to-back tcgen05.mma kind::tf32 rate (see mma_rate.cu)."""
import ctypes
import sys
from pathlib import Path

lib = ctypes.CDLL(str(Path(__file__).with_name("mma_rate.so")))
iters = 2000
for ts in ((1, 0) if "ss" in sys.argv[1:] else (1,)):
    for n in (64, 128):
        cyc = (ctypes.c_longlong * 148)()
        ms = ctypes.c_float()
        rc = lib.run(ts, n, iters, cyc, ctypes.byref(ms))
        per = sum(cyc) / 148 / (iters * 12)
        flops = 2 * 128 * n * 8 * 12 * iters * 148
        print(f"{'TS' if ts else 'SS'} N={n:3d}: {per:6.1f} cycles/MMA, {flops / (ms.value * 1e-3) / 1e12:7.1f} TFLOP/s tf32 (rc {rc})")

if "m64" in sys.argv[1:]:
    for ts in (2, 3):
        for n in (128, 256):
            cyc = (ctypes.c_longlong * 148)()
            ms = ctypes.c_float()
            rc = lib.run(ts, n, iters, cyc, ctypes.byref(ms))
            per = sum(cyc) / 148 / (iters * 12)
            flops = 2 * 64 * n * 8 * 12 * iters * 148
            print(f"{'TS' if ts == 2 else 'SS'} M=64 N={n:3d}: {per:6.1f} cycles/MMA, "
                  f"{flops / (ms.value * 1e-3) / 1e12:7.1f} TFLOP/s tf32 (rc {rc})")

chunks = 4000
for n in (64, 128):
    for mode in (0, 5, 7):
        cyc = (ctypes.c_longlong * 148)()
        rc = lib.run_proto(n, mode, chunks, cyc)
        print(f"protocol N={n} mode={mode}: {sum(cyc) / 148 / chunks:7.1f} cycles/chunk of 12 MMAs (rc {rc})")
