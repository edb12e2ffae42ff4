"""ctypes binding of the C ABI in include/smx.h (the executor boundary).

This is the same binding a Python maintainer of the reference would add; the
C++ host library links libsmx.so directly.  There is no fallback: if libsmx.so is missing or the
GPU is absent, construction fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SMX_LIB_PATH"]) if os.environ.get("SMX_LIB_PATH") else _PKG / "libsmx.so"  # override: profiling variants

SMX_OK, SMX_ECONFIG, SMX_EINTEGRITY, SMX_EDEVICE = 0, 1, 2, 3
MODEL_MLP = 0
MODEL_CNN = 1
GEMM_EXACT, GEMM_TC = 0, 1
HP_COLS = 4
MET_COLS = 2

# Every symbol include/smx.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "smx_open", "smx_close", "smx_param_count", "smx_dataset_digest", "smx_dataset_upload", "smx_dataset_read",
    "smx_host_alloc",
    "smx_host_free", "smx_hp_upload", "smx_slot_init",
    "smx_slot_load", "smx_slot_save", "smx_release_slot", "smx_ckpt_free", "smx_ckpt_peer_copy", "smx_slot_state", "smx_slot_read",
    "smx_slot_write", "smx_ckpt_read", "smx_ckpt_write", "smx_train", "smx_eval", "smx_losses", "smx_sync",
    "smx_set_timing", "smx_set_graphs", "smx_get_stats", "smx_reset_stats", "smx_bench_kernel", "smx_bench_peer_copy",
    "smx_test_gemm",
    "smx_last_error", "smx_version",
)


class SmxError(RuntimeError):
    code = SMX_EDEVICE


class SmxConfigError(SmxError):
    code = SMX_ECONFIG


class SmxIntegrityError(SmxError):
    code = SMX_EINTEGRITY


class SmxDeviceError(SmxError):
    code = SMX_EDEVICE


class ModelDesc(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("max_batch", ctypes.c_int32), ("n_train", ctypes.c_int32),
                ("n_val", ctypes.c_int32), ("max_steps", ctypes.c_int32), ("gemm_mode", ctypes.c_int32),
                ("seed", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("locksteps", ctypes.c_int64), ("stage_steps", ctypes.c_int64),
                ("forks", ctypes.c_int64), ("update_ms", ctypes.c_double), ("update_launches", ctypes.c_int64),
                ("gemm_ms", ctypes.c_double), ("gemm_launches", ctypes.c_int64), ("fork_ms", ctypes.c_double),
                ("fork_launches", ctypes.c_int64), ("lockstep_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load_library() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2006_11972_b200.build`")
        lib = ctypes.CDLL(str(LIB_PATH))
        P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        FP = ctypes.POINTER(ctypes.c_float)
        sig = {
            "smx_open": [ctypes.POINTER(ModelDesc), I, I, I, ctypes.POINTER(P)],
            "smx_close": [P],
            "smx_param_count": [P, ctypes.POINTER(I64), ctypes.POINTER(I64)],
            "smx_dataset_digest": [P, ctypes.POINTER(ctypes.c_uint64)],
            "smx_hp_upload": [P, I, I64, I64, FP],
            "smx_dataset_upload": [P, FP, P, FP, P],
            "smx_dataset_read": [P, FP, P, FP, P],
            "smx_host_alloc": [ctypes.c_uint64, ctypes.POINTER(P)],
            "smx_host_free": [P],
            "smx_slot_init": [P, I],
            "smx_slot_load": [P, I, I],
            "smx_slot_save": [P, I, I],
            "smx_ckpt_free": [P, I],
            "smx_release_slot": [P, I],
            "smx_ckpt_peer_copy": [P, I, P, I],
            "smx_slot_state": [P, I, ctypes.POINTER(I64), ctypes.POINTER(I64)],
            "smx_slot_read": [P, I, FP, FP],
            "smx_slot_write": [P, I, FP, FP, I64, I64],
            "smx_ckpt_read": [P, I, FP, FP, ctypes.POINTER(I64), ctypes.POINTER(I64)],
            "smx_ckpt_write": [P, I, FP, FP, I64, I64],
            "smx_train": [P, I, ctypes.POINTER(I), I],
            "smx_eval": [P, I, ctypes.POINTER(I), ctypes.POINTER(ctypes.c_double)],
            "smx_losses": [P, I, I64, I64, FP],
            "smx_sync": [P],
            "smx_set_timing": [P, I],
            "smx_set_graphs": [P, I],
            "smx_get_stats": [P, ctypes.POINTER(Stats)],
            "smx_reset_stats": [P],
            "smx_bench_kernel": [P, I, I, I, ctypes.POINTER(ctypes.c_double)],
            "smx_bench_peer_copy": [P, P, I, I, ctypes.POINTER(ctypes.c_double)],
            "smx_test_gemm": [P, I, I, I, I, I, FP, I, FP, I, FP],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.smx_last_error.restype = ctypes.c_char_p
        lib.smx_version.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _check(rc: int) -> None:
    if rc == SMX_OK:
        return
    msg = load_library().smx_last_error().decode()
    raise {SMX_ECONFIG: SmxConfigError, SMX_EINTEGRITY: SmxIntegrityError}.get(rc, SmxDeviceError)(msg)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


class Executor:
    """One GPU's stage executor: slot slab + checkpoint pool + grouped training kernels."""

    def __init__(self, n_slots: int, n_ckpts: int, device: int = 0, gemm_mode: int = GEMM_EXACT,
                 max_steps: int = 4096, n_train: int = 65536, n_val: int = 4096, max_batch: int = 256,
                 seed: int = 2006_11972, model: int = MODEL_MLP):
        self._lib = load_library()
        self.desc = ModelDesc(model, max_batch, n_train, n_val, max_steps, gemm_mode, seed)
        self._ctx = ctypes.c_void_p()
        _check(self._lib.smx_open(ctypes.byref(self.desc), device, n_slots, n_ckpts, ctypes.byref(self._ctx)))
        self.n_slots, self.n_ckpts, self.device = n_slots, n_ckpts, device
        self.n_train, self.n_val, self.max_batch = n_train, n_val, max_batch
        self.d_in = 32 * 32 * 4 if model == MODEL_CNN else 784
        p, pa = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.smx_param_count(self._ctx, ctypes.byref(p), ctypes.byref(pa)))
        self.p_algo, self.p_alloc = p.value, pa.value

    @property
    def handle(self):
        return self._ctx

    def close(self) -> None:
        if self._ctx:
            self._lib.smx_close(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- state store
    def dataset_digest(self) -> int:
        out = ctypes.c_uint64()
        _check(self._lib.smx_dataset_digest(self._ctx, ctypes.byref(out)))
        return out.value

    def dataset_upload(self, x: np.ndarray, y: np.ndarray, vx: np.ndarray, vy: np.ndarray) -> None:
        arrs = [np.ascontiguousarray(a) for a in (x, y, vx, vy)]
        assert arrs[0].dtype == np.float32 and arrs[1].dtype == np.int32
        _check(self._lib.smx_dataset_upload(self._ctx, _fp(arrs[0]), arrs[1].ctypes.data, _fp(arrs[2]),
                                            arrs[3].ctypes.data))

    def dataset_read(self):
        """(x, y, vx, vy): host copies of the context's dataset."""
        rows = self.n_train + self.max_batch
        x = np.empty((rows, self.d_in), np.float32)
        y = np.empty(rows, np.int32)
        vx = np.empty((self.n_val, self.d_in), np.float32)
        vy = np.empty(self.n_val, np.int32)
        _check(self._lib.smx_dataset_read(self._ctx, _fp(x), y.ctypes.data, _fp(vx), vy.ctypes.data))
        return x, y, vx, vy

    def hp_upload(self, slot: int, step0: int, rows: np.ndarray) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.float32).reshape(-1, HP_COLS)
        _check(self._lib.smx_hp_upload(self._ctx, slot, step0, rows.shape[0], _fp(rows)))

    def slot_init(self, slot: int) -> None:
        _check(self._lib.smx_slot_init(self._ctx, slot))

    def slot_load(self, slot: int, ckpt: int) -> None:
        _check(self._lib.smx_slot_load(self._ctx, slot, ckpt))

    def slot_save(self, slot: int, ckpt: int) -> None:
        _check(self._lib.smx_slot_save(self._ctx, slot, ckpt))

    def release_slot(self, slot: int) -> None:
        _check(self._lib.smx_release_slot(self._ctx, slot))

    def ckpt_free(self, ckpt: int) -> None:
        _check(self._lib.smx_ckpt_free(self._ctx, ckpt))

    def ckpt_peer_copy(self, dst_ckpt: int, src: "Executor", src_ckpt: int) -> None:
        _check(self._lib.smx_ckpt_peer_copy(self._ctx, dst_ckpt, src._ctx, src_ckpt))

    def slot_state(self, slot: int):
        s, o = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.smx_slot_state(self._ctx, slot, ctypes.byref(s), ctypes.byref(o)))
        return s.value, o.value

    def slot_read(self, slot: int):
        w = np.empty(self.p_alloc, np.float32)
        m = np.empty(self.p_alloc, np.float32)
        _check(self._lib.smx_slot_read(self._ctx, slot, _fp(w), _fp(m)))
        return w, m

    def slot_write(self, slot: int, w: np.ndarray, m: np.ndarray, step: int, offset: int) -> None:
        w = np.ascontiguousarray(w, np.float32)
        m = np.ascontiguousarray(m, np.float32)
        assert w.size == self.p_alloc and m.size == self.p_alloc
        _check(self._lib.smx_slot_write(self._ctx, slot, _fp(w), _fp(m), step, offset))

    def ckpt_read(self, ckpt: int):
        w = np.empty(self.p_alloc, np.float32)
        m = np.empty(self.p_alloc, np.float32)
        s, o = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.smx_ckpt_read(self._ctx, ckpt, _fp(w), _fp(m), ctypes.byref(s), ctypes.byref(o)))
        return w, m, s.value, o.value

    def ckpt_write(self, ckpt: int, w, m, step: int, offset: int) -> None:
        w = np.ascontiguousarray(w, np.float32)
        m = np.ascontiguousarray(m, np.float32)
        _check(self._lib.smx_ckpt_write(self._ctx, ckpt, _fp(w), _fp(m), step, offset))

    # -- execution
    def train(self, slots, n_steps: int) -> None:
        s = np.ascontiguousarray(slots, dtype=np.int32)
        _check(self._lib.smx_train(self._ctx, s.size, _ip(s), n_steps))

    def eval(self, slots) -> np.ndarray:
        s = np.ascontiguousarray(slots, dtype=np.int32)
        out = np.empty((s.size, MET_COLS), np.float64)
        _check(self._lib.smx_eval(self._ctx, s.size, _ip(s), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def losses(self, slot: int, step0: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        _check(self._lib.smx_losses(self._ctx, slot, step0, n, _fp(out)))
        return out

    def sync(self) -> None:
        _check(self._lib.smx_sync(self._ctx))

    # -- measurement
    def set_timing(self, on: bool) -> None:
        _check(self._lib.smx_set_timing(self._ctx, int(on)))

    def set_graphs(self, on: bool) -> None:
        _check(self._lib.smx_set_graphs(self._ctx, int(on)))

    def stats(self) -> dict:
        st = Stats()
        _check(self._lib.smx_get_stats(self._ctx, ctypes.byref(st)))
        return st.as_dict()

    def reset_stats(self) -> None:
        _check(self._lib.smx_reset_stats(self._ctx))

    def test_gemm(self, A: np.ndarray, B: np.ndarray, a_mn: bool, b_mn: bool, M: int | None = None,
                  N: int | None = None) -> np.ndarray:
        """C = A_logical @ B_logical^T where A_logical is A (a_mn False, [M,K]) or A.T (a_mn True,
        A stored [K,>=M], leading dimension = A.shape[1]); likewise B ([N,K] or stored [K,>=N])."""
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        K = A.shape[0] if a_mn else A.shape[1]
        M = M if M is not None else (A.shape[1] if a_mn else A.shape[0])
        N = N if N is not None else (B.shape[1] if b_mn else B.shape[0])
        C = np.empty((M, N), np.float32)
        _check(self._lib.smx_test_gemm(self._ctx, int(a_mn), int(b_mn), M, N, K, _fp(A), A.shape[1], _fp(B),
                                       B.shape[1], _fp(C)))
        return C

    def bench_peer_copy(self, src: "Executor", n: int, reps: int) -> float:
        """Mean ms per checkpoint entry copied from `src` (K7, n entries per launch)."""
        out = ctypes.c_double()
        _check(self._lib.smx_bench_peer_copy(self._ctx, src._ctx, n, reps, ctypes.byref(out)))
        return out.value

    def bench_kernel(self, kind: int, n: int, reps: int) -> float:
        out = ctypes.c_double()
        _check(self._lib.smx_bench_kernel(self._ctx, kind, n, reps, ctypes.byref(out)))
        return out.value


def version() -> str:
    return load_library().smx_version().decode()
