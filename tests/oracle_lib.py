"""TEST INFRASTRUCTURE: ctypes loaders for the CPU oracle (oracle/liboracle.so) and for the
compiled reference (oracle/_ref/libstagemerge_ref.so).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg import this module."""
from __future__ import annotations

import ctypes
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libstagemerge_ref.so"

N_TRAIN, MAX_BATCH, N_VAL, D0 = 65536, 256, 4096, 784
SEED = 2006_11972

_FP = ctypes.POINTER(ctypes.c_float)
_I64P = ctypes.POINTER(ctypes.c_int64)


@lru_cache(None)
def oracle() -> ctypes.CDLL:
    lib = ctypes.CDLL(str(ORACLE_SO))
    lib.orc_exp.argtypes = [ctypes.c_float]
    lib.orc_exp.restype = ctypes.c_float
    lib.orc_log.argtypes = [ctypes.c_float]
    lib.orc_log.restype = ctypes.c_float
    lib.orc_layout.argtypes = [_I64P, _I64P, _I64P]
    lib.orc_gen_dataset.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _FP,
                                    ctypes.c_void_p, _FP, ctypes.c_void_p]
    lib.orc_fnv.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64]
    lib.orc_fnv.restype = ctypes.c_uint64
    lib.orc_init.argtypes = [ctypes.c_uint64, _FP, _FP]
    lib.orc_train.argtypes = [_FP, _FP, _I64P, _I64P, _FP, ctypes.c_int64, ctypes.c_int, _FP, ctypes.c_void_p,
                              ctypes.c_int, _FP]
    lib.orc_train.restype = ctypes.c_int
    PP = ctypes.POINTER(_FP)
    lib.orc_train_many.argtypes = [ctypes.c_int, PP, PP, _I64P, _I64P, PP, ctypes.c_int64, ctypes.c_int, _FP,
                                   ctypes.c_void_p, ctypes.c_int, PP, ctypes.c_int]
    lib.orc_train_many.restype = ctypes.c_int
    lib.orc_eval.argtypes = [_FP, _FP, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.orc_cnn_layout.argtypes = [_I64P, _I64P, _I64P]
    lib.orc_cnn_gen_dataset.argtypes = lib.orc_gen_dataset.argtypes
    lib.orc_cnn_init.argtypes = lib.orc_init.argtypes
    lib.orc_cnn_train.argtypes = lib.orc_train.argtypes
    lib.orc_cnn_train.restype = ctypes.c_int
    lib.orc_cnn_train_many.argtypes = lib.orc_train_many.argtypes
    lib.orc_cnn_train_many.restype = ctypes.c_int
    lib.orc_cnn_eval.argtypes = lib.orc_eval.argtypes
    lib.orc_cnn_conv_fwd.argtypes = [ctypes.c_int, _FP, ctypes.c_int, _FP, _FP]
    lib.orc_cnn_conv_wgrad.argtypes = [ctypes.c_int, _FP, _FP, ctypes.c_int, _FP]
    lib.orc_cnn_conv_dgrad.argtypes = [ctypes.c_int, _FP, _FP, _FP, ctypes.c_int, _FP]
    return lib


def fp(a):
    return a.ctypes.data_as(_FP)


def layout():
    pa, pl = ctypes.c_int64(), ctypes.c_int64()
    off = (ctypes.c_int64 * 7)()
    oracle().orc_layout(ctypes.byref(pa), ctypes.byref(pl), off)
    return pa.value, pl.value, list(off)


class Dataset:
    def __init__(self, seed=SEED, n_train=N_TRAIN, max_batch=MAX_BATCH, n_val=N_VAL):
        self.n_train = n_train
        self.x = np.empty((n_train + max_batch, D0), np.float32)
        self.y = np.empty(n_train + max_batch, np.int32)
        self.vx = np.empty((n_val, D0), np.float32)
        self.vy = np.empty(n_val, np.int32)
        oracle().orc_gen_dataset(seed, n_train, max_batch, n_val, fp(self.x), self.y.ctypes.data, fp(self.vx),
                                 self.vy.ctypes.data)

    def digest(self) -> int:
        h = 0xCBF29CE484222325
        for a in (self.x, self.y, self.vx, self.vy):
            h = oracle().orc_fnv(a.ctypes.data, a.nbytes, h)
        return h


@lru_cache(None)
def dataset() -> Dataset:
    return Dataset()


class Slot:
    """One oracle training replica (w, m, step, offset, loss history)."""

    def __init__(self, seed=SEED, max_steps=4096):
        _, p_alloc, _ = layout()
        self.w = np.empty(p_alloc, np.float32)
        self.m = np.empty(p_alloc, np.float32)
        oracle().orc_init(seed, fp(self.w), fp(self.m))
        self.step = ctypes.c_int64(0)
        self.offset = ctypes.c_int64(0)
        self.loss = np.zeros(max_steps, np.float32)

    def copy(self) -> "Slot":
        s = Slot.__new__(Slot)
        s.w, s.m, s.loss = self.w.copy(), self.m.copy(), self.loss.copy()
        s.step, s.offset = ctypes.c_int64(self.step.value), ctypes.c_int64(self.offset.value)
        return s

    def train(self, hp: np.ndarray, n_steps: int, ds: Dataset | None = None) -> None:
        ds = ds or dataset()
        hp = np.ascontiguousarray(hp, np.float32)
        rc = oracle().orc_train(fp(self.w), fp(self.m), ctypes.byref(self.step), ctypes.byref(self.offset), fp(hp),
                                hp.shape[0], n_steps, fp(ds.x), ds.y.ctypes.data, ds.n_train, fp(self.loss))
        assert rc == 0, "hp table too short"

    def eval(self, ds: Dataset | None = None):
        ds = ds or dataset()
        out = (ctypes.c_double * 2)()
        oracle().orc_eval(fp(self.w), fp(ds.vx), ds.vy.ctypes.data, ds.vx.shape[0], out)
        return out[0], out[1]


@lru_cache(None)
def ref() -> ctypes.CDLL:
    lib = ctypes.CDLL(str(REF_SO))
    lib.ref_call.argtypes = [ctypes.c_char_p]
    lib.ref_call.restype = ctypes.c_char_p
    return lib


def ref_call(cmd: dict) -> dict:
    return json.loads(ref().ref_call(json.dumps(cmd).encode()))


# ---- CNN model (oracle/cnn.c) ---------------------------------------------
CNN_SAMPLE = 32 * 32 * 4


def cnn_layout():
    pa, pl = ctypes.c_int64(), ctypes.c_int64()
    off = (ctypes.c_int64 * 9)()
    oracle().orc_cnn_layout(ctypes.byref(pa), ctypes.byref(pl), off)
    return pa.value, pl.value, list(off)


class CnnDataset:
    def __init__(self, seed=SEED, n_train=N_TRAIN, max_batch=MAX_BATCH, n_val=N_VAL):
        self.n_train = n_train
        self.x = np.empty((n_train + max_batch, CNN_SAMPLE), np.float32)
        self.y = np.empty(n_train + max_batch, np.int32)
        self.vx = np.empty((n_val, CNN_SAMPLE), np.float32)
        self.vy = np.empty(n_val, np.int32)
        oracle().orc_cnn_gen_dataset(seed, n_train, max_batch, n_val, fp(self.x), self.y.ctypes.data, fp(self.vx),
                                     self.vy.ctypes.data)

    def digest(self) -> int:
        h = 0xCBF29CE484222325
        for a in (self.x, self.y, self.vx, self.vy):
            h = oracle().orc_fnv(a.ctypes.data, a.nbytes, h)
        return h


@lru_cache(None)
def cnn_dataset(n_train=N_TRAIN, n_val=N_VAL, max_batch=MAX_BATCH) -> CnnDataset:
    return CnnDataset(n_train=n_train, n_val=n_val, max_batch=max_batch)


class CnnSlot:
    """One oracle replica of the CNN (w, m, step, offset, loss history)."""

    def __init__(self, ds: CnnDataset, seed=SEED, max_steps=4096):
        _, p_alloc, _ = cnn_layout()
        self.ds = ds
        self.w = np.empty(p_alloc, np.float32)
        self.m = np.empty(p_alloc, np.float32)
        oracle().orc_cnn_init(seed, fp(self.w), fp(self.m))
        self.step = ctypes.c_int64(0)
        self.offset = ctypes.c_int64(0)
        self.loss = np.zeros(max_steps, np.float32)

    def train(self, hp: np.ndarray, n_steps: int) -> None:
        ds = self.ds
        hp = np.ascontiguousarray(hp, np.float32)
        rc = oracle().orc_cnn_train(fp(self.w), fp(self.m), ctypes.byref(self.step), ctypes.byref(self.offset),
                                    fp(hp), hp.shape[0], n_steps, fp(ds.x), ds.y.ctypes.data, ds.n_train,
                                    fp(self.loss))
        assert rc == 0, "hp table too short"

    def eval(self):
        ds = self.ds
        out = (ctypes.c_double * 2)()
        oracle().orc_cnn_eval(fp(self.w), fp(ds.vx), ds.vy.ctypes.data, ds.vx.shape[0], out)
        return out[0], out[1]
