"""ctypes loader for oracle/fold.c — TEST INFRASTRUCTURE ONLY (see __init__.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "fold.c")
LIB = os.path.join(_HERE, "liboracle_fold.so")

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile fold.c with gcc (building the checker is not using it)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_fold_f32.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                         ctypes.c_size_t, ctypes.c_float, ctypes.c_void_p]
        _lib.oracle_fold_bf16.argtypes = _lib.oracle_fold_f32.argtypes
        _lib.oracle_threads.restype = ctypes.c_int
        _lib.oracle_set_threads.argtypes = [ctypes.c_int]
    return _lib


def threads() -> int:
    return lib().oracle_threads()


def set_threads(t: int) -> None:
    """OpenMP threads of the folds (results are independent of it)."""
    lib().oracle_set_threads(int(t))


def fold_ascending(xs, scale: float = 1.0) -> np.ndarray:
    """C twin of hfr_oracle.fold_ascending (same contract, same bits)."""
    xs = [np.ascontiguousarray(x) for x in xs]
    if xs[0].dtype not in (np.float32, np.uint16) or (xs[0].dtype.metadata or {}).get("hfr"):
        raise TypeError("fold.c folds fp32 and bf16 only (use hfr_oracle for fp16 / FP8)")
    n = len(xs)
    count = xs[0].shape[0]
    ptrs = (ctypes.c_void_p * n)(*[x.ctypes.data for x in xs])
    out = np.empty(count, dtype=xs[0].dtype)
    fn = lib().oracle_fold_f32 if xs[0].dtype == np.float32 else lib().oracle_fold_bf16
    fn(ptrs, n, count, ctypes.c_float(scale), out.ctypes.data)
    return out
