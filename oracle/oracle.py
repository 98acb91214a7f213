"""TEST INFRASTRUCTURE ONLY: ctypes binding of the C oracle (liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module -- as the checker, never as the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    deps = [os.path.join(HERE, "rtgpu_oracle.c"), os.path.join(os.path.dirname(HERE), "include", "rtgpu.h")]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        p64 = ctypes.POINTER(ctypes.c_int64)
        p32 = ctypes.POINTER(ctypes.c_int32)
        _lib.oracle_analyze_batch.argtypes = [
            p64, p64, p64, ctypes.c_int64, ctypes.c_int, ctypes.c_uint, ctypes.c_int64,
            ctypes.c_int, p32, p64, p32, p64, p64, p64]
        _lib.oracle_analyze_batch.restype = ctypes.c_int
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def analyze_batch(blobs, set_off, task_base, method: int = 0, flags: int = 2,
                  budget: int = 0, threads: int = 1, detail: bool = True):
    """Run the oracle on a packed batch; returns a dict of result arrays."""
    S = len(set_off) - 1
    T = int(task_base[-1])
    out = dict(status=np.zeros(S, np.int32), evals=np.zeros(S, np.int64),
               vsm=np.zeros(T, np.int32), e2e_num=np.zeros(T, np.int64),
               den=np.ones(T, np.int64),
               detail=np.zeros(len(blobs), np.int64) if detail else None)
    blobs = np.ascontiguousarray(blobs, np.int64)
    set_off = np.ascontiguousarray(set_off, np.int64)
    task_base = np.ascontiguousarray(task_base, np.int64)
    lib().oracle_analyze_batch(
        _p(blobs, ctypes.c_int64), _p(set_off, ctypes.c_int64), _p(task_base, ctypes.c_int64),
        S, method, flags, budget, threads, _p(out["status"], ctypes.c_int32),
        _p(out["evals"], ctypes.c_int64), _p(out["vsm"], ctypes.c_int32),
        _p(out["e2e_num"], ctypes.c_int64), _p(out["den"], ctypes.c_int64),
        _p(out["detail"], ctypes.c_int64))
    return out
