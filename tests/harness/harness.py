"""TEST HARNESS ONLY: ctypes binding of engine_host.cpp (engine core on CPU)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SRC = os.path.join(HERE, "engine_host.cpp")
CORE = os.path.join(ROOT, "paper_2101_10463_b200", "csrc", "engine_core.cuh")
LAT = os.path.join(ROOT, "paper_2101_10463_b200", "csrc", "lattice.cuh")
LIB = os.path.join(HERE, "libenginehost.so")
_lib = None


def build():
    newest = max(os.path.getmtime(SRC), os.path.getmtime(CORE), os.path.getmtime(LAT))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", LIB, SRC],
                       check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
        p64 = ctypes.POINTER(ctypes.c_int64)
        p32 = ctypes.POINTER(ctypes.c_int32)
        _lib.host_analyze_batch.argtypes = [p64, p64, p64, ctypes.c_int64, ctypes.c_int, ctypes.c_uint,
                                            ctypes.c_int64, ctypes.c_int, p32, p64, p32, p64,
                                            p64, p64, p32]
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def analyze_batch(blobs, set_off, task_base, flags=2, budget=0, first_stage=0, detail=True, method=0):
    S = len(set_off) - 1
    T = int(task_base[-1])
    out = dict(status=np.zeros(S, np.int32), evals=np.zeros(S, np.int64),
               vsm=np.zeros(T, np.int32), e2e_num=np.zeros(T, np.int64),
               den=np.ones(T, np.int64),
               detail=np.zeros(len(blobs), np.int64) if detail else None,
               stage=np.zeros(S, np.int32))
    blobs = np.ascontiguousarray(blobs, np.int64)
    lib().host_analyze_batch(
        _p(blobs, ctypes.c_int64), _p(np.ascontiguousarray(set_off, np.int64), ctypes.c_int64),
        _p(np.ascontiguousarray(task_base, np.int64), ctypes.c_int64), S, method, flags, budget,
        first_stage, _p(out["status"], ctypes.c_int32), _p(out["evals"], ctypes.c_int64),
        _p(out["vsm"], ctypes.c_int32), _p(out["e2e_num"], ctypes.c_int64),
        _p(out["den"], ctypes.c_int64), _p(out["detail"], ctypes.c_int64),
        _p(out["stage"], ctypes.c_int32))
    return out


def query(sets, queries):
    """host_query over blobs (int lists) and (set, kind, task, index, horizon,
    blocking) tuples; returns (status, num, den) per query."""
    from paper_2101_10463_b200.queries import QueryC
    L = lib()
    words, offs = [], [0]
    for b in sets:
        words += b
        offs.append(len(words))
    blobs = np.asarray(words, dtype=np.int64)
    set_off = np.asarray(offs, dtype=np.int64)
    n = len(queries)
    qa = (QueryC * n)(*[QueryC(s, k, t, i, 0, h, b) for s, k, t, i, h, b in queries])
    st = np.zeros(n, np.int32)
    num = np.zeros(n, np.int64)
    den = np.ones(n, np.int64)
    L.host_query.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                             ctypes.c_int64, ctypes.POINTER(QueryC), ctypes.c_int64,
                             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                             ctypes.POINTER(ctypes.c_int64)]
    L.host_query(_p(blobs, ctypes.c_int64), _p(set_off, ctypes.c_int64), len(sets), qa, n,
                 _p(st, ctypes.c_int32), _p(num, ctypes.c_int64), _p(den, ctypes.c_int64))
    return [(int(st[i]), int(num[i]), int(den[i])) for i in range(n)]


def lattice_batch(blobs, set_off, task_base, bounds=False):
    """The lattice path alone (status 99 = handed on to the general stages)."""
    L = lib()
    p64 = ctypes.POINTER(ctypes.c_int64)
    p32 = ctypes.POINTER(ctypes.c_int32)
    L.host_lattice_batch.argtypes = [p64, p64, p64, ctypes.c_int64, ctypes.c_int, p32, p64, p32, p64, p64]
    S = len(set_off) - 1
    T = int(task_base[-1])
    out = dict(status=np.zeros(S, np.int32), evals=np.zeros(S, np.int64), vsm=np.zeros(T, np.int32),
               e2e_num=np.zeros(T, np.int64), den=np.ones(T, np.int64))
    blobs = np.ascontiguousarray(blobs, np.int64)
    L.host_lattice_batch(_p(blobs, ctypes.c_int64), _p(np.ascontiguousarray(set_off, np.int64), ctypes.c_int64),
                         _p(np.ascontiguousarray(task_base, np.int64), ctypes.c_int64), S, int(bounds),
                         _p(out["status"], ctypes.c_int32), _p(out["evals"], ctypes.c_int64),
                         _p(out["vsm"], ctypes.c_int32), _p(out["e2e_num"], ctypes.c_int64),
                         _p(out["den"], ctypes.c_int64))
    return out
