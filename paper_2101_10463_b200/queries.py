"""Batched point queries of the analysis building blocks on the GPU
(include/rtgpu.h rtgpu_query_host): suspension-core workloads and response
times, and the RTGPU per-segment recurrences with explicit GPU bounds."""
from __future__ import annotations

import ctypes
from fractions import Fraction
from typing import Optional, Sequence

import numpy as np

from . import _native
from .pack import build_blob, lcm_denominators

Q_WORKLOAD, Q_MAX_WORKLOAD, Q_SEGMENT_RESPONSE, Q_TASK_RESPONSE = 0, 1, 2, 3
Q_MEM_RESPONSE, Q_CPU_RESPONSE, Q_END_TO_END, Q_MEM_WORKLOAD, Q_CPU_WORKLOAD, Q_R2 = 4, 5, 6, 7, 8, 9
ST_OK, ST_UNDECIDED, ST_RANGE, ST_INVALID, ST_GAP_ERROR = 1, 2, 3, 4, 5


class QueryC(ctypes.Structure):
    _fields_ = [("set", ctypes.c_int64), ("kind", ctypes.c_int32), ("task", ctypes.c_int32),
                ("index", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("horizon", ctypes.c_int64), ("blocking", ctypes.c_int64)]


class InfeasibleGapError(ValueError):
    """A minimum inter-arrival gap came out negative (reference analysis.py:46)."""


def run(sets: Sequence[list], queries: Sequence[tuple]) -> list:
    """sets: blobs (int lists); queries: (set, kind, task, index, horizon_ticks,
    blocking_ticks).  Returns (status, num, den) per query."""
    L = _native.lib()
    _native.require_device()
    words, offs = [], [0]
    for b in sets:
        words += b
        offs.append(len(words))
    blobs = np.asarray(words, dtype=np.int64)
    set_off = np.asarray(offs, dtype=np.int64)
    qa = (QueryC * len(queries))(*[QueryC(s, k, t, i, 0, h, b) for s, k, t, i, h, b in queries])
    n = len(queries)
    st = np.zeros(n, np.int32)
    num = np.zeros(n, np.int64)
    den = np.ones(n, np.int64)
    P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
    L.rtgpu_query_host.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                   ctypes.c_int64, ctypes.POINTER(QueryC), ctypes.c_int64,
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int64)]
    rc = L.rtgpu_query_host(P(blobs, ctypes.c_int64), P(set_off, ctypes.c_int64), len(sets), qa, n,
                            P(st, ctypes.c_int32), P(num, ctypes.c_int64), P(den, ctypes.c_int64))
    if rc != 0:
        raise RuntimeError(f"rtgpu_query_host failed ({rc}): {_native.last_error()}")
    return [(int(st[i]), int(num[i]), int(den[i])) for i in range(n)]


def value(status: int, num: int, den: int, scale: int) -> Optional[Fraction]:
    if status == ST_GAP_ERROR:
        raise InfeasibleGapError("negative inter-arrival gap")
    if status == ST_RANGE:
        raise ArithmeticError("values exceed the engine's exact range")
    if status == ST_UNDECIDED:
        raise TimeoutError("fixed-point iteration cap reached")
    if status != ST_OK:
        raise ValueError("query rejected by the engine (invalid input)")
    return None if num < 0 else Fraction(num, den * scale)


def ticks(x, scale: int) -> int:
    v = Fraction(x) * scale
    assert v.denominator == 1
    return int(v)


__all__ = ["run", "value", "ticks", "lcm_denominators", "build_blob", "InfeasibleGapError"]
