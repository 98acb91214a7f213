"""ctypes binding of librtgpu.so (include/rtgpu.h, include/rtgpu_gen.h).

The package has no pure-Python analysis path: if the native library is
missing, or no CUDA device is visible, every analysis call raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RTGPU_LIB") or os.path.join(HERE, "librtgpu.so")

_p64 = ctypes.POINTER(ctypes.c_int64)
_p32 = ctypes.POINTER(ctypes.c_int32)
_lib = None


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run (library not built or no device)."""


class GenParamsC(ctypes.Structure):
    _fields_ = [("n_tasks", ctypes.c_int32), ("n_subtasks", ctypes.c_int32),
                ("cpu_lo", ctypes.c_int64), ("cpu_hi", ctypes.c_int64),
                ("gpu_lo", ctypes.c_int64), ("gpu_hi", ctypes.c_int64),
                ("mem_lo", ctypes.c_int64), ("mem_hi", ctypes.c_int64),
                ("util_num", ctypes.c_int64), ("util_den", ctypes.c_int64),
                ("mem_model", ctypes.c_int32), ("physical_sms", ctypes.c_int32),
                ("eps_num", ctypes.c_int64), ("eps_den", ctypes.c_int64),
                ("lofrac_num", ctypes.c_int64), ("lofrac_den", ctypes.c_int64),
                ("seg_int32", ctypes.c_int32), ("pad", ctypes.c_int32)]


EXPORTS = ("rtgpu_abi_version", "rtgpu_last_error", "rtgpu_device_info", "rtgpu_analyze_host",
           "rtgpu_analyze_device", "rtgpu_last_launch_count", "rtgpu_set_stage_timing",
           "rtgpu_last_stage_ms", "rtgpu_gen_blob_words", "rtgpu_generate", "rtgpu_sha512")


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineUnavailable(
            f"{LIB_PATH} is not built; run `python -m paper_2101_10463_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.rtgpu_abi_version.restype = ctypes.c_int
    L.rtgpu_last_error.restype = ctypes.c_char_p
    L.rtgpu_device_info.argtypes = [ctypes.POINTER(ctypes.c_int)] * 4
    L.rtgpu_analyze_host.argtypes = [_p64, _p64, _p64, ctypes.c_int64, ctypes.c_int, ctypes.c_uint,
                                     ctypes.c_int64, _p32, _p64, _p32, _p64, _p64, _p64]
    L.rtgpu_analyze_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_uint, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]
    L.rtgpu_last_launch_count.restype = ctypes.c_int64
    L.rtgpu_set_stage_timing.argtypes = [ctypes.c_int]
    L.rtgpu_last_stage_ms.argtypes = [ctypes.POINTER(ctypes.c_float), _p64]
    L.rtgpu_gen_blob_words.argtypes = [ctypes.POINTER(GenParamsC)]
    L.rtgpu_gen_blob_words.restype = ctypes.c_int64
    L.rtgpu_generate.argtypes = [ctypes.POINTER(GenParamsC), ctypes.c_int64, _p64,
                                 ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, _p64, _p64, _p64]
    L.rtgpu_sha512.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p]
    if L.rtgpu_abi_version() != 1:
        raise EngineUnavailable("librtgpu.so ABI version mismatch")
    _lib = L
    return L


def last_error() -> str:
    return lib().rtgpu_last_error().decode(errors="replace")


def device_info() -> dict:
    n, sm, ma, mi = (ctypes.c_int(0) for _ in range(4))
    rc = lib().rtgpu_device_info(ctypes.byref(n), ctypes.byref(sm), ctypes.byref(ma),
                                 ctypes.byref(mi))
    return {"ok": rc == 0, "n_devices": n.value, "sm_count": sm.value, "cc": (ma.value, mi.value)}


def require_device() -> None:
    info = device_info()
    if not info["ok"] or info["n_devices"] < 1:
        raise EngineUnavailable("no CUDA device visible: the RTGPU engine runs only on the GPU "
                                f"({last_error()})")


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def analyze_host(blobs: np.ndarray, set_off: np.ndarray, task_base: np.ndarray, method: int,
                 flags: int, budget: int, detail: bool):
    """rtgpu_analyze_host over numpy buffers; returns dict of result arrays."""
    require_device()
    S = len(set_off) - 1
    T = int(task_base[-1])
    out = dict(status=np.zeros(S, np.int32), evals=np.zeros(S, np.int64),
               vsm=np.zeros(T, np.int32), e2e_num=np.zeros(T, np.int64),
               den=np.ones(T, np.int64), detail=np.zeros(len(blobs), np.int64) if detail else None)
    blobs = np.ascontiguousarray(blobs, np.int64)
    set_off = np.ascontiguousarray(set_off, np.int64)
    task_base = np.ascontiguousarray(task_base, np.int64)
    rc = lib().rtgpu_analyze_host(
        _ptr(blobs, ctypes.c_int64), _ptr(set_off, ctypes.c_int64),
        _ptr(task_base, ctypes.c_int64), S, method, flags, budget,
        _ptr(out["status"], ctypes.c_int32), _ptr(out["evals"], ctypes.c_int64),
        _ptr(out["vsm"], ctypes.c_int32), _ptr(out["e2e_num"], ctypes.c_int64),
        _ptr(out["den"], ctypes.c_int64), _ptr(out["detail"], ctypes.c_int64))
    if rc != 0:
        raise RuntimeError(f"rtgpu_analyze_host failed ({rc}): {last_error()}")
    return out


def analyze_device(d_blobs, d_set_off, d_task_base, n_sets: int, dims: Sequence[int], method: int,
                   flags: int, budget: int, d_status, d_evals, d_vsm, d_e2e, d_den,
                   d_detail=None, stream: Optional[int] = None) -> None:
    """rtgpu_analyze_device on device pointers (ints); asynchronous on stream."""
    rc = lib().rtgpu_analyze_device(
        d_blobs, d_set_off, d_task_base, n_sets, int(dims[0]), int(dims[1]), int(dims[2]),
        method, flags, budget, d_status, d_evals, d_vsm, d_e2e, d_den, d_detail, stream)
    if rc != 0:
        raise RuntimeError(f"rtgpu_analyze_device failed ({rc}): {last_error()}")


def last_launch_count() -> int:
    return int(lib().rtgpu_last_launch_count())


def set_stage_timing(enable: bool) -> None:
    lib().rtgpu_set_stage_timing(1 if enable else 0)


def last_stage_ms():
    """(ms per stage kernel, sets per stage) of the last call, or None."""
    ms = (ctypes.c_float * 3)()
    sets = np.zeros(3, np.int64)
    if lib().rtgpu_last_stage_ms(ms, _ptr(sets, ctypes.c_int64)) != 0:
        return None
    return [float(x) for x in ms], [int(x) for x in sets]


def gen_params_c(n_tasks, n_subtasks, cpu_range, gpu_range, mem_range, util, mem_model_code,
                 physical_sms, eps, lo_frac, compact: bool = False, rec32: bool = False) -> GenParamsC:
    """compact: int32 segment areas (header word 7 = 1); rec32: int32 task
    records too (header word 7 = 2, 15% fewer bytes for 8 x 5 sets; the
    kernels and the oracle read both); neither is for detail runs."""
    from fractions import Fraction
    u, e, lf = Fraction(util), Fraction(eps), Fraction(lo_frac)
    for name, f in (("utilization", u), ("launch_overhead_frac", e), ("lo_frac", lf)):
        if not (-2**63 < f.numerator < 2**63 and 0 < f.denominator < 2**63):
            raise ValueError(f"{name} {f} does not fit the generator's int64 fraction")
    return GenParamsC(n_tasks, n_subtasks, cpu_range[0], cpu_range[1], gpu_range[0], gpu_range[1],
                      mem_range[0], mem_range[1], u.numerator, u.denominator, mem_model_code,
                      physical_sms, e.numerator, e.denominator, lf.numerator, lf.denominator,
                      2 if rec32 else (1 if compact else 0), 0)


def generate(params: GenParamsC, seeds, n_threads: int = 0):
    """Bulk generation; seeds: sequence of ints or of strs (not mixed)."""
    L = lib()
    S = len(seeds)
    words = L.rtgpu_gen_blob_words(ctypes.byref(params))
    blobs = np.zeros(S * words, np.int64)
    set_off = np.zeros(S + 1, np.int64)
    task_base = np.zeros(S + 1, np.int64)
    if n_threads <= 0:
        n_threads = min(32, os.cpu_count() or 1)
    int_seeds = None
    str_arr = None
    if S and isinstance(seeds[0], str):
        str_arr = (ctypes.c_char_p * S)(*[s.encode() for s in seeds])
    else:
        int_seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
    rc = L.rtgpu_generate(ctypes.byref(params), S, _ptr(int_seeds, ctypes.c_int64),
                          str_arr, n_threads, _ptr(blobs, ctypes.c_int64),
                          _ptr(set_off, ctypes.c_int64), _ptr(task_base, ctypes.c_int64))
    if rc == -2:
        raise ValueError("a generated deadline exceeds int64 (utilization too small)")
    if rc != 0:
        raise ValueError("invalid generator parameters")
    return blobs, set_off, task_base
