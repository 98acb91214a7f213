"""Bulk task sets as integer arrays: the packing path for callers that hold
millions of sets in numpy rather than as ``TaskSet`` objects.

``analyze_batch`` (analysis.py) takes ``TaskSet`` objects, and reading their
attributes bounds it at tens of thousands of sets per second however the
packing is written (csrc/packer.cpp reads ~420 attributes per 8 x 5 set).
``TaskArrays`` holds S sets of one shape -- n tasks of m CPU segments --
as integer arrays in one tick unit, and ``pack_arrays`` lays them out in the
engine's blob format (include/rtgpu.h) in one native pass per set (threads
over sets, csrc/packer.cpp; ``pack_arrays_np`` restates it in numpy): the
blobs are word for word what ``pack_tasksets`` makes of the same sets
written as TaskSets (tests/test_arrays.py), compact (int32 segment areas)
when every value fits, so verdict runs take the fast kernel.
``analyze_arrays`` runs them and returns arrays: status, the allocation in
virtual SMs and, with ``bounds=True``, the end-to-end bounds as exact
numerator / denominator pairs -- the same values ``analyze_batch``'s reports
carry (reference analysis.py:275-298), without building report objects.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Optional, Union

import numpy as np

from . import engine
from .model import (AnalysisMethod, ExecBounds, GpuKernelModel, MemModel, PlatformConfig, TaskSet,
                    TaskSpec, expected_mem_count)
from .pack import F_BOUNDS, HDR_WORDS, MAX_M, MAX_TASKS, METHOD_CODES, NONE, TASK_WORDS

I32_MIN, I32_MAX = -(1 << 31), (1 << 31) - 1


@dataclass
class TaskArrays:
    """S task sets of n tasks with m CPU segments each (reference model.py:70
    field for field).  Durations are integers in one tick unit of the
    caller's choice (microseconds for the reference's generator); results
    come back in the same unit.  p = 2m - 2 (two-copy) or m - 1 (one-copy)
    memory copies, g = m - 1 kernels (0 and 0 when m == 1)."""

    deadline: np.ndarray          # [S, n]
    period: np.ndarray            # [S, n]
    priority: np.ndarray          # [S, n]   (lower value = higher priority)
    cpu_lo: np.ndarray            # [S, n, m]
    cpu_hi: np.ndarray            # [S, n, m]
    mem_lo: np.ndarray            # [S, n, p]
    mem_hi: np.ndarray            # [S, n, p]
    work_lo: np.ndarray           # [S, n, g]  single-SM kernel work bounds
    work_hi: np.ndarray           # [S, n, g]
    overhead: np.ndarray          # [S, n, g]  critical-path (launch) overhead
    ratio_num: np.ndarray         # [S, n, g]  interleave ratio = ratio_num / ratio_den
    ratio_den: int = 1
    physical_sms: Union[int, np.ndarray] = 10   # scalar or [S]
    mem_model: MemModel = MemModel.TWO_COPY

    @property
    def shape(self) -> tuple[int, int, int]:
        S, n, m = np.shape(self.cpu_lo)
        return S, n, m

    def check(self) -> None:
        """Shapes and engine limits (pack._check_shape); ValueError if violated."""
        S, n, m = self.shape
        if not 1 <= n <= MAX_TASKS:
            raise ValueError(f"engine supports 1..{MAX_TASKS} tasks per set")
        if not 1 <= m <= MAX_M:
            raise ValueError(f"engine supports 1..{MAX_M} CPU segments")
        p, g = expected_mem_count(m, MemModel(self.mem_model)), m - 1
        want = {"deadline": (S, n), "period": (S, n), "priority": (S, n), "cpu_lo": (S, n, m),
                "cpu_hi": (S, n, m), "mem_lo": (S, n, p), "mem_hi": (S, n, p), "work_lo": (S, n, g),
                "work_hi": (S, n, g), "overhead": (S, n, g), "ratio_num": (S, n, g)}
        for name, shp in want.items():
            if np.shape(getattr(self, name)) != shp:
                raise ValueError(f"{name}: shape {np.shape(getattr(self, name))}, expected {shp}")
        if int(self.ratio_den) < 1:
            raise ValueError("ratio_den must be >= 1")
        if np.ndim(self.physical_sms) not in (0, 1) or (np.ndim(self.physical_sms) == 1
                                                        and len(self.physical_sms) != S):
            raise ValueError("physical_sms: a scalar or one value per set")

    @classmethod
    def from_blobs(cls, blobs: np.ndarray, set_off: np.ndarray) -> "TaskArrays":
        """The sets of a batch of same-shape blobs (e.g. the native
        generator's, workbench.generate_blobs) as arrays, tasks in their
        TaskSet.tasks order (task record word 6); the inverse of pack_arrays
        for integer-tick sets."""
        blobs = np.asarray(blobs, np.int64)
        set_off = np.asarray(set_off, np.int64)
        S = len(set_off) - 1
        W = int(set_off[1] - set_off[0]) if S else 0
        if S == 0 or not np.all(np.diff(set_off) == W):
            raise ValueError("from_blobs: sets of one shape (equal blob sizes) expected")
        B = blobs[int(set_off[0]):int(set_off[-1])].reshape(S, W)
        n, mm, cform = int(B[0, 0]), int(B[0, 2]), int(B[0, 7])
        rw = TASK_WORDS // 2 if cform == 2 else TASK_WORDS  # int64 words per record (2: packed records)
        rec = B[:, HDR_WORDS:HDR_WORDS + rw * n].reshape(S, n, rw)
        if cform == 2:  # D, T, m | p << 8 | index << 16, priority (int32) | seg_off << 32
            w = rec
            rec = np.zeros((S, n, TASK_WORDS), np.int64)
            rec[:, :, 0] = w[:, :, 2] & 0xff
            rec[:, :, 1] = (w[:, :, 2] >> 8) & 0xff
            rec[:, :, 2] = w[:, :, 0]
            rec[:, :, 3] = w[:, :, 1]
            rec[:, :, 4] = (w[:, :, 3] & 0xffffffff).astype(np.uint32).view(np.int32)
            rec[:, :, 5] = w[:, :, 3] >> 32
            rec[:, :, 6] = w[:, :, 2] >> 16
        m, p = int(rec[0, 0, 0]), int(rec[0, 0, 1])
        g = m - 1
        if not (np.all(B[:, 0] == n) and np.all(B[:, 2] == mm) and np.all(B[:, 7] == cform)
                and np.all(rec[:, :, 0] == m) and np.all(rec[:, :, 1] == p)):
            raise ValueError("from_blobs: sets of one shape expected")
        per = 2 * m + 2 * p + 4 * g
        base = HDR_WORDS + rw * n
        area = B[:, base:].copy().view(np.int32) if cform else B[:, base:]
        start = rec[:, :, 5] - (2 * base if cform else base)  # [S, n] offsets inside the area
        idx = start[:, :, None] + np.arange(per)[None, None, :]
        seg = np.take_along_axis(area, idx.reshape(S, n * per), axis=1).reshape(S, n, per).astype(np.int64)
        inv = np.argsort(rec[:, :, 6], axis=1)  # caller task i at blob position inv[s, i]
        put = lambda x: np.take_along_axis(x, inv if x.ndim == 2 else inv[:, :, None], axis=1)  # noqa: E731
        o = np.cumsum([0, m, m, p, p, g, g, g, g])
        f = [put(seg[:, :, o[k]:o[k + 1]]) for k in range(8)]
        A = B[:, 3]
        den = int(np.lcm.reduce(A))
        return cls(deadline=put(rec[:, :, 2]), period=put(rec[:, :, 3]), priority=put(rec[:, :, 4]),
                   cpu_lo=f[0], cpu_hi=f[1], mem_lo=f[2], mem_hi=f[3], work_lo=f[4], work_hi=f[5],
                   overhead=f[6], ratio_num=f[7] * (den // A)[:, None, None], ratio_den=den,
                   physical_sms=B[:, 1].copy(), mem_model=MemModel.TWO_COPY if mm == 0 else MemModel.ONE_COPY)

    def taskset(self, k: int) -> TaskSet:
        """Set k as a TaskSet (task ids t0..t{n-1}) -- for cross-checks with
        the object API."""
        S, n, m = self.shape
        den = int(self.ratio_den)
        tasks = []
        for i in range(n):
            cpu = tuple(ExecBounds(Fraction(int(self.cpu_lo[k, i, j])), Fraction(int(self.cpu_hi[k, i, j])))
                        for j in range(m))
            mem = tuple(ExecBounds(Fraction(int(a)), Fraction(int(b)))
                        for a, b in zip(self.mem_lo[k, i], self.mem_hi[k, i]))
            gpu = tuple(GpuKernelModel(ExecBounds(Fraction(int(self.work_lo[k, i, j])),
                                                  Fraction(int(self.work_hi[k, i, j]))),
                                       Fraction(int(self.overhead[k, i, j])),
                                       Fraction(int(self.ratio_num[k, i, j]), den))
                        for j in range(m - 1))
            tasks.append(TaskSpec(f"t{i}", cpu, mem, gpu, Fraction(int(self.deadline[k, i])),
                                  Fraction(int(self.period[k, i])), int(self.priority[k, i])))
        sms = int(np.broadcast_to(np.asarray(self.physical_sms), (S,))[k])
        return TaskSet(tuple(tasks), MemModel(self.mem_model), PlatformConfig(sms))


@dataclass
class ArrayPack:
    """pack_arrays' output: the batch buffers plus each set's task order."""

    blobs: np.ndarray      # int64 [S * W]
    set_off: np.ndarray    # int64 [S + 1]
    task_base: np.ndarray  # int64 [S + 1]
    order: np.ndarray      # int64 [S, n]: blob position r holds caller task order[s, r]
    compact: bool

    @property
    def n_sets(self) -> int:
        return len(self.set_off) - 1


def pack_arrays(a: TaskArrays, compact: Optional[bool] = None) -> ArrayPack:
    """TaskArrays -> engine blobs (include/rtgpu.h), vectorised over sets.

    Per set: tasks in stable priority order (TaskSet.by_priority, reference
    model.py:107), time scale 1 (integer ticks), interleave denominator A =
    the lcm of the reduced ratio denominators.  compact=None packs int32
    segment areas when every segment value fits (the form the fast and
    lattice kernels read), True requires it, False keeps int64."""
    a.check()
    try:
        from . import _packer
    except ImportError:
        _packer = None
    if _packer is not None:
        return _pack_native(_packer, a, compact)
    return pack_arrays_np(a, compact)


def _pack_native(_packer, a: TaskArrays, compact: Optional[bool]) -> ArrayPack:
    """csrc/packer.cpp's pack_arrays: one pass per set, threads over sets."""
    S, n, m = a.shape
    mm = MemModel(a.mem_model)
    p, g = expected_mem_count(m, mm), m - 1
    c = lambda x: np.ascontiguousarray(x, np.int64)  # noqa: E731
    ins = [c(a.deadline), c(a.period), c(a.priority), c(a.cpu_lo), c(a.cpu_hi), c(a.mem_lo), c(a.mem_hi),
           c(a.work_lo), c(a.work_hi), c(a.overhead), c(a.ratio_num),
           c(np.broadcast_to(np.asarray(a.physical_sms, np.int64), (S,)))]
    per = 2 * m + 2 * p + 4 * g
    mmc = 0 if mm is MemModel.TWO_COPY else 1
    order = np.empty((S, n), np.int64)
    for want in ((True, False) if compact is None else (bool(compact),)):
        W = HDR_WORDS + TASK_WORDS * n + ((n * per + 1) // 2 if want else n * per)
        out = np.empty(S * W, np.int64)
        try:
            _packer.pack_arrays(S, n, m, p, g, int(a.ratio_den), mmc, int(want), *ins, out, order)
        except OverflowError:
            if compact:
                raise ValueError("segment values exceed int32: pack with compact=False") from None
            continue
        return ArrayPack(out, np.arange(S + 1, dtype=np.int64) * W, np.arange(S + 1, dtype=np.int64) * n,
                         order, want)
    raise AssertionError("unreachable")


def pack_arrays_np(a: TaskArrays, compact: Optional[bool] = None) -> ArrayPack:
    """pack_arrays in whole-array numpy (the restatement the native packer is
    tested against; also used when the extension is not built)."""
    a.check()
    S, n, m = a.shape
    mm = MemModel(a.mem_model)
    p, g = expected_mem_count(m, mm), m - 1
    i64 = np.int64
    order = np.argsort(np.asarray(a.priority, i64), axis=1, kind="stable").astype(i64)

    def by_prio(x, k):
        x = np.asarray(x, i64).reshape(S, n, k)
        return np.take_along_axis(x, order[:, :, None], axis=1)

    # interleave denominator: lcm_j(den / gcd(num_j, den)) = den / gcd(den, nums)
    den = int(a.ratio_den)
    rn = by_prio(a.ratio_num, g)
    G = np.gcd(np.gcd.reduce(rn.reshape(S, n * g), axis=1), den) if g else np.full(S, den, i64)
    A = den // G
    alpha = rn // G[:, None, None]
    # segment area per task: cl_lo[m] cl_hi[m] ml_lo[p] ml_hi[p] gw_lo[g] gw_hi[g] gl[g] alpha[g]
    segs = np.concatenate([by_prio(a.cpu_lo, m), by_prio(a.cpu_hi, m), by_prio(a.mem_lo, p),
                           by_prio(a.mem_hi, p), by_prio(a.work_lo, g), by_prio(a.work_hi, g),
                           by_prio(a.overhead, g), alpha], axis=2)
    per = 2 * m + 2 * p + 4 * g
    fits = bool(segs.size == 0 or (segs.min() >= I32_MIN and segs.max() <= I32_MAX))
    if compact is None:
        compact = fits
    elif compact and not fits:
        raise ValueError("segment values exceed int32: pack with compact=False")
    base = HDR_WORDS + TASK_WORDS * n
    seg_words = (n * per + 1) // 2 if compact else n * per
    W = base + seg_words
    out = np.zeros((S, W), i64)
    out[:, 0] = n
    out[:, 1] = np.broadcast_to(np.asarray(a.physical_sms, i64), (S,))
    out[:, 2] = 0 if mm is MemModel.TWO_COPY else 1
    out[:, 3] = A
    out[:, 4] = W
    out[:, 5] = m
    out[:, 6] = p
    out[:, 7] = 1 if compact else 0
    rec = out[:, HDR_WORDS:base].reshape(S, n, TASK_WORDS)
    rec[:, :, 0] = m
    rec[:, :, 1] = p
    rec[:, :, 2] = np.take_along_axis(np.asarray(a.deadline, i64), order, axis=1)
    rec[:, :, 3] = np.take_along_axis(np.asarray(a.period, i64), order, axis=1)
    rec[:, :, 4] = np.take_along_axis(np.asarray(a.priority, i64), order, axis=1)
    r = np.arange(n, dtype=i64)
    rec[:, :, 5] = (2 * base if compact else base) + r * per
    rec[:, :, 6] = order
    if compact:
        area = np.zeros((S, 2 * seg_words), np.int32)
        area[:, :n * per] = segs.reshape(S, n * per)
        out[:, base:] = area.view(i64)
    else:
        out[:, base:] = segs.reshape(S, n * per)
    set_off = np.arange(S + 1, dtype=i64) * W
    task_base = np.arange(S + 1, dtype=i64) * n
    return ArrayPack(out.reshape(-1), set_off, task_base, order, compact)


@dataclass
class ArrayReport:
    """analyze_arrays' results, tasks in the caller's order."""

    status: np.ndarray     # int32 [S]: 0 unschedulable, 1 schedulable (pack.UNDECIDED .. INVALID)
    vsm: np.ndarray        # int32 [S, n]: virtual SMs (2 x physical) per task, 0 if none
    e2e_num: Optional[np.ndarray]  # int64 [S, n] end-to-end bound numerators (ticks), -1 = None
    e2e_den: Optional[np.ndarray]  # int64 [S, n]
    evals: np.ndarray      # int64 [S] task evaluations of the allocation search

    @property
    def schedulable(self) -> np.ndarray:
        return self.status == 1

    def end_to_end(self, s: int, i: int) -> Optional[Fraction]:
        """Task i of set s as the reference's exact Fraction (None = no bound)."""
        if self.e2e_num is None:
            raise ValueError("analyze_arrays(bounds=True) computes the bounds")
        v = int(self.e2e_num[s, i])
        return None if v == NONE or v < 0 else Fraction(v, int(self.e2e_den[s, i]))


def analyze_arrays(a: TaskArrays, method: AnalysisMethod = AnalysisMethod.RTGPU,
                   bounds: bool = False, budget: int = 0) -> ArrayReport:
    """Verdicts and allocations (and with bounds=True every task's
    end-to-end bound) of S same-shape sets in one engine call: the batch form
    of analyze_rtgpu / the baselines (reference analysis.py:275, :319, :355).
    budget <= 0: unlimited allocation search."""
    S, n, _ = a.shape
    if S == 0:
        a.check()
        z = np.zeros((0, n), np.int64)
        return ArrayReport(np.zeros(0, np.int32), np.zeros((0, n), np.int32), z if bounds else None,
                           z.copy() if bounds else None, np.zeros(0, np.int64))
    pk = pack_arrays(a)
    flags = F_BOUNDS if bounds else 0
    res = engine.analyze_packed(pk.blobs, pk.set_off, pk.task_base, METHOD_CODES[AnalysisMethod(method)],
                                flags, budget)
    inv = np.argsort(pk.order, axis=1)  # caller task i sits at blob position inv[s, i]

    def caller(x):
        return np.take_along_axis(np.asarray(x).reshape(S, n), inv, axis=1)

    num = den = None
    if bounds:
        num, den = caller(res.e2e_num), caller(res.den)
    return ArrayReport(res.status, caller(res.vsm), num, den, res.evals)
