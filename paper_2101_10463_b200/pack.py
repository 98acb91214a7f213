"""Packing of TaskSets into the engine's int64 blob layout and unpacking of
engine results into ``AnalysisReport`` objects.

The layout is documented in ``include/rtgpu.h``.  Every exact rational of a
task set is brought to integers with one per-set time scale S (lcm of all
duration denominators, normally 1 for integer-microsecond tasksets) and one
interleave-ratio denominator A (lcm of the ratio denominators, normally a
divisor of 100).  The engine returns numerator / denominator pairs in input
ticks; dividing by S gives microseconds again, so results are bit-exact
Fractions, not floats.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from typing import Optional, Sequence

import numpy as np

from .model import (
    AnalysisMethod,
    AnalysisReport,
    ExecBounds,
    MemModel,
    SmAllocation,
    TaskReport,
    TaskSet,
    expected_mem_count,
)

HDR_WORDS = 8
TASK_WORDS = 8
MAX_TASKS = 64
MAX_M = 16
INT64_MAX = (1 << 63) - 1

# status codes (include/rtgpu.h)
UNSCHEDULABLE, SCHEDULABLE, UNDECIDED, RANGE, INVALID = 0, 1, 2, 3, 4
NONE, ABSENT = -1, -2
METHOD_CODES = {AnalysisMethod.RTGPU: 0, AnalysisMethod.SELF_SUSPENSION: 1,
                AnalysisMethod.BUSY_WAITING: 2}
F_BOUNDS, F_DETAIL = 1, 2


class EngineRangeError(ArithmeticError):
    """The exact values of a task set exceed the engine's integer range."""


@dataclass
class SetMeta:
    """What the unpacker needs to turn engine output back into a report."""

    ts: TaskSet
    order: tuple  # TaskSpec objects in by_priority() order (blob order)
    time_scale: int
    word_off: int
    task_base: int


@dataclass
class PackedBatch:
    blobs: np.ndarray      # int64 [W]
    set_off: np.ndarray    # int64 [S + 1]
    task_base: np.ndarray  # int64 [S + 1]
    metas: list

    @property
    def n_sets(self) -> int:
        return len(self.metas)


class _NativeMetas:
    """SetMeta records of a natively packed batch, built when read: a sweep
    that wants verdicts only never pays for them."""

    __slots__ = ("tasksets", "scales", "orders", "set_off", "task_base")

    def __init__(self, tasksets, scales, orders, set_off, task_base):
        self.tasksets, self.scales, self.orders = tasksets, scales, orders
        self.set_off, self.task_base = set_off, task_base

    def __len__(self) -> int:
        return len(self.scales)

    def __getitem__(self, k: int) -> SetMeta:
        if k < 0:
            k += len(self.scales)
        if not 0 <= k < len(self.scales):
            raise IndexError(k)
        return SetMeta(self.tasksets[k], self.orders[k], self.scales[k], int(self.set_off[k]),
                       int(self.task_base[k]))

    def __iter__(self):
        return (self[k] for k in range(len(self.scales)))


def _lcm_all(values) -> int:
    out = 1
    for v in values:
        out = out * v // math.gcd(out, v)
    return out


def _durations(ts: TaskSet):
    for t in ts.tasks:
        yield t.deadline
        yield t.period
        for b in t.cpu_segments:
            yield b.lo
            yield b.hi
        for b in t.mem_segments:
            yield b.lo
            yield b.hi
        for g in t.gpu_segments:
            yield g.work.lo
            yield g.work.hi
            yield g.critical_path_overhead


def _check_shape(ts: TaskSet) -> None:
    if len(ts.tasks) > MAX_TASKS:
        raise ValueError(f"engine supports at most {MAX_TASKS} tasks per set")
    for t in ts.tasks:
        m = len(t.cpu_segments)
        if not 0 <= m <= MAX_M:
            raise ValueError(f"task {t.id}: engine supports 0..{MAX_M} CPU segments")
        if len(t.gpu_segments) != max(m - 1, 0):
            raise ValueError(f"task {t.id}: gpu segment count != {max(m - 1, 0)}")
        want = expected_mem_count(m, ts.mem_model)
        if len(t.mem_segments) != want:
            raise ValueError(f"task {t.id}: mem segment count != {want}")


def build_blob(rows: Sequence[dict], physical_sms: int, mem_model_code: int, alpha_den: int) -> list[int]:
    """Blob from integer task rows (keys: m, p, D, T, prio, idx, cl_lo, cl_hi,
    ml_lo, ml_hi, gw_lo, gw_hi, gl, an), already in priority order."""
    n = len(rows)
    header = [n, physical_sms, mem_model_code, alpha_den, 0,
              max((r["m"] for r in rows), default=0), max((r["p"] for r in rows), default=0), 0]
    records: list[int] = []
    segs: list[int] = []
    base = HDR_WORDS + TASK_WORDS * n
    for r in rows:
        records += [r["m"], r["p"], r["D"], r["T"], r["prio"], base + len(segs), r["idx"], 0]
        for key in ("cl_lo", "cl_hi", "ml_lo", "ml_hi", "gw_lo", "gw_hi", "gl", "an"):
            segs += list(r[key])
    blob = header + records + segs
    blob[4] = len(blob)
    for v in blob:
        if not -INT64_MAX <= v <= INT64_MAX:
            raise EngineRangeError("task set values exceed int64 after scaling")
    return blob


def lcm_denominators(values) -> int:
    return _lcm_all(Fraction(v).denominator for v in values)


def _den(x) -> int:
    """Denominator of an int / Fraction duration without building a Fraction."""
    d = getattr(x, "denominator", None)
    return d if d is not None else Fraction(x).denominator


def pack_set(ts: TaskSet) -> tuple[list[int], int, tuple]:
    """One blob as a list of Python ints plus its time scale and task order."""
    _check_shape(ts)
    S = _lcm_all(_den(d) for d in _durations(ts))
    A = _lcm_all(_den(g.interleave_ratio) for t in ts.tasks for g in t.gpu_segments)
    order = ts.by_priority()
    index_of = {id(t): i for i, t in enumerate(ts.tasks)}
    n = len(order)

    def tick(x) -> int:
        # x * S exactly: S is a multiple of x's denominator (integer
        # arithmetic, no Fraction objects on the hot path of bulk packing)
        num, den = getattr(x, "numerator", None), getattr(x, "denominator", None)
        if num is None:
            f = Fraction(x)
            num, den = f.numerator, f.denominator
        q, r = divmod(S, den)
        assert r == 0
        return num * q

    header = [n, ts.platform.physical_sms,
              0 if ts.mem_model is MemModel.TWO_COPY else 1, A, 0,
              max((len(t.cpu_segments) for t in order), default=0),
              max((len(t.mem_segments) for t in order), default=0), 0]
    records: list[int] = []
    segs: list[int] = []
    seg_base = HDR_WORDS + TASK_WORDS * n
    for t in order:
        m, p = len(t.cpu_segments), len(t.mem_segments)
        records += [m, p, tick(t.deadline), tick(t.period), t.priority,
                    seg_base + len(segs), index_of[id(t)], 0]
        segs += [tick(b.lo) for b in t.cpu_segments]
        segs += [tick(b.hi) for b in t.cpu_segments]
        segs += [tick(b.lo) for b in t.mem_segments]
        segs += [tick(b.hi) for b in t.mem_segments]
        segs += [tick(g.work.lo) for g in t.gpu_segments]
        segs += [tick(g.work.hi) for g in t.gpu_segments]
        segs += [tick(g.critical_path_overhead) for g in t.gpu_segments]
        for g in t.gpu_segments:
            r = g.interleave_ratio
            num, den = getattr(r, "numerator", None), getattr(r, "denominator", None)
            if num is None:
                f = Fraction(r)
                num, den = f.numerator, f.denominator
            segs.append(num * (A // den))
    blob = header + records + segs
    blob[4] = len(blob)
    for v in blob:
        if not -INT64_MAX <= v <= INT64_MAX:
            raise EngineRangeError("task set values exceed int64 after scaling")
    return blob, S, order


def pack_tasksets(tasksets: Sequence[TaskSet], compact: bool = False) -> PackedBatch:
    """The batch of blobs: the native packer (csrc/packer.cpp, the same
    words) when built; a set it refuses (values beyond int64, a shape the
    engine does not take) is packed by pack_set for the exact exception."""
    try:
        from . import _packer
    except ImportError:
        _packer = None
    if _packer is not None and tasksets:
        try:
            b, so, tb, scales, orders = _packer.pack(tasksets, compact)
        except (ValueError, OverflowError, TypeError, AttributeError):
            pass
        else:
            blobs = np.frombuffer(b, dtype=np.int64)
            set_off = np.frombuffer(so, dtype=np.int64)
            task_base = np.frombuffer(tb, dtype=np.int64)
            return PackedBatch(blobs, set_off, task_base,
                               _NativeMetas(tasksets, scales, orders, set_off, task_base))
    return pack_tasksets_py(tasksets)


def pack_tasksets_py(tasksets: Sequence[TaskSet]) -> PackedBatch:
    """Python packer (reference for the native one; exact exceptions)."""
    words: list[int] = []
    set_off = [0]
    task_base = [0]
    metas = []
    for ts in tasksets:
        blob, S, order = pack_set(ts)
        metas.append(SetMeta(ts, order, S, len(words), task_base[-1]))
        words += blob
        set_off.append(len(words))
        task_base.append(task_base[-1] + len(order))
    return PackedBatch(np.asarray(words, dtype=np.int64).reshape(-1),
                       np.asarray(set_off, dtype=np.int64),
                       np.asarray(task_base, dtype=np.int64), metas)


@dataclass
class RawResults:
    status: np.ndarray   # int32 [S]
    evals: np.ndarray    # int64 [S]
    vsm: np.ndarray      # int32 [T]
    e2e_num: np.ndarray  # int64 [T]
    den: np.ndarray      # int64 [T]
    detail: Optional[np.ndarray]  # int64 [W] or None

    @classmethod
    def empty(cls, batch: PackedBatch, detail: bool) -> "RawResults":
        S = batch.n_sets
        T = int(batch.task_base[-1])
        return cls(np.zeros(S, np.int32), np.zeros(S, np.int64), np.zeros(T, np.int32),
                   np.zeros(T, np.int64), np.ones(T, np.int64),
                   np.zeros(len(batch.blobs), np.int64) if detail else None)


def _val(num: int, den: int, S: int) -> Optional[Fraction]:
    if num == NONE:
        return None
    return Fraction(int(num), int(den) * S)


def unpack_report(batch: PackedBatch, res: RawResults, s: int,
                  method: AnalysisMethod) -> AnalysisReport:
    """AnalysisReport of set s, shaped exactly like the reference's."""
    meta: SetMeta = batch.metas[s]
    st = int(res.status[s])
    if st == INVALID:
        raise ValueError("critical-path overhead exceeds inflated work "
                         "(or a task set the reference cannot analyse)")
    if st == RANGE:
        raise EngineRangeError("exact values of this task set exceed the 127-bit range")
    if st == UNDECIDED:
        raise TimeoutError("allocation search exceeded its evaluation budget")
    S = meta.time_scale
    tb = meta.task_base
    allocation = None
    if st == SCHEDULABLE:
        by_id = {t.id: int(res.vsm[tb + i]) for i, t in enumerate(meta.order)}
        gpu_ids = [t.id for t in meta.order if t.gpu_segments]
        pure_ids = [t.id for t in meta.ts.tasks if not t.gpu_segments]
        allocation = SmAllocation({**{i: by_id[i] for i in gpu_ids},
                                   **{i: 0 for i in pure_ids}})
    per_task: dict[str, TaskReport] = {}
    for i, t in enumerate(meta.order):
        num = int(res.e2e_num[tb + i])
        if num == ABSENT:
            continue
        den = int(res.den[tb + i])
        e2e = _val(num, den, S)
        gpu_r: tuple = ()
        mem_r: tuple = ()
        cpu_r: tuple = ()
        if res.detail is not None:
            rec = batch.blobs[meta.word_off + HDR_WORDS + TASK_WORDS * i:
                              meta.word_off + HDR_WORDS + TASK_WORDS * (i + 1)]
            m, p = int(rec[0]), int(rec[1])
            g = max(m - 1, 0)
            base = meta.word_off + int(rec[5])
            d = res.detail[base: base + 2 * m + 2 * p + 4 * g]
            gl = d[2 * m + 2 * p: 2 * m + 2 * p + g]
            gh = d[2 * m + 2 * p + g: 2 * m + 2 * p + 2 * g]
            gpu_r = tuple(ExecBounds(_val(int(a), den, S), _val(int(b), den, S))
                          for a, b in zip(gl, gh))
            if method is AnalysisMethod.RTGPU:
                mem_r = tuple(_val(int(x), den, S) for x in d[2 * m: 2 * m + p])
                cpu_r = tuple(_val(int(x), den, S) for x in d[:m])
        per_task[t.id] = TaskReport(gpu_r=gpu_r, mem_r_up=mem_r, cpu_r_up=cpu_r,
                                    end_to_end_up=e2e)
    return AnalysisReport(st == SCHEDULABLE, method, allocation, per_task)
