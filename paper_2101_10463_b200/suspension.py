"""Multi-segment self-suspension analysis (reference: suspension.py).

``workload``, ``max_workload``, ``segment_response`` and ``task_response``
run on the GPU (point queries, include/rtgpu.h) and return exact Fractions.
``inter_arrival`` is the closed-form gap accessor; ``chain_workload`` and
``fixed_point`` keep the reference's generic callable-based signatures (they
take Python callbacks, which cannot cross the C ABI) and are host helpers --
the engine runs its own closed-form chain walk and accelerated fixed point.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Callable, Optional, Sequence

from . import queries as Q
from .model import ExecBounds

ZERO = Fraction(0)


# ---------------------------------------------------------------- GPU path

def _rows(tasks: Sequence[SuspTask], S: int) -> list[dict]:
    """SuspTasks as engine rows: a two-copy task whose even copies carry the
    suspension bounds and whose kernels have zero length (so the CPU chain's
    gaps are exactly the suspension lower bounds)."""
    rows = []
    for i, t in enumerate(tasks):
        m = t.m
        ml_lo, ml_hi = [], []
        for s in t.susp_segments:
            ml_lo += [Q.ticks(s.lo, S), 0]
            ml_hi += [Q.ticks(s.hi, S), 0]
        rows.append({"m": m, "p": 2 * m - 2, "D": Q.ticks(t.deadline, S),
                     "T": Q.ticks(t.period, S), "prio": i + 1, "idx": i,
                     "cl_lo": [Q.ticks(b.lo, S) for b in t.exec_segments],
                     "cl_hi": [Q.ticks(b.hi, S) for b in t.exec_segments],
                     "ml_lo": ml_lo, "ml_hi": ml_hi, "gw_lo": [0] * (m - 1),
                     "gw_hi": [0] * (m - 1), "gl": [0] * (m - 1), "an": [1] * (m - 1)})
    return rows


def _scale(tasks: Sequence[SuspTask], *extra) -> int:
    vals = list(extra)
    for t in tasks:
        vals += [t.deadline, t.period]
        for b in t.exec_segments + t.susp_segments:
            vals += [b.lo, b.hi]
    return Q.lcm_denominators(vals)


def _query(tasks: Sequence[SuspTask], kind: int, index: int, horizon=ZERO, blocking=ZERO):
    S = _scale(tasks, horizon, blocking)
    blob = Q.build_blob(_rows(tasks, S), 1, 0, 1)
    (st, num, den), = Q.run([blob], [(0, kind, len(tasks) - 1, index,
                                      Q.ticks(max(horizon, ZERO), S), Q.ticks(blocking, S))])
    return Q.value(st, num, den, S)


def workload(t: SuspTask, h: int, horizon: Fraction) -> Fraction:
    """W_t^h(horizon), Lemma 1 (suspension.py:107), on the GPU."""
    if not 0 <= h < t.m:
        raise ValueError(f"start segment {h} out of range")
    if horizon <= 0:
        return ZERO
    return _query([t], Q.Q_WORKLOAD, h, Fraction(horizon))


def max_workload(t: SuspTask, horizon: Fraction) -> Fraction:
    """max over start segments (suspension.py:116), on the GPU."""
    if horizon <= 0:
        return ZERO
    return _query([t], Q.Q_MAX_WORKLOAD, 0, Fraction(horizon))


def segment_response(k: SuspTask, j: int, hp: Sequence[SuspTask],
                     blocking: Fraction = ZERO) -> Optional[Fraction]:
    """Lemma 2 recurrence for segment j of k (suspension.py:140), on the GPU."""
    if not 0 <= j < k.m:
        raise IndexError("segment index out of range")
    return _query(list(hp) + [k], Q.Q_SEGMENT_RESPONSE, j, ZERO, Fraction(blocking))


def task_response(k: SuspTask, hp: Sequence[SuspTask],
                  blocking: Fraction = ZERO) -> Optional[Fraction]:
    """Lemma 3: min(R1, R2) or None (suspension.py:155), on the GPU."""
    return _query(list(hp) + [k], Q.Q_TASK_RESPONSE, 0, ZERO, Fraction(blocking))


# ---------------------------------------------------------------- task model, host helpers

@dataclass(frozen=True)
class SuspTask:
    """m execution segments, m-1 suspensions, deadline and period
    (suspension.py:23); rejects a packed length beyond the period."""

    exec_segments: tuple[ExecBounds, ...]
    susp_segments: tuple[ExecBounds, ...]
    deadline: Fraction
    period: Fraction

    def __post_init__(self):
        m = len(self.exec_segments)
        if m < 1:
            raise ValueError("need at least one execution segment")
        if len(self.susp_segments) != m - 1:
            raise ValueError("need exactly m-1 suspension segments")
        if not 0 < self.deadline <= self.period:
            raise ValueError("deadline must satisfy 0 < D <= T")
        for b in self.exec_segments + self.susp_segments:
            if not 0 <= b.lo <= b.hi:
                raise ValueError(f"bad bounds {b}")
        if self.total_exec_up + sum((b.lo for b in self.susp_segments), ZERO) > self.period:
            raise ValueError("sum of execution uppers and suspension lowers exceeds the period")

    @property
    def m(self) -> int:
        return len(self.exec_segments)

    @property
    def total_exec_up(self) -> Fraction:
        return sum((b.hi for b in self.exec_segments), ZERO)

    @property
    def total_susp_up(self) -> Fraction:
        return sum((b.hi for b in self.susp_segments), ZERO)


def inter_arrival(t: SuspTask, j: int) -> Fraction:
    """Minimum gap after execution segment j (j counts across jobs):
    S_lo, then T - D after the first job, then the wrap-around gap."""
    m = t.m
    if j % m != m - 1:
        return t.susp_segments[j % m].lo
    if j == m - 1:
        return t.period - t.deadline
    return t.period - t.total_exec_up - sum((b.lo for b in t.susp_segments), ZERO)


def chain_workload(exec_up: Sequence[Fraction], gap: Callable[[int], Fraction], h: int,
                   horizon: Fraction) -> Fraction:
    """Greedy packing of a cyclic exec/gap chain into a window (host helper
    with the reference's callback signature, suspension.py:77)."""
    p = len(exec_up)
    if p == 0 or horizon <= 0:
        return ZERO
    cum = work = ZERO
    j = h
    while True:
        seg, g = exec_up[j % p], gap(j)
        if cum + seg + g > horizon:
            return work + max(ZERO, min(seg, horizon - cum))
        cum += seg + g
        work += seg
        j += 1


def fixed_point(base: Fraction, interference: Callable[[Fraction], Fraction],
                bound: Fraction) -> Optional[Fraction]:
    """Least fixed point of r = base + interference(r) from base, None past
    bound (host helper with the reference's callback signature)."""
    if base > bound:
        return None
    r = base
    while True:
        nxt = base + interference(r)
        if nxt == r:
            return r
        if nxt > bound:
            return None
        r = nxt
