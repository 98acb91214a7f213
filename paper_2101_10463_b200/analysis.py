"""Schedulability analyses (reference: analysis.py), run by the CUDA engine.

``analyze_rtgpu`` / ``analyze`` keep the reference signatures and return the
same ``AnalysisReport`` -- verdict, the first schedulable SM allocation of the
grid search (Algorithm 2) and every bound as an exact Fraction -- but the
search and all fixed points run on the GPU (include/rtgpu.h).  Many task sets
go through ``analyze_batch`` in one launch.
"""
from __future__ import annotations

from typing import Sequence

from . import engine
from .model import AnalysisMethod, AnalysisReport, TaskSet
from .pack import F_BOUNDS, F_DETAIL, METHOD_CODES, pack_tasksets, unpack_report


def analyze_batch(tasksets: Sequence[TaskSet], method: AnalysisMethod = AnalysisMethod.RTGPU,
                  detail: bool = True, budget: int = 0) -> list[AnalysisReport]:
    """Reports for many task sets in one engine call.

    detail=False skips the per-segment bounds (mem_r_up / cpu_r_up / gpu_r
    stay empty) but keeps verdict, allocation and end_to_end_up.
    """
    method = AnalysisMethod(method)
    if not tasksets:
        return []
    # compact blobs (int32 segment areas: the fast / lattice kernels' form)
    # unless the per-segment report needs the int64 detail layout
    batch = pack_tasksets(tasksets, compact=not detail)
    flags = F_DETAIL if detail else F_BOUNDS
    res = engine.analyze_packed(batch.blobs, batch.set_off, batch.task_base,
                                METHOD_CODES[method], flags, budget)
    return [unpack_report(batch, res, s, method) for s in range(batch.n_sets)]


def analyze_rtgpu(ts: TaskSet) -> AnalysisReport:
    """Grid-searched federated allocation with the decomposed bus/CPU
    self-suspension analysis (reference analysis.py:275)."""
    return analyze_batch([ts], AnalysisMethod.RTGPU)[0]


def analyze_self_suspension_baseline(ts: TaskSet) -> AnalysisReport:
    """Baseline 2 of the paper (reference analysis.py:319)."""
    return analyze_batch([ts], AnalysisMethod.SELF_SUSPENSION)[0]


def analyze_busy_waiting_baseline(ts: TaskSet) -> AnalysisReport:
    """Baseline 3 of the paper (reference analysis.py:355)."""
    return analyze_batch([ts], AnalysisMethod.BUSY_WAITING)[0]


ANALYZERS = {
    AnalysisMethod.RTGPU: analyze_rtgpu,
    AnalysisMethod.SELF_SUSPENSION: analyze_self_suspension_baseline,
    AnalysisMethod.BUSY_WAITING: analyze_busy_waiting_baseline,
}


def analyze(ts: TaskSet, method: AnalysisMethod) -> AnalysisReport:
    return ANALYZERS[AnalysisMethod(method)](ts)


# ---------------------------------------------------------------------------
# Building blocks with an explicit GPU-bound cache (analysis.py:57-225).
# The cache maps task id -> list of ExecBounds (GR lo/hi per kernel), as
# gpu.gpu_bounds_cache returns; the GPU evaluates them exactly.
# ---------------------------------------------------------------------------

from fractions import Fraction as _F  # noqa: E402
from typing import Optional as _Opt  # noqa: E402

from . import queries as _Q  # noqa: E402
from .model import MemModel as _MM, TaskSpec as _TS  # noqa: E402

InfeasibleGapError = _Q.InfeasibleGapError
GpuBoundsCache = dict
ZERO = _F(0)


def _check(gap, task_id: str, what: str):
    if gap < 0:
        raise InfeasibleGapError(f"task {task_id}: negative {what} gap {gap}")
    return gap


def mem_inter_arrival(ts: TaskSet, i: _TS, j: int, cache: GpuBoundsCache) -> _F:
    """Minimum gap after memory segment j of task i (analysis.py:57)."""
    p = len(i.mem_segments)
    if p == 0:
        raise ValueError("task has no memory segments")
    m, jp, gr, cl = i.n_subtasks, j % p, cache[i.id], i.cpu_segments
    if jp != p - 1:
        if ts.mem_model is _MM.TWO_COPY:
            return gr[jp // 2].lo if jp % 2 == 0 else cl[(jp + 1) // 2].lo
        return gr[jp].lo + cl[jp + 1].lo
    if j == p - 1:
        extra = gr[m - 2].lo if ts.mem_model is _MM.ONE_COPY else ZERO
        return _check(i.period - i.deadline + extra + cl[m - 1].lo + cl[0].lo, i.id,
                      "deadline-side")
    wrap = (i.period - sum((b.hi for b in i.mem_segments), ZERO)
            - sum((cl[q].lo for q in range(1, m - 1)), ZERO) - sum((g.lo for g in gr), ZERO))
    return _check(wrap, i.id, "wrap-around")


def cpu_inter_arrival(ts: TaskSet, i: _TS, j: int, cache: GpuBoundsCache) -> _F:
    """Minimum gap after CPU segment j of task i (analysis.py:89)."""
    m, jp, gr, ml = i.n_subtasks, j % i.n_subtasks, cache[i.id], i.mem_segments
    if jp != m - 1:
        if ts.mem_model is _MM.TWO_COPY:
            return ml[2 * jp].lo + gr[jp].lo + ml[2 * jp + 1].lo
        return ml[jp].lo + gr[jp].lo
    if j == m - 1:
        return i.period - i.deadline
    wrap = (i.period - sum((b.hi for b in i.cpu_segments), ZERO)
            - sum((b.lo for b in ml), ZERO) - sum((g.lo for g in gr), ZERO))
    return _check(wrap, i.id, "wrap-around")


def _explicit_blob(ts: TaskSet, cache: GpuBoundsCache, *extra):
    """ts with each kernel packed as one SM, alpha 1, GL 0, GW = 2 * GR."""
    from .pack import _check_shape
    _check_shape(ts)
    order = ts.by_priority()
    vals = list(extra)
    for t in ts.tasks:
        vals += [t.deadline, t.period]
        for b in t.cpu_segments + t.mem_segments:
            vals += [b.lo, b.hi]
        for b in cache.get(t.id, []):
            vals += [b.lo, b.hi]
    S = _Q.lcm_denominators(vals)
    T = _Q.ticks
    rows = []
    for t in order:
        g = len(t.gpu_segments)
        gr = cache.get(t.id, [])
        if len(gr) != g:
            raise KeyError(f"cache has no bounds for task {t.id}")
        rows.append({"m": t.n_subtasks, "p": len(t.mem_segments), "D": T(t.deadline, S),
                     "T": T(t.period, S), "prio": t.priority, "idx": 0,
                     "cl_lo": [T(b.lo, S) for b in t.cpu_segments],
                     "cl_hi": [T(b.hi, S) for b in t.cpu_segments],
                     "ml_lo": [T(b.lo, S) for b in t.mem_segments],
                     "ml_hi": [T(b.hi, S) for b in t.mem_segments],
                     "gw_lo": [2 * T(b.lo, S) for b in gr], "gw_hi": [2 * T(b.hi, S) for b in gr],
                     "gl": [0] * g, "an": [1] * g})
    blob = _Q.build_blob(rows, 1, 0 if ts.mem_model is _MM.TWO_COPY else 1, 1)
    return blob, S, [t.id for t in order]


def _block_query(ts, k: _TS, cache, kind: int, index: int = 0, horizon=ZERO):
    blob, S, ids = _explicit_blob(ts, cache, horizon)
    (st, num, den), = _Q.run([blob], [(0, kind, ids.index(k.id), index,
                                       _Q.ticks(max(horizon, ZERO), S), 0)])
    return _Q.value(st, num, den, S)


def mem_workload(ts: TaskSet, i: _TS, h: int, horizon: _F, cache: GpuBoundsCache) -> _F:
    """Lemma 5 bus workload of task i from memory segment h (analysis.py:109)."""
    if not i.mem_segments or horizon <= 0:
        return ZERO
    return _block_query(ts, i, cache, _Q.Q_MEM_WORKLOAD, h, _F(horizon))


def cpu_workload(ts: TaskSet, i: _TS, h: int, horizon: _F, cache: GpuBoundsCache) -> _F:
    """Lemma 7 CPU workload of task i from CPU segment h (analysis.py:118)."""
    if horizon <= 0:
        return ZERO
    return _block_query(ts, i, cache, _Q.Q_CPU_WORKLOAD, h, _F(horizon))


def mem_response(ts: TaskSet, k: _TS, j: int, cache: GpuBoundsCache, memo=None,
                 alloc=None) -> _Opt[_F]:
    """Lemma 6 (analysis.py:156) on the GPU; None when unschedulable."""
    return _block_query(ts, k, cache, _Q.Q_MEM_RESPONSE, j)


def cpu_response(ts: TaskSet, k: _TS, j: int, cache: GpuBoundsCache, memo=None,
                 alloc=None) -> _Opt[_F]:
    """Lemma 8 (analysis.py:175) on the GPU; None when unschedulable."""
    return _block_query(ts, k, cache, _Q.Q_CPU_RESPONSE, j)


def end_to_end(ts: TaskSet, k: _TS, cache: GpuBoundsCache, memo=None, alloc=None,
               mem_rs=None, cpu_rs=None) -> _Opt[_F]:
    """Theorem 1: min(R1, R2) (analysis.py:191) on the GPU."""
    if mem_rs is None and cpu_rs is None:
        return _block_query(ts, k, cache, _Q.Q_END_TO_END)
    if mem_rs is None:
        mem_rs = [mem_response(ts, k, j, cache) for j in range(len(k.mem_segments))]
    if cpu_rs is None:
        cpu_rs = [cpu_response(ts, k, j, cache) for j in range(k.n_subtasks)]
    if any(r is None for r in mem_rs):
        return None
    gr_up = sum((b.hi for b in cache[k.id]), ZERO)
    mr_up = sum(mem_rs, ZERO)
    r1 = None
    if all(r is not None for r in cpu_rs):
        cand = gr_up + mr_up + sum(cpu_rs, ZERO)
        if cand <= k.deadline:
            r1 = cand
    base = gr_up + mr_up + sum((b.hi for b in k.cpu_segments), ZERO)
    try:
        r2 = _block_query(ts, k, cache, _Q.Q_R2, 0, base)
    except InfeasibleGapError:
        r2 = None
    cands = [r for r in (r1, r2) if r is not None]
    return min(cands) if cands else None
