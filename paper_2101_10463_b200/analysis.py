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
    batch = pack_tasksets(tasksets)
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
