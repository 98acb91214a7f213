"""Multi-GPU acceptance sweeps: one process per GPU (torch.distributed over
NCCL), task sets sharded across ranks, one all_reduce of the acceptance
counts.  Task sets are independent, so there is no data-path collective:
each rank generates and analyses only its own slice of every sweep cell
(cell seeds do not depend on the rank, so the global result equals the
single-GPU sweep), and the per-cell counts -- a few KB -- are summed.
"""
from __future__ import annotations

import dataclasses
from fractions import Fraction
from typing import Callable, Optional, Sequence

import numpy as np

from .model import AnalysisMethod
from .pack import METHOD_CODES, SCHEDULABLE, UNSCHEDULABLE
from .workbench import (SweepConfig, SweepRow, apply_dimension, cell_seed, format_value,
                        generate_blobs)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [a, b) slice of n items for rank."""
    return (n * rank // world, n * (rank + 1) // world)


def concat_batches(parts):
    blobs, offs, tbs, wb, tb = [], [], [], 0, 0
    for b, so, t in parts:
        blobs.append(b)
        offs.append(so[:-1] + wb)
        tbs.append(t[:-1] + tb)
        wb += int(so[-1])
        tb += int(t[-1])
    set_off = np.concatenate(offs + [np.array([wb])]).astype(np.int64)
    task_base = np.concatenate(tbs + [np.array([tb])]).astype(np.int64)
    return np.concatenate(blobs), set_off, task_base


def gpu_status(blobs, set_off, task_base, method_code: int) -> np.ndarray:
    """Default analysis: the CUDA engine, verdicts only."""
    from .engine import analyze_packed
    return analyze_packed(blobs, set_off, task_base, method_code, 0, 0).status


def sharded_sweep(cfg: SweepConfig, rank: int = 0, world: int = 1, group=None,
                  analyze: Optional[Callable] = None, device=None) -> list[SweepRow]:
    """acceptance_sweep with the task sets of every cell split across ranks
    and the accepted counts summed with one all_reduce (every rank returns
    the global rows)."""
    import torch
    analyze = analyze or gpu_status
    a, b = shard_range(cfg.tasksets_per_point, rank, world)
    cells, parts = [], []
    for value in cfg.values:
        point = apply_dimension(cfg.params, cfg.dimension, value)
        for u in cfg.utilizations:
            gen = dataclasses.replace(point, target_utilization=Fraction(u))
            seeds = [cell_seed(cfg.master_seed, u, i) for i in range(a, b)]
            for mm in cfg.mem_models:
                cells.append((value, u, mm))
                if seeds:
                    parts.append(generate_blobs(dataclasses.replace(gen, mem_model=mm), seeds,
                                                compact=True))
    # one extra column: this rank's count of sets that are neither schedulable
    # nor unschedulable; it is reduced with the counts, so every rank learns
    # of a failure after the collective instead of one rank raising before it
    # and leaving the others blocked in all_reduce
    local = np.zeros((len(cfg.methods), len(cells) + 1), dtype=np.int64)
    if parts:
        blobs, set_off, task_base = concat_batches(parts)
        for mi, method in enumerate(cfg.methods):
            st = np.asarray(analyze(blobs, set_off, task_base,
                                    METHOD_CODES[AnalysisMethod(method)])).reshape(len(cells), b - a)
            local[mi, :-1] = (st == SCHEDULABLE).sum(axis=1)
            local[mi, -1] = int(np.sum((st != SCHEDULABLE) & (st != UNSCHEDULABLE)))
    counts = torch.from_numpy(local)
    if world > 1:
        import torch.distributed as dist
        if device is None and dist.get_backend(group) == "nccl":
            device = torch.device("cuda", torch.cuda.current_device())  # NCCL reduces device tensors only
    if device is not None:
        counts = counts.to(device)
    if world > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    counts = counts.cpu().numpy()
    if counts[:, -1].any():
        raise RuntimeError(f"{int(counts[:, -1].sum())} undecided task sets in the sweep")
    rows = []
    ci = 0
    per = cfg.tasksets_per_point
    for value in cfg.values:
        for u in cfg.utilizations:
            first = ci
            for mi, method in enumerate(cfg.methods):
                for k, mm in enumerate(cfg.mem_models):
                    rows.append(SweepRow(cfg.dimension, format_value(value), AnalysisMethod(method),
                                         mm, Fraction(u), Fraction(int(counts[mi, first + k]), per)))
            ci += len(cfg.mem_models)
    return rows
