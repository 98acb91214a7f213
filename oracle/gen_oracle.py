"""TEST INFRASTRUCTURE ONLY: the reference's task-set generator restated in
plain Python, packed into the engine's compact blob layout.

Restates /root/reference/pkg/src/gpusched/workbench.py:101 generate_taskset
(and :83 merge_memory_copies for the one-copy model) with the same RNG --
CPython's ``random.Random(seed)`` -- and exact ``Fraction`` arithmetic, so
it is an independent second implementation next to the product generator
(paper_2101_10463_b200/csrc/taskgen.cpp).  tests/test_gen_oracle.py checks
the two produce identical words.

bench.py's reference arm uses this module to build its inputs, so the
reference arm never loads the product library.  Blob layout: include/rtgpu.h
(header word 7 = 1: int32 segment areas).
"""
from __future__ import annotations

import random
from fractions import Fraction
from math import gcd

import numpy as np

KERNEL_CLASS_ALPHA_CAPS = (145, 170, 170, 180)  # workbench.py:38
HDR_WORDS, TASK_WORDS = 8, 8


def _lo(hi: int, lo_frac: Fraction) -> int:
    # workbench.py:78 _bounds
    lo = int(Fraction(hi) * lo_frac)
    return min(lo, hi)


def gen_blob(n: int, m: int, seed, physical_sms: int, target_utilization: Fraction,
             cpu_range=(1000, 20000), gpu_range=(1000, 20000), mem_range=None,
             mem_model: int = 0, launch_overhead_frac=Fraction(12, 100),
             lo_frac=Fraction(1)) -> list[int]:
    """One compact blob of workbench.generate_taskset(params, seed)."""
    if mem_range is None:  # workbench.py:58 effective_mem_range
        mem_range = (max(1, gpu_range[0] // 4), gpu_range[1] // 4)
    rng = random.Random(seed)
    while True:
        raw = [Fraction(rng.random()) for _ in range(n)]
        total = sum(raw, Fraction(0))
        if total > 0 and all(r > 0 for r in raw):
            break
    U = Fraction(target_utilization)
    utils = [r * U / total for r in raw]
    drafts = []
    for i in range(n):
        cpu = []
        for _ in range(m):
            hi = rng.randint(*cpu_range)
            cpu.append((_lo(hi, lo_frac), hi))
        mem = []
        for _ in range(2 * (m - 1)):
            hi = rng.randint(*mem_range)
            mem.append((_lo(hi, lo_frac), hi))
        gpu = []
        for _ in range(m - 1):
            hi = rng.randint(*gpu_range)
            lo = _lo(hi, lo_frac)
            cap = KERNEL_CLASS_ALPHA_CAPS[rng.randrange(4)]
            pct = rng.randint(100, cap)
            ov = min(int(Fraction(launch_overhead_frac) * hi), lo)
            gpu.append((lo, hi, ov, pct))
        demand = sum(h for _, h in cpu) + sum(h for _, h in mem) + sum(g[1] for g in gpu)
        deadline = max(1, int(Fraction(demand) / utils[i]))
        drafts.append((deadline, i, cpu, mem, gpu))
    order = sorted(range(n), key=lambda i: (drafts[i][0], i))
    if mem_model == 1:  # workbench.py:83 merge_memory_copies
        drafts = [(d, i, c, [(mm[2 * j][0] + mm[2 * j + 1][0], mm[2 * j][1] + mm[2 * j + 1][1])
                             for j in range(m - 1)], g)
                  for d, i, c, mm, g in drafts]
    A = 1
    for d in drafts:
        for g in d[4]:
            den = 100 // gcd(g[3], 100)
            A = A * den // gcd(A, den)
    pm = 0 if m < 2 else (m - 1 if mem_model == 1 else 2 * m - 2)
    header = [n, physical_sms, mem_model, A, 0, m, pm, 1]
    records, segs = [], []
    seg = (HDR_WORDS + TASK_WORDS * n) * 2  # int32 element offset
    for r, i in enumerate(order):
        D, idx, cpu, mem, gpu = drafts[i]
        records += [m, pm, D, D, r + 1, seg + len(segs), idx, 0]
        segs += [c[0] for c in cpu] + [c[1] for c in cpu]
        segs += [x[0] for x in mem] + [x[1] for x in mem]
        segs += [g[0] for g in gpu] + [g[1] for g in gpu] + [g[2] for g in gpu]
        segs += [g[3] * A // 100 for g in gpu]
    if len(segs) % 2:
        segs.append(0)
    s32 = np.asarray(segs, dtype=np.int32)
    words = header + records + [int(w) for w in s32.view(np.int64)]
    words[4] = len(words)
    return words


def gen_batch(n: int, m: int, seeds, physical_sms: int, target_utilization, **kw):
    """(blobs, set_off, task_base) for the given seeds, like _native.generate."""
    words, offs, tb = [], [0], [0]
    for sd in seeds:
        b = gen_blob(n, m, sd, physical_sms, target_utilization, **kw)
        words += b
        offs.append(len(words))
        tb.append(tb[-1] + n)
    return (np.asarray(words, dtype=np.int64), np.asarray(offs, dtype=np.int64),
            np.asarray(tb, dtype=np.int64))
