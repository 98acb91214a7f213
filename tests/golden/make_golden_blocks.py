"""Golden fixtures for the analysis building blocks, produced by the REFERENCE.

    python tests/golden/make_golden_blocks.py      (needs /root/reference)

Writes tests/golden/blocks_golden.json:
  * "susp": random SuspTasks (exact rationals) with suspension.workload,
    max_workload, segment_response and task_response results, plus the
    worked examples of the reference spec;
  * "rtgpu": task sets with explicit GPU-bound caches (random rationals) and
    analysis.mem_response / cpu_response / end_to_end / mem_workload /
    cpu_workload results (or the exception the reference raised).
"""
from __future__ import annotations

import json
import os
import random
import sys
from fractions import Fraction

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "blocks_golden.json")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import gpusched as g  # noqa: E402
import gpusched.analysis as an  # noqa: E402
from gpusched.suspension import (SuspTask, max_workload, segment_response,  # noqa: E402
                                 task_response, workload)
from make_golden import fs, hand_taskset, ts_to_exact  # noqa: E402

F = Fraction


def susp_to_exact(t: SuspTask) -> dict:
    return {"exec": [[fs(b.lo), fs(b.hi)] for b in t.exec_segments],
            "susp": [[fs(b.lo), fs(b.hi)] for b in t.susp_segments],
            "deadline": fs(t.deadline), "period": fs(t.period)}


def rand_frac(rng, hi, den_choices=(1, 1, 1, 2, 3)):
    d = rng.choice(den_choices)
    return F(rng.randint(0, hi * d), d)


def rand_susp(rng) -> SuspTask:
    while True:
        m = rng.choice([1, 1, 2, 2, 3, 4])
        ex = []
        for _ in range(m):
            hi = rand_frac(rng, 6)
            ex.append(g.ExecBounds(rng.choice([hi, rand_frac(rng, int(hi)) if hi >= 1 else hi]), hi))
        su = []
        for _ in range(m - 1):
            hi = rand_frac(rng, 5)
            lo = min(hi, rand_frac(rng, 5))
            su.append(g.ExecBounds(lo, hi))
        packed = sum((b.hi for b in ex), F(0)) + sum((b.lo for b in su), F(0))
        T = packed + rand_frac(rng, 12)
        if T <= 0:
            continue
        D = T if rng.random() < 0.5 else max(F(1, 3), T - rand_frac(rng, 6))
        if not 0 < D <= T:
            continue
        try:
            return SuspTask(tuple(ex), tuple(su), D, T)
        except ValueError:
            continue


def susp_cases(rng, n=400):
    out = []
    for _ in range(n):
        k = rand_susp(rng)
        hp = [rand_susp(rng) for _ in range(rng.choice([0, 1, 1, 2, 3]))]
        B = rng.choice([F(0), F(0), rand_frac(rng, 4)])
        hz = [rand_frac(rng, 40, (1, 2, 3, 7)) for _ in range(3)]
        rec = {"k": susp_to_exact(k), "hp": [susp_to_exact(t) for t in hp], "blocking": fs(B),
               "horizons": [fs(h) for h in hz]}
        rec["workload"] = [[fs(workload(k, h, x)) for h in range(k.m)] for x in hz]
        rec["max_workload"] = [fs(max_workload(k, x)) for x in hz]
        rec["segment_response"] = [
            None if (r := segment_response(k, j, hp, B)) is None else fs(r) for j in range(k.m)]
        r = task_response(k, hp, B)
        rec["task_response"] = None if r is None else fs(r)
        out.append(rec)
    # worked examples of the reference spec (suspension_core examples)
    E = g.ExecBounds
    ex = SuspTask((E(F(2), F(2)), E(F(3), F(3))), (E(F(1), F(1)),), F(10), F(10))
    out.append({"k": susp_to_exact(ex), "hp": [], "blocking": "0", "horizons": ["2", "6", "0"],
                "workload": [[fs(workload(ex, h, F(x))) for h in range(2)] for x in (2, 6, 0)],
                "max_workload": [fs(max_workload(ex, F(x))) for x in (2, 6, 0)],
                "segment_response": [fs(segment_response(ex, j, [], F(0))) for j in range(2)],
                "task_response": fs(task_response(ex, [], F(0)))})
    return out


def rand_cache(rng, ts):
    cache = {}
    for t in ts.tasks:
        bounds = []
        for _ in t.gpu_segments:
            lo = rand_frac(rng, 8, (1, 2, 3, 4))
            hi = lo + rand_frac(rng, 6, (1, 2, 5))
            bounds.append(g.ExecBounds(lo, hi))
        cache[t.id] = bounds
    return cache


def call(fn, *a):
    try:
        r = fn(*a)
        return None if r is None else fs(r)
    except Exception as exc:  # reference raised
        return {"raises": type(exc).__name__}


def rtgpu_cases(rng, n=160):
    out = []
    for i in range(n):
        ts = hand_taskset(g, random.Random(9000 + i))
        cache = rand_cache(rng, ts)
        rec = {"taskset": ts_to_exact(ts),
               "cache": {k: [[fs(b.lo), fs(b.hi)] for b in v] for k, v in cache.items()},
               "tasks": []}
        for t in ts.by_priority():
            hz = rand_frac(rng, 60, (1, 2, 3))
            e = {"id": t.id, "horizon": fs(hz),
                 "mem_response": [call(an.mem_response, ts, t, j, cache)
                                  for j in range(len(t.mem_segments))],
                 "cpu_response": [call(an.cpu_response, ts, t, j, cache)
                                  for j in range(t.n_subtasks)],
                 "end_to_end": call(an.end_to_end, ts, t, cache),
                 "mem_workload": [call(an.mem_workload, ts, t, h, hz, cache)
                                  for h in range(len(t.mem_segments))],
                 "cpu_workload": [call(an.cpu_workload, ts, t, h, hz, cache)
                                  for h in range(t.n_subtasks)]}
            rec["tasks"].append(e)
        out.append(rec)
    return out


def main():
    rng = random.Random(2101)
    data = {"source": "reference gpusched, see make_golden_blocks.py",
            "susp": susp_cases(rng), "rtgpu": rtgpu_cases(rng)}
    with open(OUT, "w") as fh:
        json.dump(data, fh, separators=(",", ":"))
    print(f"wrote {len(data['susp'])} susp and {len(data['rtgpu'])} rtgpu cases to {OUT}")


if __name__ == "__main__":
    main()
