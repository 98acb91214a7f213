"""Golden simulator traces produced by the REFERENCE (needs /root/reference).

    python tests/golden/make_golden_sim.py

Runs gpusched.simulator.simulate (and check_against_analysis for accepted
sets) on generated and hand-built task sets -- both memory models, both
length policies, int / negative / large / str seeds, default and fractional
horizons, overloaded sets with deadline misses, several live jobs per task
and truncation -- and stores the full traces compactly in
tests/golden/sim_golden.json.  Nothing at test time reads /root/reference.
"""
from __future__ import annotations

import json
import os
import random
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import _ref, fs, hand_taskset, ts_to_exact  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sim_golden.json")


def allocation_for(g, ts, rng):
    """The analysis' allocation when it accepts; else a feasible one."""
    rep = g.analyze_rtgpu(ts)
    if rep.schedulable:
        return rep, dict(rep.allocation.per_task_virtual_sms)
    alloc, left = {}, ts.platform.physical_sms
    gpu_tasks = [t for t in ts.tasks if t.gpu_segments]
    if len(gpu_tasks) > left:
        return rep, None
    for t in ts.tasks:
        alloc[t.id] = 0
    for t in gpu_tasks:
        alloc[t.id] = 2
        left -= 1
    for t in gpu_tasks:  # spread the rest at random
        extra = rng.randint(0, max(0, left))
        alloc[t.id] += 2 * extra
        left -= extra
    return rep, alloc


def encode_trace(tr):
    """Full events for small traces; always the SHA-256 of to_jsonl()."""
    import hashlib
    return {
        "n_events": len(tr.events),
        "jsonl_sha256": hashlib.sha256(tr.to_jsonl().encode()).hexdigest(),
        "events": ([[fs(e.time), e.task, e.job, e.kind, e.segment, e.action] for e in tr.events]
                   if len(tr.events) <= 300 else None),
        "responses": [[t, j, fs(r)] for (t, j), r in tr.responses.items()],
        "releases": [[t, j, fs(r)] for (t, j), r in tr.releases.items()],
        "truncated": [[t, j] for t, j in tr.truncated],
    }


def main():
    g = _ref()
    from gpusched.simulator import LengthPolicy, SimConfig, check_against_analysis, simulate
    rng = random.Random(2101)
    cases = []
    specs = []
    for k, (n, m, gn, u, mm, lo) in enumerate([
            (2, 2, 4, "1/2", "two_copy", "1"), (3, 3, 6, "1", "two_copy", "1/2"),
            (3, 2, 4, "3/2", "one_copy", "1/2"), (4, 3, 10, "4/5", "two_copy", "3/5"),
            (4, 4, 8, "2", "one_copy", "1/2"), (5, 3, 10, "5/2", "two_copy", "1/2"),
            (2, 1, 2, "1", "two_copy", "1/2"), (3, 3, 3, "3", "two_copy", "1/2"),
            (6, 2, 12, "6/5", "one_copy", "3/5"), (5, 5, 10, "3/2", "two_copy", "1/2")]):
        gp = g.GenParams(n_tasks=n, n_subtasks=m, physical_sms=gn,
                         target_utilization=Fraction(u), mem_model=g.MemModel(mm),
                         lo_frac=Fraction(lo))
        specs.append(("gen", g.generate_taskset(gp, 500 + k), {"n": n, "m": m, "gn": gn, "u": u,
                                                                "mm": mm, "lo": lo}))
    hr = random.Random(77)
    while len(specs) < 24:
        ts = hand_taskset(g, hr)
        if g.validate_taskset(ts):
            continue
        if any(not (x.critical_path_overhead <= x.work.hi * x.interleave_ratio)
               for t in ts.tasks for x in t.gpu_segments):
            continue
        specs.append(("hand", ts, {}))
    seeds = [0, 1, 12345, -7, 2 ** 40 + 3, "abc", 3 ** 70]
    for ci, (kind, ts, params) in enumerate(specs):
        rep, alloc = allocation_for(g, ts, rng)
        if alloc is None:
            continue
        maxT = max(t.period for t in ts.tasks)
        for pol in (LengthPolicy.WORST_CASE, LengthPolicy.UNIFORM_RANDOM):
            horizon = None if ci % 3 else maxT * 3 + Fraction(1, 3)
            seed = seeds[(ci + (pol is LengthPolicy.UNIFORM_RANDOM)) % len(seeds)]
            cfg = SimConfig(horizon=horizon, seed=seed, length_policy=pol)
            tr = simulate(ts, g.SmAllocation(alloc), cfg)
            rec = {"kind": kind, "params": params, "taskset": ts_to_exact(ts),
                   "allocation": alloc, "policy": pol.value,
                   "horizon": None if horizon is None else fs(horizon),
                   "seed": seed, "trace": encode_trace(tr)}
            if rep.schedulable:
                from gpusched.model import report_to_dict
                rec["report"] = report_to_dict(rep)
                rec["violations"] = check_against_analysis(tr, rep)
                # the same check against bounds scaled by 3/4 (violations appear)
                import dataclasses
                tight = dataclasses.replace(rep, per_task={
                    tid: dataclasses.replace(
                        r, mem_r_up=tuple(None if x is None else x * 3 / 4 for x in r.mem_r_up),
                        cpu_r_up=tuple(None if x is None else x * 3 / 4 for x in r.cpu_r_up),
                        gpu_r=tuple(g.ExecBounds(b.lo * 3 / 4, b.hi * 3 / 4) for b in r.gpu_r),
                        end_to_end_up=None if r.end_to_end_up is None else r.end_to_end_up * 3 / 4)
                    for tid, r in rep.per_task.items()})
                rec["violations_tight"] = check_against_analysis(tr, tight)
            cases.append(rec)
    # error behaviour: an infeasible allocation and an invalid task set
    ts = specs[1][1]
    bad = {t.id: (2 if t.gpu_segments else 0) for t in ts.tasks}
    bad[ts.tasks[0].id] = 3 if ts.tasks[0].gpu_segments else 2
    try:
        simulate(ts, g.SmAllocation(bad), SimConfig())
        err = None
    except Exception as exc:
        err = [type(exc).__name__, str(exc)]
    cases.append({"kind": "error", "taskset": ts_to_exact(ts), "allocation": bad,
                  "policy": "worst", "horizon": None, "seed": 0, "raises": err})
    with open(OUT, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_sim.py (reference gpusched.simulator)",
                   "cases": cases}, fh, separators=(",", ":"))
    nev = sum(c["trace"]["n_events"] for c in cases if "trace" in c)
    print(f"{len(cases)} cases, {nev} events -> {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
