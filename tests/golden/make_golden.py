"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``gpusched`` from /root/reference/pkg/src, generates task sets
(with the reference generator and with a small hand-rolled generator that
exercises T > D, lo < hi, pure-CPU tasks and invalid overheads), runs the
three analyses and writes ``tests/golden/rtgpu_golden.json`` (task sets in an
exact text form, reports in the reference's report_to_dict schema, or the
exception class name the reference raised).

The reference's two baselines raise NameError as shipped: analysis.py uses
SuspTask, task_response and ExecBounds without importing them.  This script
injects those three names into gpusched.analysis before calling the
baselines, i.e. it records the code "as written" -- the behaviour the oracle
restates -- and marks those entries "patched_imports": true.

Nothing at test time reads /root/reference; the tests only read the JSON.
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import random
import sys
from fractions import Fraction

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rtgpu_golden.json")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gpusched  # noqa: F401
    import gpusched.analysis as an
    from gpusched.model import ExecBounds
    from gpusched.suspension import SuspTask, task_response
    an.SuspTask, an.task_response, an.ExecBounds = SuspTask, task_response, ExecBounds
    return gpusched


def fs(x) -> str:
    x = Fraction(x)
    return str(x.numerator) if x.denominator == 1 else f"{x.numerator}/{x.denominator}"


def ts_to_exact(ts) -> dict:
    return {
        "mem_model": ts.mem_model.value,
        "physical_sms": ts.platform.physical_sms,
        "launch_overhead_frac": fs(ts.platform.launch_overhead_frac),
        "tasks": [{
            "id": t.id, "priority": t.priority, "deadline": fs(t.deadline),
            "period": fs(t.period),
            "cpu": [[fs(b.lo), fs(b.hi)] for b in t.cpu_segments],
            "mem": [[fs(b.lo), fs(b.hi)] for b in t.mem_segments],
            "gpu": [[fs(g.work.lo), fs(g.work.hi), fs(g.critical_path_overhead),
                     fs(g.interleave_ratio)] for g in t.gpu_segments],
        } for t in ts.tasks],
    }


def hand_taskset(g, rng: random.Random):
    """Small random task set with the shapes the generator never produces."""
    M = g.MemModel.TWO_COPY if rng.random() < 0.6 else g.MemModel.ONE_COPY
    n = rng.randint(1, 4)
    gn = rng.randint(1, 6)
    tasks = []
    prios = list(range(1, n + 1))
    rng.shuffle(prios)
    for i in range(n):
        m = rng.choice([1, 1, 2, 2, 3, 4])
        def eb(lo_max, hi_max):
            hi = rng.randint(0, hi_max)
            lo = rng.randint(0, hi) if rng.random() < 0.5 else hi
            return g.ExecBounds(Fraction(lo), Fraction(hi))
        cpu = tuple(eb(5, 6) for _ in range(m))
        nm = 0 if m == 1 else (2 * m - 2 if M is g.MemModel.TWO_COPY else m - 1)
        mem = tuple(eb(3, 4) for _ in range(nm))
        gpu = []
        for _ in range(m - 1):
            w = eb(20, 24)
            if w.hi == 0:
                w = g.ExecBounds(Fraction(0), Fraction(1))
            ov = Fraction(rng.randint(0, int(w.lo))) if rng.random() < 0.95 else w.hi + 3
            alpha = Fraction(rng.randint(100, 180), 100)
            gpu.append(g.GpuKernelModel(w, ov, alpha))
        demand = sum(b.hi for b in cpu) + sum(b.hi for b in mem) + sum(x.work.hi for x in gpu)
        D = Fraction(max(1, int(demand * Fraction(rng.randint(8, 40), 10))))
        if rng.random() < 0.2:
            D = D / rng.choice([2, 3, 7])  # non-integer deadline
        T = D + rng.choice([0, 0, 0, rng.randint(1, 20)])
        tasks.append(g.TaskSpec(f"h{i}", cpu, mem, tuple(gpu), D, T, prios[i]))
    return g.TaskSet(tuple(tasks), M, g.PlatformConfig(gn))


def run_case(case):
    g = _ref()
    kind, payload = case
    if kind == "gen":
        params, seed = payload
        gp = g.GenParams(
            n_tasks=params["n"], n_subtasks=params["m"], physical_sms=params["gn"],
            target_utilization=Fraction(params["u"]),
            mem_model=g.MemModel(params["mm"]), lo_frac=Fraction(params["lo"]),
            **({"gpu_range_us": tuple(params["gpu"])} if "gpu" in params else {}))
        ts = g.generate_taskset(gp, seed)
        rec = {"kind": "gen", "params": params, "seed": seed}
    else:
        rng = random.Random(payload)
        ts = hand_taskset(g, rng)
        rec = {"kind": "hand", "seed": payload}
    rec["taskset"] = ts_to_exact(ts)
    for method in ("rtgpu", "selfsusp", "busywait"):
        try:
            rep = g.analyze(ts, g.AnalysisMethod(method))
            from gpusched.model import report_to_dict
            rec[method] = report_to_dict(rep)
        except Exception as exc:  # the reference raised
            rec[method] = {"raises": type(exc).__name__}
    rec["patched_imports"] = True
    return rec


def cases():
    out = []
    grid = [(2, 2, 3), (3, 3, 4), (3, 3, 10), (4, 3, 10), (5, 3, 10), (3, 4, 6), (4, 2, 2)]
    k = 0
    for (n, m, gn) in grid:
        for u in ("1/5", "1/2", "4/5", "1", "3/2"):
            for mm in ("two_copy", "one_copy"):
                for lo in ("1", "3/5"):
                    p = {"n": n, "m": m, "gn": gn, "u": u, "mm": mm, "lo": lo}
                    out.append(("gen", (p, k)))
                    k += 1
    # the reference sweep's string cell seeds
    for idx in range(12):
        p = {"n": 3, "m": 3, "gn": 10, "u": "1/2", "mm": "two_copy", "lo": "1"}
        out.append(("gen", (p, f"7:{Fraction(1, 2)}:{idx}")))
    # the benchmark shape (8 tasks x 5 segments, 10 SMs), low utilisation only
    for s in range(6):
        p = {"n": 8, "m": 5, "gn": 10, "u": "1/5", "mm": "two_copy", "lo": "1"}
        out.append(("gen", (p, 1000 + s)))
    for s in range(240):
        out.append(("hand", 5000 + s))
    return out


def main():
    cs = cases()
    with mp.Pool(min(8, os.cpu_count() or 1)) as pool:
        recs = pool.map(run_case, cs, chunksize=1)
    with open(OUT, "w") as fh:
        json.dump({"source": "reference gpusched (pkg/src), see make_golden.py",
                   "cases": recs}, fh, separators=(",", ":"))
    print(f"wrote {len(recs)} cases to {OUT}")


if __name__ == "__main__":
    main()
