"""Independent parity at scale: the GPU engine (product API, device path)
against the oracle's enumeration -- full lexicographic enumeration on small
platforms, the prefix-pruned enumeration (ORACLE_PREFIX: exact, relies only
on the prefix property, not on the engine's monotonicity / dominance
argument) up to 48 SMs -- on generator sets and adversarial sets
(tests/blobtools.py: tight wrap-around gaps at g_min, lo < hi, irregular
copies, CPU-only tasks, equal priorities), both memory models.  Verdicts,
allocations and (bounds runs) end-to-end bounds are compared on every set
the oracle decides within its budget.

    python scripts/parity_scale.py [--minutes M] [--log FILE] [--seed S]

Writes one JSON line per shape and a final summary line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from blobtools import adversarial, compact  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.engine import DeviceBatch  # noqa: E402
from paper_2101_10463_b200.pack import F_BOUNDS  # noqa: E402

PREFIX = 0x200
UNDECIDED = 2


def generated(n, m, gn, u, count, mm, lo, seed):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), mm, gn,
                              Fraction(12, 100), Fraction(lo), compact=False)
    return _native.generate(gp, [f"{seed}:{u}:{i}" for i in range(count)])


def engine(b, so, tb, flags):
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=flags)
    return out.to_host()


def compare(o, e, so, tb, bounds):
    dec = o["status"] != UNDECIDED
    bad = []
    for s in np.where(dec)[0]:
        t0, t1 = tb[s], tb[s + 1]
        ok = o["status"][s] == e.status[s] and np.array_equal(o["vsm"][t0:t1], e.vsm[t0:t1])
        if ok and bounds:
            for t in range(t0, t1):
                a, c = int(o["e2e_num"][t]), int(e.e2e_num[t])
                if a < 0 or c < 0:
                    ok = ok and a == c
                else:
                    ok = ok and Fraction(a, int(o["den"][t])) == Fraction(c, int(e.den[t]))
        if not ok:
            bad.append(int(s))
    return int(dec.sum()), bad


def shapes(rng):
    """(label, generator) pairs, small platforms first (full enumeration)."""
    out = []
    for gn in (4, 6, 8, 10):
        for n in (3, 4, 5):
            out.append(("full", n, gn))
    for gn in (16, 24, 32, 48):
        for n in (6, 8):
            out.append(("prefix", n, gn))
    rng.shuffle(out)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=20.0)
    ap.add_argument("--log", default=os.path.join(ROOT, "gpurun_out", "parity_scale.jsonl"))
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--budget", type=int, default=50000)
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.log), exist_ok=True)
    oracle.build()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + 60 * args.minutes
    tot = dict(sets=0, decided=0, mismatches=0, schedulable=0, shapes=0)
    rnd = 0
    with open(args.log, "a") as log:
        while time.time() < t_end:
            for mode, n, gn in shapes(rng):
                if time.time() >= t_end:
                    break
                rnd += 1
                mm = int(rng.integers(0, 2))
                m = int(rng.integers(2, 7))
                kind = ["gen", "adv", "adv-irreg"][rnd % 3]
                count = 5000 if mode == "full" else 500
                seed = args.seed * 100003 + rnd
                if kind == "gen":
                    u = Fraction(int(rng.integers(1, 11)), 10)
                    lo = Fraction(int(rng.integers(5, 11)), 10)
                    b, so, tb = generated(n, m, gn, u, count, mm, lo, seed)
                    desc = f"generator u={u} lo={lo}"
                else:
                    ut = float(rng.choice([0.3, 0.5, 0.8]))
                    b, so, tb = adversarial(seed, count, n, m, gn, mm, u_total=ut,
                                            p_irreg=0.25 if kind == "adv-irreg" else 0.0)
                    desc = f"{kind} u_total={ut}"
                bounds = bool(rng.integers(0, 2))
                flags = F_BOUNDS if bounds else 0
                t0 = time.time()
                o = oracle.analyze_batch(b, so, tb, method=0, flags=(PREFIX if mode == "prefix" else 0)
                                         | (1 if bounds else 0), budget=args.budget if mode == "prefix" else 0,
                                         threads=threads, detail=False)
                t_or = time.time() - t0
                res = []
                for form in ("int64", "compact"):
                    bb = (b, so, tb) if form == "int64" else compact(b, so, tb)
                    e = engine(*bb, flags)
                    dec, bad = compare(o, e, so, tb, bounds)
                    res.append({"blob": form, "decided": dec, "mismatches": len(bad), "first_bad": bad[:5]})
                    tot["mismatches"] += len(bad)
                tot["sets"] += 2 * count
                tot["decided"] += 2 * res[0]["decided"]
                tot["schedulable"] += 2 * int((o["status"] == 1).sum())
                tot["shapes"] += 1
                line = {"oracle": mode, "n": n, "m_max": m, "gn": gn, "mem_model": mm, "sets": count,
                        "kind": desc, "bounds": bounds, "schedulable": int((o["status"] == 1).sum()),
                        "undecided": int((o["status"] == UNDECIDED).sum()), "oracle_s": round(t_or, 1),
                        "engine": res}
                log.write(json.dumps(line) + "\n")
                log.flush()
    summary = {"summary": True, **tot, "threads": threads, "budget": args.budget}
    with open(args.log, "a") as log:
        log.write(json.dumps(summary) + "\n")
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
