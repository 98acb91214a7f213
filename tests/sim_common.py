"""Shared helpers for the simulator tests (golden traces, oracle traces)."""
from __future__ import annotations

import hashlib
import json
from fractions import Fraction

from golden_io import load_cases, ts_from_exact
from paper_2101_10463_b200.model import SmAllocation, duration_to_str


def sim_cases():
    return [c for c in load_cases("sim_golden.json") if c["kind"] != "error"]


def error_cases():
    return [c for c in load_cases("sim_golden.json") if c["kind"] == "error"]


def case_inputs(c):
    ts = ts_from_exact(c["taskset"])
    alloc = SmAllocation(dict(c["allocation"]))
    horizon = None if c["horizon"] is None else Fraction(c["horizon"])
    return ts, alloc, horizon, c["seed"], c["policy"] == "uniform"


def jsonl(events) -> str:
    """SimTrace.to_jsonl of (time, task, job, kind, segment, action) tuples."""
    lines = [json.dumps({"time": duration_to_str(Fraction(t)), "task": task, "job": job,
                         "kind": kind, "segment": seg, "action": act})
             for t, task, job, kind, seg, act in events]
    return "\n".join(lines) + ("\n" if lines else "")


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def golden_events(c):
    ev = c["trace"]["events"]
    return None if ev is None else [(Fraction(t), task, job, kind, seg, act)
                                    for t, task, job, kind, seg, act in ev]


def golden_responses(c):
    return [(t, j, Fraction(r)) for t, j, r in c["trace"]["responses"]]


def golden_releases(c):
    return [(t, j, Fraction(r)) for t, j, r in c["trace"]["releases"]]


def golden_truncated(c):
    return [(t, j) for t, j in c["trace"]["truncated"]]
