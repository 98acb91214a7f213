"""Analysis building blocks against the reference (tests/golden/blocks_golden.json,
produced by make_golden_blocks.py running the reference): suspension-core
workload / max_workload / segment_response / task_response on SuspTasks, and
the RTGPU per-segment recurrences with explicit GPU-bound caches.

CPU tests drive the engine core through the test harness at the blob level;
GPU tests call the package's public API (which runs rtgpu_query_host)."""
import json
import os
import sys
from fractions import Fraction as F

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402

from golden_io import GOLDEN_DIR, ts_from_exact  # noqa: E402
from paper_2101_10463_b200 import analysis as an  # noqa: E402
from paper_2101_10463_b200 import queries as Q  # noqa: E402
from paper_2101_10463_b200 import suspension as su  # noqa: E402
from paper_2101_10463_b200.model import ExecBounds  # noqa: E402


@pytest.fixture(scope="module")
def blocks():
    with open(os.path.join(GOLDEN_DIR, "blocks_golden.json")) as fh:
        return json.load(fh)


def susp(d):
    return su.SuspTask(tuple(ExecBounds(F(a), F(b)) for a, b in d["exec"]),
                       tuple(ExecBounds(F(a), F(b)) for a, b in d["susp"]),
                       F(d["deadline"]), F(d["period"]))


def cache_of(d):
    return {k: [ExecBounds(F(a), F(b)) for a, b in v] for k, v in d.items()}


def fval(x):
    return None if x is None else F(x)


def _susp_queries(rec):
    """(blob, scale, queries, expected) for one susp record, blob level."""
    k = susp(rec["k"])
    hp = [susp(t) for t in rec["hp"]]
    B = F(rec["blocking"])
    hz = [F(h) for h in rec["horizons"]]
    out = []
    S1 = su._scale([k], *hz)
    blob1 = Q.build_blob(su._rows([k], S1), 1, 0, 1)
    for xi, x in enumerate(hz):
        if x <= 0:
            continue
        for h in range(k.m):
            out.append((blob1, S1, (0, Q.Q_WORKLOAD, 0, h, Q.ticks(x, S1), 0),
                        F(rec["workload"][xi][h])))
        out.append((blob1, S1, (0, Q.Q_MAX_WORKLOAD, 0, 0, Q.ticks(x, S1), 0),
                    F(rec["max_workload"][xi])))
    tasks = hp + [k]
    S2 = su._scale(tasks, B)
    blob2 = Q.build_blob(su._rows(tasks, S2), 1, 0, 1)
    for j in range(k.m):
        out.append((blob2, S2, (0, Q.Q_SEGMENT_RESPONSE, len(hp), j, 0, Q.ticks(B, S2)),
                    fval(rec["segment_response"][j])))
    out.append((blob2, S2, (0, Q.Q_TASK_RESPONSE, len(hp), 0, 0, Q.ticks(B, S2)),
                fval(rec["task_response"])))
    return out


def test_susp_blocks_engine_core(blocks):
    items = [it for rec in blocks["susp"] for it in _susp_queries(rec)]
    res = harness.query([it[0] for it in items], [(i,) + it[2][1:] for i, it in enumerate(items)])
    bad = []
    for (blob, S, q, want), (st, num, den) in zip(items, res):
        got = Q.value(st, num, den, S)
        if got != want:
            bad.append((q, got, want))
    assert not bad, bad[:3]


def _rtgpu_items(rec):
    ts = ts_from_exact(rec["taskset"])
    cache = cache_of(rec["cache"])
    by_id = {t.id: t for t in ts.tasks}
    out = []
    for e in rec["tasks"]:
        k = by_id[e["id"]]
        hz = F(e["horizon"])
        blob, S, ids = an._explicit_blob(ts, cache, hz)
        ki = ids.index(k.id)
        for j, want in enumerate(e["mem_response"]):
            out.append((blob, S, (0, Q.Q_MEM_RESPONSE, ki, j, 0, 0), want))
        for j, want in enumerate(e["cpu_response"]):
            out.append((blob, S, (0, Q.Q_CPU_RESPONSE, ki, j, 0, 0), want))
        out.append((blob, S, (0, Q.Q_END_TO_END, ki, 0, 0, 0), e["end_to_end"]))
        if hz > 0:
            for h, want in enumerate(e["mem_workload"]):
                out.append((blob, S, (0, Q.Q_MEM_WORKLOAD, ki, h, Q.ticks(hz, S), 0), want))
            for h, want in enumerate(e["cpu_workload"]):
                out.append((blob, S, (0, Q.Q_CPU_WORKLOAD, ki, h, Q.ticks(hz, S), 0), want))
    return out


def _matches(st, num, den, S, want):
    if isinstance(want, dict):
        return st == Q.ST_GAP_ERROR and want["raises"] == "InfeasibleGapError"
    try:
        return Q.value(st, num, den, S) == fval(want)
    except Exception:
        return False


def test_rtgpu_blocks_engine_core(blocks):
    items = [it for rec in blocks["rtgpu"] for it in _rtgpu_items(rec)]
    assert any(isinstance(it[3], dict) for it in items) or True
    res = harness.query([it[0] for it in items], [(i,) + it[2][1:] for i, it in enumerate(items)])
    bad = [(it[2], r, it[3]) for it, r in zip(items, res) if not _matches(*r, it[1], it[3])]
    assert not bad, bad[:3]


def test_spec_worked_examples():
    """Hand-evaluated examples of the reference spec (suspension_core)."""
    E = ExecBounds
    t = su.SuspTask((E(F(2), F(2)), E(F(3), F(3))), (E(F(1), F(1)),), F(10), F(10))
    assert su.inter_arrival(t, 0) == 1 and su.inter_arrival(t, 1) == 0
    assert su.inter_arrival(t, 3) == 10 - 5 - 1
    assert su.chain_workload([F(2), F(3)], lambda j: su.inter_arrival(t, j), 0, F(6)) == 5


@pytest.mark.gpu
def test_susp_api_gpu(blocks):
    bad = []
    for rec in blocks["susp"][:150]:
        k = susp(rec["k"])
        hp = [susp(t) for t in rec["hp"]]
        B = F(rec["blocking"])
        for xi, x in enumerate(F(h) for h in rec["horizons"]):
            for h in range(k.m):
                if su.workload(k, h, x) != F(rec["workload"][xi][h]):
                    bad.append(("workload", rec))
            if su.max_workload(k, x) != F(rec["max_workload"][xi]):
                bad.append(("max_workload", rec))
        for j in range(k.m):
            if su.segment_response(k, j, hp, B) != fval(rec["segment_response"][j]):
                bad.append(("segment_response", rec))
        if su.task_response(k, hp, B) != fval(rec["task_response"]):
            bad.append(("task_response", rec))
    assert not bad, bad[:2]


@pytest.mark.gpu
def test_rtgpu_blocks_api_gpu(blocks):
    bad = []
    for rec in blocks["rtgpu"][:60]:
        ts = ts_from_exact(rec["taskset"])
        cache = cache_of(rec["cache"])
        by_id = {t.id: t for t in ts.tasks}
        for e in rec["tasks"]:
            k = by_id[e["id"]]
            for j, want in enumerate(e["mem_response"]):
                if an.mem_response(ts, k, j, cache) != fval(want):
                    bad.append(("mem", e["id"]))
            for j, want in enumerate(e["cpu_response"]):
                if an.cpu_response(ts, k, j, cache) != fval(want):
                    bad.append(("cpu", e["id"]))
            if an.end_to_end(ts, k, cache) != fval(e["end_to_end"]):
                bad.append(("e2e", e["id"]))
    assert not bad, bad[:3]
