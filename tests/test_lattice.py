"""The lattice path (csrc/lattice.cuh: per-task scales, fixed points on the
lattice base + Z) checked on the CPU through the test-only sequential
harness: against the reference's own reports (golden, re-packed into the
compact blob form the path reads) and against the oracle on generated sets,
from 10 SMs up to BASELINE's 148-SM shapes."""
import os
import sys
from fractions import Fraction

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402

from golden_io import load_cases, ts_from_exact  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.pack import pack_tasksets  # noqa: E402

GREEDY = 0x100
ESCALATE = 99
HDR, TW = 8, 8


def compact(blobs, set_off, task_base):
    """Test helper: int64 blobs -> the compact form (int32 segment areas,
    header word 7 = 1) wherever every segment value fits int32."""
    words, offs = [], [0]
    for s in range(len(set_off) - 1):
        b = [int(x) for x in blobs[set_off[s]:set_off[s + 1]]]
        n = b[0]
        base = HDR + TW * n
        seg = b[base:]
        if b[7] == 0 and all(-2**31 <= v < 2**31 for v in seg):
            recs = b[HDR:base]
            for i in range(n):
                recs[TW * i + 5] = 2 * base + (recs[TW * i + 5] - base)  # int32 element offset
            if len(seg) % 2:
                seg = seg + [0]
            packed = np.asarray(seg, np.int32).view(np.int64).tolist()
            b = b[:HDR] + recs + packed
            b[7] = 1
            b[4] = len(b)
        words += b
        offs.append(len(words))
    return np.asarray(words, np.int64), np.asarray(offs, np.int64), np.asarray(task_base, np.int64)


def same_bounds(a, b, tasks):
    for t in tasks:
        x, y = int(a["e2e_num"][t]), int(b["e2e_num"][t])
        if x < 0 or y < 0:
            assert x == y, (t, x, y)
        else:
            assert Fraction(x, int(a["den"][t])) == Fraction(y, int(b["den"][t])), t


def decided_tasks(st, task_base):
    return np.concatenate([np.arange(task_base[s], task_base[s + 1]) for s in np.where(st)[0]]
                          + [np.zeros(0, np.int64)])


@pytest.fixture(scope="module")
def golden_compact():
    cases = load_cases()
    b = pack_tasksets([ts_from_exact(c["taskset"]) for c in cases])
    return compact(b.blobs, b.set_off, b.task_base)


@pytest.mark.parametrize("bounds", [False, True])
def test_lattice_matches_general_path_on_golden(golden_compact, bounds):
    """Every golden set the lattice path takes gets the general path's
    verdict, allocation and end-to-end bounds (the general path is pinned to
    the reference's reports in test_engine_logic)."""
    b, so, tb = golden_compact
    lat = harness.lattice_batch(b, so, tb, bounds=bounds)
    gen = harness.analyze_batch(b, so, tb, flags=1 if bounds else 0, detail=False)
    took = lat["status"] != ESCALATE
    assert took.sum() > 120, took.sum()  # 224 of the 398 cases are inputs the reference rejects
    assert np.array_equal(lat["status"][took], gen["status"][took])
    t = decided_tasks(took, tb)
    sched = decided_tasks(took & (gen["status"] == 1), tb)
    assert np.array_equal(lat["vsm"][sched], gen["vsm"][sched])
    if bounds:
        same_bounds(lat, gen, t)


def gen(n, m, gn, u, count, mm=0, lo=Fraction(1), seed="5"):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), mm,
                              gn, Fraction(12, 100), lo, compact=True)
    return _native.generate(gp, [f"{seed}:{u}:{i}" for i in range(count)])


@pytest.mark.parametrize("n,m,gn,u,mm,lo,count,greedy", [
    (8, 5, 10, "1/2", 0, 1, 300, False),
    (8, 5, 10, "4/5", 1, "7/10", 300, False),
    (5, 3, 14, "1", 0, "7/10", 300, False),
    (16, 9, 148, "1/5", 0, 1, 120, True),
    (16, 9, 148, "2/5", 1, "7/10", 120, True),
    (16, 5, 48, "3/10", 0, "1/2", 150, True),
    (64, 5, 148, "3/10", 0, 1, 12, True),
    (32, 9, 148, "1/5", 1, 1, 12, True),
])
@pytest.mark.parametrize("bounds", [False, True])
def test_lattice_matches_oracle(n, m, gn, u, mm, lo, count, greedy, bounds):
    b, so, tb = gen(n, m, gn, u, count, mm, Fraction(lo))
    lat = harness.lattice_batch(b, so, tb, bounds=bounds)
    o = oracle.analyze_batch(b, so, tb, method=0, flags=(GREEDY if greedy else 0) | int(bounds),
                             threads=8, detail=False)
    took = lat["status"] != ESCALATE
    assert took.mean() > 0.95
    assert np.array_equal(lat["status"][took], o["status"][took])
    assert np.array_equal(lat["vsm"][decided_tasks(took, tb)], o["vsm"][decided_tasks(took, tb)])
    if bounds:
        same_bounds(lat, o, decided_tasks(took, tb))
