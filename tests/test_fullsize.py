"""Parity at BASELINE's full shapes (16 tasks x 9 segments and 64 tasks on
148 SMs), where the reference's lexicographic enumeration cannot finish.

The checker is the oracle's greedy mode: it chooses, task by task, the
smallest SM count at which the oracle's *faithful* per-allocation evaluation
(literal walks, literal fixed-point iteration, exact 128-bit rationals)
passes.  It is first shown equal to the oracle's full enumeration on sets
small enough to enumerate (the dominance argument of DESIGN.md section 3),
then compared with the engine at full size."""
import os
import sys
from fractions import Fraction

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2101_10463_b200 import _native  # noqa: E402

GREEDY = 0x100


def gen(n, m, gn, u, count, mm=0, seed0=0, compact=False):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), mm,
                              gn, Fraction(12, 100), Fraction(1), compact=compact)
    return _native.generate(gp, list(range(seed0, seed0 + count)))


def same(a, b, sched_only=False):
    assert np.array_equal(a["status"], b["status"])
    assert np.array_equal(a["vsm"], b["vsm"])
    for i in range(len(a["e2e_num"])):
        x, y = int(a["e2e_num"][i]), int(b["e2e_num"][i])
        if x < 0 or y < 0:
            assert x == y
        else:
            assert Fraction(x, int(a["den"][i])) == Fraction(y, int(b["den"][i]))


@pytest.mark.parametrize("n,m,gn,u,mm", [(5, 3, 10, "1", 0), (6, 2, 20, "1", 1),
                                         (8, 5, 10, "1/2", 0), (4, 4, 6, "4/5", 1)])
def test_greedy_oracle_equals_full_enumeration(n, m, gn, u, mm):
    b, so, tb = gen(n, m, gn, u, 150, mm)
    full = oracle.analyze_batch(b, so, tb, flags=1, threads=8, detail=False)
    greedy = oracle.analyze_batch(b, so, tb, flags=1 | GREEDY, threads=8, detail=False)
    same(full, greedy)


@pytest.mark.parametrize("n,m,u,count", [(16, 9, "1/5", 24), (16, 9, "2/5", 24),
                                         (64, 5, "1", 4), (32, 9, "1/2", 6)])
def test_engine_core_full_size(n, m, u, count):
    b, so, tb = gen(n, m, 148, u, count)
    greedy = oracle.analyze_batch(b, so, tb, flags=1 | GREEDY, threads=8, detail=False)
    h = harness.analyze_batch(b, so, tb, flags=1, detail=False)
    same(greedy, h)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,u,count", [(16, 9, "1/10", 200), (16, 9, "1/5", 200),
                                         (16, 9, "2/5", 200), (16, 9, "1", 100),
                                         (64, 5, "1", 30), (64, 16, "2", 10)])
def test_gpu_full_size(n, m, u, count):
    from paper_2101_10463_b200.engine import DeviceBatch
    b, so, tb = gen(n, m, 148, u, count, seed0=77)
    greedy = oracle.analyze_batch(b, so, tb, flags=1 | GREEDY, threads=16, detail=False)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=1)
    g = out.to_host()
    same(greedy, {"status": g.status, "vsm": g.vsm, "e2e_num": g.e2e_num, "den": g.den})


def same_verdicts(ref, status, vsm, task_base):
    assert np.array_equal(ref["status"], status)
    sched = np.repeat(ref["status"] == 1, np.diff(task_base))
    assert np.array_equal(ref["vsm"][sched], vsm[sched])


@pytest.mark.parametrize("n,m,u,count", [(16, 9, "1/5", 30), (16, 9, "1", 30),
                                         (64, 5, "1", 6), (64, 5, "2", 6)])
def test_engine_core_full_size_verdicts(n, m, u, count):
    """Verdict runs on compact blobs at 148 SMs: the fast path takes the sets
    whose candidate counts stay small enough for its fixed scale, the
    general path the rest; both agree with the greedy oracle."""
    b, so, tb = gen(n, m, 148, u, count, compact=True)
    greedy = oracle.analyze_batch(b, so, tb, flags=1 | GREEDY, threads=8, detail=False)
    h = harness.analyze_batch(b, so, tb, flags=0, detail=False)
    same_verdicts(greedy, h["status"], h["vsm"], tb)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,u,count", [(16, 9, "1/5", 200), (16, 9, "1", 100),
                                         (64, 5, "1", 30), (64, 5, "2", 30)])
def test_gpu_full_size_verdicts(n, m, u, count):
    from paper_2101_10463_b200.engine import DeviceBatch, analyze_packed
    b, so, tb = gen(n, m, 148, u, count, seed0=91, compact=True)
    greedy = oracle.analyze_batch(b, so, tb, flags=1 | GREEDY, threads=16, detail=False)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=0)
    g = out.to_host()
    same_verdicts(greedy, g.status, g.vsm, tb)
    h = analyze_packed(b, so, tb, 0, 0)  # the streamed end-to-end path
    same_verdicts(greedy, h.status, h.vsm, tb)
