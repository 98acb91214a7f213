"""int32 task records (blob header word 7 = 2, include/rtgpu.h): the same task
sets as the compact form (word 7 = 1) with 4 int64 words per record instead
of 8.  The generator's two forms must carry identical sets, and every reader
(the oracle, the engine core on the CPU harness, the product on the GPU) must
give identical results on both."""
import os
import sys
from fractions import Fraction

import numpy as np
import pytest

from paper_2101_10463_b200 import _native
from paper_2101_10463_b200.arrays import TaskArrays

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402  (test harness: the engine core on the CPU)

GREEDY = 0x100  # the oracle's greedy mode (tests/test_fullsize.py): 148-SM sets in seconds


def gen(n, m, gn, u, count, rec32, mm=0):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), mm, gn,
                              Fraction(12, 100), Fraction(1), compact=True, rec32=rec32)
    return _native.generate(gp, [f"r32:{u}:{i}" for i in range(count)])


SHAPES = [(8, 5, 10, "3/10", 0), (8, 5, 10, "1/2", 1), (16, 9, 148, "1/5", 0), (5, 3, 6, "2/5", 0)]


@pytest.mark.parametrize("n,m,gn,u,mm", SHAPES)
def test_rec32_blobs_carry_the_same_sets(n, m, gn, u, mm):
    b1, so1, tb1 = gen(n, m, gn, u, 40, False, mm)
    b2, so2, tb2 = gen(n, m, gn, u, 40, True, mm)
    assert int(b2[7]) == 2 and int(b1[7]) == 1
    assert np.array_equal(tb1, tb2)
    w1, w2 = int(so1[1] - so1[0]), int(so2[1] - so2[0])
    assert w1 - w2 == 4 * n  # half of every record
    a1, a2 = TaskArrays.from_blobs(b1, so1), TaskArrays.from_blobs(b2, so2)
    for f in ("deadline", "period", "priority", "cpu_lo", "cpu_hi", "mem_lo", "mem_hi", "work_lo",
              "work_hi", "overhead", "ratio_num"):
        assert np.array_equal(getattr(a1, f), getattr(a2, f)), f


@pytest.mark.parametrize("n,m,gn,u,mm", SHAPES)
def test_rec32_oracle_and_core_match_compact(n, m, gn, u, mm):
    from oracle import oracle
    b1, so1, tb1 = gen(n, m, gn, u, 30, False, mm)
    b2, so2, tb2 = gen(n, m, gn, u, 30, True, mm)
    o1 = oracle.analyze_batch(b1, so1, tb1, method=0, flags=1 | GREEDY, threads=4, detail=False)
    o2 = oracle.analyze_batch(b2, so2, tb2, method=0, flags=1 | GREEDY, threads=4, detail=False)
    for k in ("status", "vsm", "e2e_num", "den"):
        assert np.array_equal(o1[k], o2[k]), k
    # the engine core (fast path, then the general stages) and the lattice path
    h2 = harness.analyze_batch(b2, so2, tb2, flags=0, detail=False)
    assert np.array_equal(h2["status"], o2["status"])
    assert np.array_equal(h2["vsm"], o2["vsm"])
    l1 = harness.lattice_batch(b1, so1, tb1, bounds=True)
    l2 = harness.lattice_batch(b2, so2, tb2, bounds=True)
    for k in ("status", "vsm", "e2e_num", "den"):
        assert np.array_equal(l1[k], l2[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,gn,u,mm", SHAPES)
@pytest.mark.parametrize("flags", [0, 1])
def test_rec32_gpu_matches_compact(n, m, gn, u, mm, flags):
    from paper_2101_10463_b200.engine import DeviceBatch
    res = []
    for rec32 in (False, True):
        b, so, tb = gen(n, m, gn, u, 300, rec32, mm)
        batch = DeviceBatch(b, so, tb, device="cuda:0")
        out = batch.alloc_results()
        batch.run(out, flags=flags)
        res.append(out.to_host())
    assert np.array_equal(res[0].status, res[1].status)
    assert np.array_equal(res[0].vsm, res[1].vsm)
    if flags:
        assert np.array_equal(res[0].e2e_num, res[1].e2e_num)
        assert np.array_equal(res[0].den, res[1].den)


@pytest.mark.gpu
def test_rec32_host_entry_matches_oracle():
    """rtgpu_analyze_host (the streamed end-to-end call) on int32-record blobs."""
    from oracle import oracle
    b, so, tb = gen(8, 5, 10, "2/5", 4000, True)
    got = _native.analyze_host(b, so, tb, 0, 0, 0, False)
    want = oracle.analyze_batch(b, so, tb, method=0, flags=GREEDY, threads=8, detail=False)
    assert np.array_equal(got["status"], want["status"])
    assert np.array_equal(got["vsm"], want["vsm"])
