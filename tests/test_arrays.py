"""The bulk array path (paper_2101_10463_b200/arrays.py).

CPU: pack_arrays writes word for word what the TaskSet packer writes for the
same sets (TaskArrays.taskset) -- int64 form against pack_tasksets_py,
compact form against tests/blobtools.compact -- including equal priorities,
CPU-only tasks, reducible interleave ratios and per-set SM counts.
GPU: analyze_arrays' verdicts, allocations and exact end-to-end bounds equal
the oracle's (full lexicographic enumeration) on the same blobs, and the
object API's reports on a sample."""
from fractions import Fraction

import numpy as np
import pytest

from blobtools import compact
from paper_2101_10463_b200.arrays import TaskArrays, analyze_arrays, pack_arrays, pack_arrays_np
from paper_2101_10463_b200.model import MemModel
from paper_2101_10463_b200.pack import pack_tasksets_py


def random_arrays(S, n, m, mm=MemModel.TWO_COPY, seed=0, u=0.5, gn=10, ties=False, den=100):
    """Sets shaped like the reference generator's (workbench.py:101): segment
    lengths in the paper's ranges, periods from a per-task utilisation."""
    rng = np.random.default_rng(seed)
    p = 0 if m < 2 else (2 * m - 2 if mm is MemModel.TWO_COPY else m - 1)
    g = m - 1
    cpu_hi = rng.integers(1000, 20001, (S, n, m))
    mem_hi = rng.integers(250, 5001, (S, n, p))
    work_hi = rng.integers(1000, 20001, (S, n, g))
    lo = lambda x: (x * rng.uniform(0.5, 1.0, x.shape)).astype(np.int64)  # noqa: E731
    total = cpu_hi.sum(2) + mem_hi.sum(2) + work_hi.sum(2) // 4
    period = (total / (u / n) * rng.uniform(0.8, 1.2, (S, n))).astype(np.int64) + 1
    prio = rng.integers(0, 3, (S, n)) if ties else np.argsort(rng.random((S, n)), axis=1)
    return TaskArrays(deadline=period.copy(), period=period, priority=prio,
                      cpu_lo=lo(cpu_hi), cpu_hi=cpu_hi, mem_lo=lo(mem_hi), mem_hi=mem_hi,
                      work_lo=lo(work_hi), work_hi=work_hi, overhead=(work_hi * 3) // 25,
                      ratio_num=rng.choice([100, 120, 125, 150, 180], (S, n, g)), ratio_den=den,
                      physical_sms=rng.integers(gn // 2, gn + 1, S) if gn > 1 else gn, mem_model=mm)


CASES = [(8, 5, MemModel.TWO_COPY, False), (16, 9, MemModel.ONE_COPY, True), (3, 1, MemModel.TWO_COPY, True),
         (4, 2, MemModel.ONE_COPY, False)]


@pytest.mark.parametrize("n,m,mm,ties", CASES)
def test_pack_arrays_equals_taskset_packer(n, m, mm, ties):
    a = random_arrays(40, n, m, mm, seed=n * 31 + m, ties=ties)
    want = pack_tasksets_py([a.taskset(k) for k in range(40)])
    got = pack_arrays(a, compact=False)
    assert np.array_equal(got.blobs, want.blobs)
    assert np.array_equal(got.set_off, want.set_off) and np.array_equal(got.task_base, want.task_base)
    for k in range(40):
        assert tuple(f"t{i}" for i in got.order[k]) == tuple(t.id for t in want.metas[k].order)
        assert want.metas[k].time_scale == 1
    cb, co, ct = compact(want.blobs, want.set_off, want.task_base)
    gc = pack_arrays(a)
    assert gc.compact
    assert np.array_equal(gc.blobs, cb) and np.array_equal(gc.set_off, co)
    for c in (None, False):  # the numpy restatement writes the same words
        x, y = pack_arrays_np(a, c), pack_arrays(a, c)
        assert np.array_equal(x.blobs, y.blobs) and np.array_equal(x.order, y.order) and x.compact == y.compact


def test_native_pack_arrays_threads():
    a = random_arrays(40000, 4, 3, seed=9, ties=True)  # > 8192 sets: several threads
    x, y = pack_arrays_np(a), pack_arrays(a)
    assert np.array_equal(x.blobs, y.blobs) and np.array_equal(x.order, y.order)


@pytest.mark.parametrize("compact_form", [None, False])
def test_from_blobs_round_trip(compact_form):
    a = random_arrays(50, 6, 4, MemModel.ONE_COPY, seed=4, ties=True)
    pk = pack_arrays(a, compact=compact_form)
    b = TaskArrays.from_blobs(pk.blobs, pk.set_off)
    again = pack_arrays(b, compact=compact_form)
    assert np.array_equal(again.blobs, pk.blobs)
    for name in ("deadline", "period", "priority", "cpu_lo", "mem_hi", "work_lo", "overhead"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


def test_from_blobs_of_the_generator():
    """The native generator's compact blobs (the bench's sets) read back into
    arrays pack to the same words."""
    from paper_2101_10463_b200.workbench import GenParams, generate_blobs
    gp = GenParams(n_tasks=8, n_subtasks=5, target_utilization=Fraction(1, 2))
    b, so, tb = generate_blobs(gp, [f"g{i}" for i in range(200)], compact=True)
    a = TaskArrays.from_blobs(b, so)
    assert np.array_equal(pack_arrays(a, compact=True).blobs, b)


def test_pack_arrays_reduces_ratio_denominator():
    a = random_arrays(10, 4, 3, seed=3, den=1000)
    a.ratio_num = a.ratio_num * 10  # same ratios over 1000: A must come out as the reduced lcm
    want = pack_tasksets_py([a.taskset(k) for k in range(10)])
    assert np.array_equal(pack_arrays(a, compact=False).blobs, want.blobs)


def test_pack_arrays_int64_when_values_exceed_int32():
    a = random_arrays(4, 3, 3, seed=5)
    a.cpu_hi[0, 0, 0] = 1 << 40
    assert not pack_arrays(a).compact
    with pytest.raises(ValueError):
        pack_arrays(a, compact=True)


def test_pack_arrays_rejects_bad_shapes():
    a = random_arrays(4, 3, 3)
    a.mem_lo = a.mem_lo[:, :, :1]
    with pytest.raises(ValueError, match="mem_lo"):
        pack_arrays(a)
    b = random_arrays(2, 65, 2)
    with pytest.raises(ValueError, match="tasks per set"):
        pack_arrays(b)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,mm,ties", CASES)
@pytest.mark.parametrize("bounds", [False, True])
def test_analyze_arrays_matches_oracle(n, m, mm, ties, bounds):
    from oracle import oracle
    a = random_arrays(300, n, m, mm, seed=7 * n + m, ties=ties)
    rep = analyze_arrays(a, bounds=bounds)
    pk = pack_arrays(a, compact=False)
    o = oracle.analyze_batch(pk.blobs, pk.set_off, pk.task_base, method=0, flags=1 if bounds else 0,
                             budget=0, threads=8, detail=False)
    assert np.array_equal(rep.status, o["status"])
    S = pk.n_sets
    ovsm = np.asarray(o["vsm"]).reshape(S, n)
    inv = np.argsort(pk.order, axis=1)
    assert np.array_equal(rep.vsm, np.take_along_axis(ovsm, inv, axis=1))
    if bounds:
        onum = np.take_along_axis(np.asarray(o["e2e_num"]).reshape(S, n), inv, axis=1)
        oden = np.take_along_axis(np.asarray(o["den"]).reshape(S, n), inv, axis=1)
        for s in range(S):
            for i in range(n):
                x, y = int(onum[s, i]), int(rep.e2e_num[s, i])
                if x < 0 or y < 0:
                    assert x == y, (s, i)
                else:
                    assert Fraction(x, int(oden[s, i])) == rep.end_to_end(s, i), (s, i)


@pytest.mark.gpu
def test_analyze_arrays_matches_object_api():
    from paper_2101_10463_b200 import analyze_rtgpu
    a = random_arrays(60, 8, 5, seed=11)
    rep = analyze_arrays(a, bounds=True)
    for k in range(60):
        r = analyze_rtgpu(a.taskset(k))
        assert bool(rep.schedulable[k]) == r.schedulable
        if r.allocation is not None:
            for i in range(8):
                assert rep.vsm[k, i] == r.allocation.virtual_sms(f"t{i}"), (k, i)
        for i in range(8):
            if f"t{i}" in r.per_task:
                assert rep.end_to_end(k, i) == r.per_task[f"t{i}"].end_to_end_up, (k, i)


def test_empty_batch():
    a = random_arrays(0, 4, 3)
    assert pack_arrays(a).n_sets == 0
    rep = analyze_arrays(a, bounds=True)
    assert rep.status.shape == (0,) and rep.vsm.shape == (0, 4) and rep.e2e_num.shape == (0, 4)
