"""Parity that does not lean on the engine's own search argument.

The engine finds the lexicographically first schedulable allocation by a
greedy descent justified by monotonicity and dominance (DESIGN.md section
3); the oracle's greedy mode rests on the same argument.  Here the checker
is the oracle's full lexicographic enumeration (small platforms) or its
prefix-pruned enumeration (ORACLE_PREFIX, exact, uses only the prefix
property visible in analysis.py:156-217), on adversarial sets built around
the argument's boundary (tests/blobtools.py: wrap-around gaps within ticks
of zero at g_min, lo < hi, irregular copies, CPU-only tasks, equal
priorities), up to 48 SMs.  Undecided sets (enumeration budget) are not
counted.  CPU: the engine core through the sequential harness (general
path on int64 blobs, fast / lattice paths on compact blobs); GPU: the
product library, device path."""
import os
import sys
from fractions import Fraction

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402

from blobtools import adversarial, compact  # noqa: E402
from oracle import oracle  # noqa: E402

PREFIX = 0x200
UNDECIDED, ESCALATE = 2, 99

SHAPES = [  # n, m_max, GN, mem model, kwargs, oracle mode
    (5, 3, 8, 0, dict(u_total=0.5), "full"),
    (6, 4, 12, 1, dict(u_total=0.5, p_irreg=0.3), "full"),
    (4, 5, 10, 0, dict(u_total=0.8, p_tight=0.5), "full"),
    (6, 4, 16, 0, dict(u_total=0.5), "prefix"),
    (8, 5, 24, 1, dict(u_total=0.5), "prefix"),
    (8, 4, 32, 0, dict(u_total=0.4, p_irreg=0.2), "prefix"),
    (10, 4, 48, 0, dict(u_total=0.4), "prefix"),
]


def run_oracle(b, so, tb, mode, bounds):
    flags = (PREFIX if mode == "prefix" else 0) | (1 if bounds else 0)
    return oracle.analyze_batch(b, so, tb, method=0, flags=flags,
                                budget=100000 if mode == "prefix" else 0, threads=8, detail=False)


def check(o, e, tb, sel, bounds):
    sel = sel & (o["status"] != UNDECIDED)
    assert np.array_equal(o["status"][sel], np.asarray(e["status"])[sel])
    for s in np.where(sel)[0]:
        t0, t1 = tb[s], tb[s + 1]
        assert np.array_equal(o["vsm"][t0:t1], np.asarray(e["vsm"])[t0:t1]), s
        if bounds:
            for t in range(t0, t1):
                a, c = int(o["e2e_num"][t]), int(e["e2e_num"][t])
                if a < 0 or c < 0:
                    assert a == c, (s, t)
                else:
                    assert Fraction(a, int(o["den"][t])) == Fraction(c, int(e["den"][t])), (s, t)
    return int(sel.sum())


@pytest.mark.parametrize("n,m,gn,mm,kw,mode", SHAPES)
def test_engine_core_matches_enumeration_on_adversarial_sets(n, m, gn, mm, kw, mode):
    count = 120 if mode == "full" else 40
    b, so, tb = adversarial(7 + n * gn, count, n, m, gn, mm, **kw)
    bc, soc, tbc = compact(b, so, tb)
    for bounds in (False, True):
        o = run_oracle(b, so, tb, mode, bounds)
        assert (o["status"] != UNDECIDED).mean() > 0.5
        general = harness.analyze_batch(b, so, tb, flags=1 if bounds else 0, detail=False)
        decided = check(o, general, tb, np.ones(len(so) - 1, bool), bounds)
        fast = harness.analyze_batch(bc, soc, tbc, flags=1 if bounds else 0, detail=False)
        check(o, fast, tb, np.ones(len(so) - 1, bool), bounds)
        lat = harness.lattice_batch(bc, soc, tbc, bounds=bounds)
        took = lat["status"] != ESCALATE
        check(o, lat, tb, took, bounds)
        assert decided > 0


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,gn,mm,kw,mode", SHAPES)
def test_gpu_matches_enumeration_on_adversarial_sets(n, m, gn, mm, kw, mode):
    from paper_2101_10463_b200.engine import DeviceBatch
    from paper_2101_10463_b200.pack import F_BOUNDS
    count = 600 if mode == "full" else 120
    b, so, tb = adversarial(1000 + n * gn, count, n, m, gn, mm, **kw)
    for bounds in (False, True):
        o = run_oracle(b, so, tb, mode, bounds)
        for blobs in ((b, so, tb), compact(b, so, tb)):
            batch = DeviceBatch(*blobs)
            out = batch.alloc_results()
            batch.run(out, flags=F_BOUNDS if bounds else 0)
            h = out.to_host()
            e = {"status": h.status, "vsm": h.vsm, "e2e_num": h.e2e_num, "den": h.den}
            assert check(o, e, tb, np.ones(len(so) - 1, bool), bounds) > count // 2
