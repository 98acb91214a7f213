"""The engine core (engine_core.cuh, the code the kernels run) checked on the
CPU through the test-only sequential harness: against the reference's own
reports (golden) in every arithmetic stage, and against the oracle on
generated sets.  The CUDA build is checked the same way in test_gpu_parity."""
import sys
import os
from fractions import Fraction

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402

from golden_io import load_cases, ts_from_exact  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.model import AnalysisMethod, report_to_dict  # noqa: E402
from paper_2101_10463_b200.pack import (INVALID, RawResults, pack_tasksets,  # noqa: E402
                                        unpack_report)


@pytest.fixture(scope="module")
def golden():
    cases = load_cases()
    return cases, pack_tasksets([ts_from_exact(c["taskset"]) for c in cases])


METHODS = [AnalysisMethod.RTGPU, AnalysisMethod.SELF_SUSPENSION, AnalysisMethod.BUSY_WAITING]


@pytest.mark.parametrize("stage", [0, 1, 2])
@pytest.mark.parametrize("mi", [0, 1, 2])
def test_engine_core_matches_reference_reports(golden, stage, mi):
    cases, batch = golden
    method = METHODS[mi]
    out = harness.analyze_batch(batch.blobs, batch.set_off, batch.task_base, flags=2,
                                first_stage=stage, method=mi)
    assert (out["stage"] == stage).all()
    res = RawResults(out["status"], out["evals"], out["vsm"], out["e2e_num"], out["den"],
                     out["detail"])
    bad = []
    for s, c in enumerate(cases):
        want = c[method.value]
        if "raises" in want:
            if res.status[s] != INVALID:
                bad.append(s)
            continue
        if report_to_dict(unpack_report(batch, res, s, method)) != want:
            bad.append(s)
    assert not bad, bad[:5]


def compare(o, h):
    assert np.array_equal(o["status"], h["status"])
    assert np.array_equal(o["vsm"], h["vsm"])
    for i in range(len(o["e2e_num"])):
        a, b = int(o["e2e_num"][i]), int(h["e2e_num"][i])
        if a < 0 or b < 0:
            assert a == b
        else:
            assert Fraction(a, int(o["den"][i])) == Fraction(b, int(h["den"][i]))


@pytest.mark.parametrize("mi", [0, 1, 2])
@pytest.mark.parametrize("n,m,gn,u,mm", [(8, 5, 10, "2/5", 0), (5, 5, 10, "3/5", 1),
                                         (4, 3, 6, "1", 0), (6, 2, 12, "4/5", 1)])
def test_engine_core_matches_oracle_generated(n, m, gn, u, mm, mi):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), mm,
                              gn, Fraction(12, 100), Fraction(1) if mm == 0 else Fraction(7, 10))
    b, so, tb = _native.generate(gp, list(range(120)))
    o = oracle.analyze_batch(b, so, tb, method=mi, flags=1, threads=8, detail=False)
    h = harness.analyze_batch(b, so, tb, method=mi, flags=1, detail=False)
    compare(o, h)


@pytest.mark.parametrize("n,m,gn,u,mm", [(8, 5, 10, "1/10", 0), (8, 5, 10, "2/5", 0),
                                         (8, 5, 10, "3/5", 1), (5, 3, 10, "1", 0),
                                         (6, 2, 20, "4/5", 0), (16, 9, 10, "1/5", 0)])
def test_verdict_fast_path_matches_oracle(n, m, gn, u, mm):
    """Verdict-only runs on compact (int32) blobs take the fast path
    (flags = 0); int64 blobs of the same sets go to the general path and
    give the same verdicts."""
    for compact in (True, False):
        gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u),
                                  mm, gn, Fraction(12, 100),
                                  Fraction(1) if mm == 0 else Fraction(7, 10), compact=compact)
        b, so, tb = _native.generate(gp, [f"3:{u}:{i}" for i in range(200)])
        o = oracle.analyze_batch(b, so, tb, flags=0, threads=8, detail=False)
        h = harness.analyze_batch(b, so, tb, flags=0, detail=False)
        if compact and gn <= 12:  # the fast path needs 2*A*lcm(1..GN) to fit FP64 exactly
            assert (h["stage"] == -1).mean() > 0.5
        if not compact:
            assert (h["stage"] >= 0).all()
        assert np.array_equal(o["status"], h["status"])
        sched = np.repeat(o["status"] == 1, n)
        assert np.array_equal(o["vsm"][sched], h["vsm"][sched])
