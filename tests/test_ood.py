"""Inputs validate_taskset rejects but the reference's analyze() takes --
deadline beyond the period (D > T), lower bound above upper bound (lo > hi)
and tasks without segments (m = 0) -- give the reference's reports
(tests/golden/ood_golden.json, made by tests/golden/make_golden_ood.py
running the reference), all three methods: through the engine core on the
CPU harness and through the product API on the GPU."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness"))
import harness  # noqa: E402

from golden_io import load_cases, ts_from_exact  # noqa: E402
from paper_2101_10463_b200.model import AnalysisMethod, report_to_dict  # noqa: E402
from paper_2101_10463_b200.pack import INVALID, RawResults, pack_tasksets, unpack_report  # noqa: E402

METHODS = [AnalysisMethod.RTGPU, AnalysisMethod.SELF_SUSPENSION, AnalysisMethod.BUSY_WAITING]


@pytest.fixture(scope="module")
def ood():
    cases = load_cases("ood_golden.json")
    return cases, pack_tasksets([ts_from_exact(c["taskset"]) for c in cases])


@pytest.mark.parametrize("mi", [0, 1, 2])
def test_engine_core_matches_reference_out_of_domain(ood, mi):
    cases, batch = ood
    method = METHODS[mi]
    out = harness.analyze_batch(batch.blobs, batch.set_off, batch.task_base, flags=2, method=mi)
    res = RawResults(out["status"], out["evals"], out["vsm"], out["e2e_num"], out["den"], out["detail"])
    bad = []
    for s, c in enumerate(cases):
        want = c[method.value]
        if "raises" in want:
            if res.status[s] != INVALID:
                bad.append((s, c["kind"]))
            continue
        if report_to_dict(unpack_report(batch, res, s, method)) != want:
            bad.append((s, c["kind"]))
    assert not bad, bad[:8]


@pytest.mark.gpu
@pytest.mark.parametrize("mi", [0, 1, 2])
def test_gpu_matches_reference_out_of_domain(ood, mi):
    from paper_2101_10463_b200.analysis import analyze
    cases, _ = ood
    method = METHODS[mi]
    bad = []
    for s, c in enumerate(cases):
        want = c[method.value]
        try:
            got = report_to_dict(analyze(ts_from_exact(c["taskset"]), method))
        except ValueError:
            got = {"raises": "ValueError"}
        if ("raises" in want) != ("raises" in got) or ("raises" not in want and got != want):
            bad.append((s, c["kind"]))
    assert not bad, bad[:8]
