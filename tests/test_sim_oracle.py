"""Pin the simulator oracle (oracle/sim_oracle.py) against traces produced by
the reference's own simulate() (tests/golden/sim_golden.json): every event in
order, the response / release dictionaries in insertion order, truncation."""
import pytest

from oracle import sim_oracle
from sim_common import (case_inputs, golden_events, golden_releases, golden_responses,
                        golden_truncated, jsonl, sha, sim_cases)

CASES = sim_cases()


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_oracle_trace_matches_reference(ci):
    c = CASES[ci]
    ts, alloc, horizon, seed, uniform = case_inputs(c)
    ev, resp, rels, trunc = sim_oracle.simulate(ts, alloc, horizon, seed, uniform)
    assert len(ev) == c["trace"]["n_events"]
    want = golden_events(c)
    if want is not None:
        assert ev == want
    assert sha(jsonl(ev)) == c["trace"]["jsonl_sha256"]
    assert [(t, j, r) for (t, j), r in resp.items()] == golden_responses(c)
    assert [(t, j, r) for (t, j), r in rels.items()] == golden_releases(c)
    assert trunc == golden_truncated(c)


def test_golden_covers_the_interesting_cases():
    kinds = {e[5] for c in CASES if c["trace"]["events"] for e in c["trace"]["events"]}
    assert {"release", "start", "preempt", "resume", "finish", "deadline-miss"} <= kinds
    assert any(c["trace"]["truncated"] for c in CASES)
    assert any(c["policy"] == "uniform" and isinstance(c["seed"], str) for c in CASES)
    assert any(c.get("violations_tight") for c in CASES)
