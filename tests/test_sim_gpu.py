"""GPU simulator (csrc/simulator.cu) against the reference's own traces and
against the oracle on fresh random task sets.  Bit-exact: every event, time
and list must be identical (times are exact rationals)."""
import dataclasses
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import sim_oracle
from sim_common import (case_inputs, error_cases, golden_events, golden_releases,
                        golden_responses, golden_truncated, jsonl, sha, sim_cases)

pytestmark = pytest.mark.gpu

CASES = sim_cases()


def _cfg(horizon, seed, uniform):
    from paper_2101_10463_b200.simulator import LengthPolicy, SimConfig
    return SimConfig(horizon=horizon, seed=seed,
                     length_policy=LengthPolicy.UNIFORM_RANDOM if uniform
                     else LengthPolicy.WORST_CASE)


def _tuples(trace):
    return [(e.time, e.task, e.job, e.kind, e.segment, e.action) for e in trace.events]


@pytest.fixture(scope="module")
def gpu_traces():
    """All golden cases in one batched launch (plus the drop-in per case below)."""
    from paper_2101_10463_b200.simulator import simulate_batch
    items, cfgs = [], []
    for c in CASES:
        ts, alloc, horizon, seed, uniform = case_inputs(c)
        items.append((ts, alloc))
        cfgs.append(_cfg(horizon, seed, uniform))
    b = simulate_batch(items, cfgs, events=True)
    return [b.trace(s) for s in range(len(CASES))]


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_batch_trace_matches_reference(gpu_traces, ci):
    c, tr = CASES[ci], gpu_traces[ci]
    assert len(tr.events) == c["trace"]["n_events"]
    want = golden_events(c)
    if want is not None:
        assert _tuples(tr) == want
    assert sha(tr.to_jsonl()) == c["trace"]["jsonl_sha256"]
    assert [(t, j, r) for (t, j), r in tr.responses.items()] == golden_responses(c)
    assert [(t, j, r) for (t, j), r in tr.releases.items()] == golden_releases(c)
    assert tr.truncated == golden_truncated(c)


def test_small_record_pool_reruns_overloaded_sets(gpu_traces):
    """A 2-record pool overflows on most sets; those are re-run with one
    record per release point and the merged traces are unchanged."""
    from paper_2101_10463_b200.simulator import simulate_batch
    items, cfgs = [], []
    for c in CASES:
        ts, alloc, horizon, seed, uniform = case_inputs(c)
        items.append((ts, alloc))
        cfgs.append(_cfg(horizon, seed, uniform))
    b = simulate_batch(items, cfgs, events=True, pool=2)
    for s, tr in enumerate(gpu_traces):
        assert b.trace(s).to_jsonl() == tr.to_jsonl()
        assert b.trace(s).truncated == tr.truncated


def test_device_resident_batch_matches_host_path(gpu_traces):
    from paper_2101_10463_b200.simulator import DeviceSimBatch, pack_simulation
    packs = []
    for c in CASES[:12]:
        ts, alloc, horizon, seed, uniform = case_inputs(c)
        packs.append(pack_simulation(ts, alloc, _cfg(horizon, seed, uniform), 0))
    d = DeviceSimBatch(packs, events=True)
    d.run()
    h = d.to_host()
    for s in range(len(packs)):
        assert h.trace(s).to_jsonl() == gpu_traces[s].to_jsonl()


@pytest.mark.parametrize("ci", [0, 5, 11, 20, len(CASES) - 1])
def test_dropin_simulate_and_check(ci):
    from paper_2101_10463_b200.model import report_from_dict
    from paper_2101_10463_b200.simulator import check_against_analysis, simulate
    c = CASES[ci]
    ts, alloc, horizon, seed, uniform = case_inputs(c)
    tr = simulate(ts, alloc, _cfg(horizon, seed, uniform))
    assert sha(tr.to_jsonl()) == c["trace"]["jsonl_sha256"]
    tr2 = simulate(ts, alloc, _cfg(horizon, seed, uniform))
    assert tr2.to_jsonl() == tr.to_jsonl()  # deterministic given the seed
    if "report" in c:
        assert check_against_analysis(tr, report_from_dict(c["report"])) == c["violations"]


def _tight(rep):
    from paper_2101_10463_b200.model import ExecBounds
    q = Fraction(3, 4)
    return dataclasses.replace(rep, per_task={
        tid: dataclasses.replace(
            r, mem_r_up=tuple(None if x is None else x * q for x in r.mem_r_up),
            cpu_r_up=tuple(None if x is None else x * q for x in r.cpu_r_up),
            gpu_r=tuple(ExecBounds(b.lo * q, b.hi * q) for b in r.gpu_r),
            end_to_end_up=None if r.end_to_end_up is None else r.end_to_end_up * q)
        for tid, r in rep.per_task.items()})


def test_check_against_analysis_matches_reference(gpu_traces):
    from paper_2101_10463_b200.model import report_from_dict
    from paper_2101_10463_b200.simulator import check_against_analysis
    n = 0
    for c, tr in zip(CASES, gpu_traces):
        if "report" not in c:
            continue
        rep = report_from_dict(c["report"])
        assert check_against_analysis(tr, rep) == c["violations"]
        assert check_against_analysis(tr, _tight(rep)) == c["violations_tight"]
        n += 1
    assert n >= 5


def test_errors_match_reference():
    from paper_2101_10463_b200.simulator import SimConfig, simulate
    for c in error_cases():
        ts, alloc, _, _, _ = case_inputs(c)
        with pytest.raises(ValueError) as ei:
            simulate(ts, alloc, SimConfig())
        assert [type(ei.value).__name__, str(ei.value)] == c["raises"]


def _random_items(n_sets, seed):
    """Random generated task sets with a feasible allocation each."""
    from paper_2101_10463_b200.analysis import analyze_batch
    from paper_2101_10463_b200.model import MemModel, SmAllocation
    from paper_2101_10463_b200.workbench import GenParams, generate_taskset
    rng = random.Random(seed)
    sets = []
    for i in range(n_sets):
        gp = GenParams(n_tasks=rng.randint(2, 6), n_subtasks=rng.randint(1, 4),
                       physical_sms=rng.randint(6, 16),
                       target_utilization=Fraction(rng.randint(2, 30), 10),
                       mem_model=rng.choice([MemModel.TWO_COPY, MemModel.ONE_COPY]),
                       lo_frac=Fraction(rng.randint(3, 10), 10))
        sets.append(generate_taskset(gp, 10_000 * seed + i))
    reps = analyze_batch(sets)
    items = []
    for ts, rep in zip(sets, reps):
        if rep.schedulable:
            alloc = rep.allocation
        else:
            alloc = SmAllocation({t.id: (2 if t.gpu_segments else 0) for t in ts.tasks})
            if alloc.total_physical() > ts.platform.physical_sms:
                continue
        items.append((ts, alloc, rep))
    return items


@pytest.mark.parametrize("uniform", [False, True])
def test_batch_matches_oracle_on_random_sets(uniform):
    """Many fresh simulations in one launch: traces equal the oracle's, and the
    device-side per-segment maxima give check_against_analysis's verdict."""
    from paper_2101_10463_b200.simulator import check_against_analysis, simulate_batch
    items = _random_items(48, 3 if uniform else 4)
    cfgs = [_cfg(None, 17 * s + 1, uniform) for s in range(len(items))]
    b = simulate_batch([(ts, al) for ts, al, _ in items], cfgs, events=True)
    checked = 0
    for s, ((ts, al, rep), cfg) in enumerate(zip(items, cfgs)):
        tr = b.trace(s)
        ev, resp, rels, trunc = sim_oracle.simulate(ts, al, None, cfg.seed, uniform)
        assert _tuples(tr) == ev, s
        assert list(tr.responses.items()) == list(resp.items())
        assert tr.truncated == trunc
        if rep.schedulable:
            for r in (rep, _tight(rep)):
                assert (not b.check(s, r)) == (not check_against_analysis(tr, r))
            checked += 1
    assert checked >= 5


def test_worst_case_soundness_on_accepted_sets():
    """SPEC simulator property: analysis-accepted sets under worst-case
    lengths show no deadline miss and no response above its bound."""
    from paper_2101_10463_b200.simulator import SimConfig, simulate_batch
    items = [x for x in _random_items(96, 9) if x[2].schedulable]
    b = simulate_batch([(ts, rep.allocation) for ts, _, rep in items], SimConfig())
    assert int(b.misses.sum()) == 0
    for s, (_, _, rep) in enumerate(items):
        assert b.check(s, rep) == []
