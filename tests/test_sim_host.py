"""Host side of the GPU simulator: packing (exact time scale, release counts,
event capacity), Python-identical seeding of the Mersenne Twister, error
behaviour, and no CPU fallback."""
import random
from fractions import Fraction

import pytest

from paper_2101_10463_b200 import _native
from paper_2101_10463_b200.simulator import (LengthPolicy, SimConfig, _seed_key,
                                             pack_simulation)
from sim_common import case_inputs, error_cases, sim_cases

REFERENCE_ALL = {  # gpusched.__all__ (reference __init__.py)
    "AnalysisMethod", "AnalysisReport", "ExecBounds", "GenParams", "GpuKernelModel",
    "LengthPolicy", "MemModel", "PlatformConfig", "SimConfig", "SimTrace", "SmAllocation",
    "SuspTask", "SweepConfig", "TaskReport", "TaskSet", "TaskSpec", "TasksetFormatError",
    "ThroughputScope", "acceptance_sweep", "analyze", "analyze_busy_waiting_baseline",
    "analyze_rtgpu", "analyze_self_suspension_baseline", "check_against_analysis",
    "cpu_response", "end_to_end", "feasible_allocations", "generate_taskset",
    "gpu_response_bounds", "kernel_time", "load_report", "load_taskset", "max_workload",
    "mem_response", "merge_memory_copies", "save_report", "save_taskset", "segment_response",
    "simulate", "sweep_to_csv", "task_response", "throughput_improvement", "validate_taskset",
    "workload"}


def test_public_api_covers_reference():
    import paper_2101_10463_b200 as p
    assert REFERENCE_ALL <= set(p.__all__)
    for name in p.__all__:
        assert hasattr(p, name), name


def _mt_from_key(key):
    """MT19937 init_by_array (the algorithm CPython's random.seed uses)."""
    mt = [0] * 624
    mt[0] = 19650218
    for i in range(1, 624):
        mt[i] = (1812433253 * (mt[i - 1] ^ (mt[i - 1] >> 30)) + i) & 0xFFFFFFFF
    i, j = 1, 0
    for _ in range(max(624, len(key))):
        mt[i] = ((mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525)) + key[j] + j) & 0xFFFFFFFF
        i, j = i + 1, j + 1
        if i >= 624:
            mt[0], i = mt[623], 1
        if j >= len(key):
            j = 0
    for _ in range(623):
        mt[i] = ((mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941)) - i) & 0xFFFFFFFF
        i += 1
        if i >= 624:
            mt[0], i = mt[623], 1
    mt[0] = 0x80000000
    return mt


@pytest.mark.parametrize("seed", [0, 1, -7, 12345, 2 ** 40 + 3, 3 ** 70, "abc", "", b"xy",
                                  2.5])
def test_seed_key_matches_python_random(seed):
    state = random.Random(seed).getstate()[1][:624]
    assert tuple(_mt_from_key(_seed_key(seed))) == state


@pytest.mark.parametrize("ci", range(0, len(sim_cases()), 5))
def test_pack_scales_exactly(ci):
    c = sim_cases()[ci]
    ts, alloc, horizon, seed, uniform = case_inputs(c)
    cfg = SimConfig(horizon=horizon, seed=seed,
                    length_policy=LengthPolicy.UNIFORM_RANDOM if uniform else LengthPolicy.WORST_CASE)
    pk = pack_simulation(ts, alloc, cfg)
    b = pk.blob
    H = horizon if horizon is not None else 20 * max(t.period for t in ts.tasks)
    assert Fraction(int(b[2]), pk.Q) == H
    assert pk.R == len(c["trace"]["releases"])
    assert pk.evcap >= c["trace"]["n_events"]
    for i, t in enumerate(pk.tasks):
        r = 16 + 8 * i
        assert Fraction(int(b[r + 1]), pk.Q) == t.period
        assert Fraction(int(b[r + 2]), pk.Q) == t.deadline


def test_errors_match_reference_on_host():
    """Allocation errors are raised while packing (before any device call)."""
    for c in error_cases():
        ts, alloc, _, _, _ = case_inputs(c)
        with pytest.raises(ValueError) as ei:
            pack_simulation(ts, alloc, SimConfig())
        assert [type(ei.value).__name__, str(ei.value)] == c["raises"]


@pytest.mark.skipif(_native.device_info()["n_devices"] > 0, reason="GPU present")
def test_simulate_has_no_cpu_fallback():
    from paper_2101_10463_b200.simulator import simulate
    c = sim_cases()[0]
    ts, alloc, horizon, seed, uniform = case_inputs(c)
    with pytest.raises(_native.EngineUnavailable):
        simulate(ts, alloc, SimConfig())
