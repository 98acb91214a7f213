"""Workbench drop-in: generate_taskset equals the reference's task sets,
acceptance_sweep equals the reference's CSV (golden files made by the
reference), plus the throughput formulas and config parsing."""
import json
import os
from fractions import Fraction as F

import pytest

from golden_io import GOLDEN_DIR, load_cases, ts_from_exact
from paper_2101_10463_b200 import workbench as wb
from paper_2101_10463_b200.model import (ExecBounds, GpuKernelModel, MemModel, PlatformConfig,
                                         SmAllocation, TaskSet, TaskSpec, validate_taskset)


def test_generate_taskset_equals_reference():
    cases = [c for c in load_cases() if c["kind"] == "gen"]
    for c in cases:
        p = c["params"]
        gp = wb.GenParams(n_tasks=p["n"], n_subtasks=p["m"], physical_sms=p["gn"],
                          target_utilization=F(p["u"]), mem_model=MemModel(p["mm"]),
                          lo_frac=F(p["lo"]))
        got = wb.generate_taskset(gp, c["seed"])
        want = ts_from_exact(c["taskset"])
        assert got == want, (c["seed"], p)
        assert validate_taskset(got) == []


def test_merge_memory_copies_matches_generator_one_copy():
    gp = wb.GenParams(n_tasks=4, n_subtasks=3)
    two = wb.generate_taskset(gp, 5)
    one = wb.generate_taskset(wb.GenParams(n_tasks=4, n_subtasks=3, mem_model=MemModel.ONE_COPY), 5)
    assert wb.merge_memory_copies(two) == one


def test_throughput_formulas():
    mk = lambda i, a: TaskSpec(f"t{i}", (ExecBounds.exact(1), ExecBounds.exact(1)),  # noqa: E731
                              (ExecBounds.exact(1), ExecBounds.exact(1)),
                              (GpuKernelModel(ExecBounds.exact(10), F(1), a),), F(100), F(100), i)
    alphas = [F(145, 100), F(17, 10), F(17, 10), F(18, 10), F(3, 2)]
    ts = TaskSet(tuple(mk(i + 1, a) for i, a in enumerate(alphas)), MemModel.TWO_COPY,
                 PlatformConfig(10))
    alloc = SmAllocation({f"t{i + 1}": 2 for i in range(5)})
    used = wb.throughput_improvement(ts, alloc, wb.ThroughputScope.USED_SMS)
    assert used == sum(F(1, 5) * (2 / a - 1) for a in alphas)
    whole = wb.throughput_improvement(ts, alloc, wb.ThroughputScope.WHOLE_GPU)
    assert whole == used / 2 and 0 <= whole <= 1


def test_sweep_config_parsing_errors():
    with pytest.raises(Exception):
        wb.sweep_config_from_dict({"utilizations": []})
    with pytest.raises(Exception):
        wb.gen_params_from_dict({"bogus": 1})


@pytest.mark.gpu
def test_acceptance_sweep_equals_reference_csv():
    with open(os.path.join(GOLDEN_DIR, "sweep_golden.json")) as fh:
        sweeps = json.load(fh)["sweeps"]
    for s in sweeps:
        rows = wb.acceptance_sweep(wb.sweep_config_from_dict(s["config"]))
        assert wb.sweep_to_csv(rows) == s["csv"]
