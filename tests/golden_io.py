"""Loading of the golden fixtures (tests/golden/*.json) into package types."""
from __future__ import annotations

import json
import os
from fractions import Fraction

from paper_2101_10463_b200.model import (
    ExecBounds,
    GpuKernelModel,
    MemModel,
    PlatformConfig,
    TaskSet,
    TaskSpec,
)

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def ts_from_exact(d: dict) -> TaskSet:
    F = Fraction
    tasks = []
    for t in d["tasks"]:
        tasks.append(TaskSpec(
            id=t["id"], priority=t["priority"], deadline=F(t["deadline"]),
            period=F(t["period"]),
            cpu_segments=tuple(ExecBounds(F(a), F(b)) for a, b in t["cpu"]),
            mem_segments=tuple(ExecBounds(F(a), F(b)) for a, b in t["mem"]),
            gpu_segments=tuple(GpuKernelModel(ExecBounds(F(a), F(b)), F(o), F(r))
                               for a, b, o, r in t["gpu"])))
    return TaskSet(tuple(tasks), MemModel(d["mem_model"]),
                   PlatformConfig(d["physical_sms"], F(d["launch_overhead_frac"])))


def load_cases(name: str = "rtgpu_golden.json") -> list:
    with open(os.path.join(GOLDEN_DIR, name)) as fh:
        return json.load(fh)["cases"]
