"""Executor run-path probe: kernel spans in rtgpu_exec_run under task mixes."""
import sys

sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex  # noqa: E402

parts = [[0], [1], [2], [3, 4]]


def mk(copies, cpu=100):
    return [ex.ExecTaskDef(cpu_us=[cpu] * 3, copy_bytes=[1 << 20] * (4 if copies else 0),
                           kernel_items=[1000, 1500], period_us=25000, deadline_us=25000)
            for _ in range(4)]


def show(tag, res, n):
    for i in range(n):
        r = res[i]
        print(tag, i, "jobs", r.jobs, "span", [round(r.seg_max_span_us[j], 1) for j in range(2)],
              "event", [round(r.seg_max_kernel_us[j], 1) for j in range(2)],
              "wall", [round(r.seg_max_wall_us[j], 1) for j in range(2)],
              "mhz", round(r.min_mhz), flush=True)


for tag, n, copies, bus in (("alone", 1, False, 1), ("4-nocopy", 4, False, 1),
                            ("4-copy-bus", 4, True, 1), ("4-copy-free", 4, True, 0),
                            ("alone-copy", 1, True, 1)):
    d = mk(copies)[:n]
    res = ex.run_tasks(d, parts[:n], 2048, 1.0e6, cpu_mode=0, bus_mode=bus)
    show(tag, res, n)
