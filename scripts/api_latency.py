"""Drop-in API latency: analyze_rtgpu on one task set, analyze_batch on 1k."""
import sys
import time
from fractions import Fraction

sys.path.insert(0, ".")
from paper_2101_10463_b200 import analyze_batch, analyze_rtgpu, simulate, SimConfig  # noqa: E402
from paper_2101_10463_b200.workbench import GenParams, generate_taskset  # noqa: E402

gp = GenParams(n_tasks=8, n_subtasks=5, physical_sms=10, target_utilization=Fraction(1, 2))
sets = [generate_taskset(gp, f"lat:{i}") for i in range(1000)]
analyze_rtgpu(sets[0])
t = time.perf_counter()
for s in sets[:100]:
    analyze_rtgpu(s)
print(f"analyze_rtgpu: {(time.perf_counter() - t) / 100 * 1e3:.2f} ms per call")
analyze_batch(sets[:10])
t = time.perf_counter()
reps = analyze_batch(sets)
print(f"analyze_batch(1000): {(time.perf_counter() - t) * 1e3:.1f} ms")
acc = [(s, r) for s, r in zip(sets, reps) if r.schedulable][:20]
t = time.perf_counter()
for s, r in acc:
    simulate(s, r.allocation, SimConfig(horizon=Fraction(2) * max(x.period for x in s.tasks)))
print(f"simulate (2 x max period): {(time.perf_counter() - t) / len(acc) * 1e3:.2f} ms per call")
