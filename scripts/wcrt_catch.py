"""Run the executor experiment until a kernel overruns its Lemma-4 bound,
then print that run's per-kernel detail (span, event time, SM clock, items)."""
import sys

sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex  # noqa: E402

for attempt in range(12):
    for seed, util in ((5, 2.5), (8, 4.0), (1, 4.0), (7, 3.0)):
        r = ex.wcrt_experiment(n_tasks=4, m=3, horizon_us=1.0e6, seed=seed, utilization=util)
        print(attempt, seed, util, round(r.max_ratio, 3), round(r.max_kernel_ratio, 3), flush=True)
        if r.max_kernel_ratio > 1.05:
            for t in r.tasks:
                print("   ", t["task"], t["sms"], t["kernel_span_us_vs_gr_up"], t["kernel_event_us"],
                      t["worst_launch"], "min_mhz", t["min_sm_mhz"], "jobs", t["jobs"])
            sys.exit(0)
