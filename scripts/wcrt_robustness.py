"""Executor robustness: measured WCRT / R_k and kernel span / GR_up over
many seeds and utilisations (default host models).  Writes a JSON list."""
import json
import sys

sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex  # noqa: E402

out = []
for seed in range(1, 9):
    for util in (2.5, 3.0, 4.0):
        r = ex.wcrt_experiment(n_tasks=4, m=3, horizon_us=1.0e6, seed=seed, utilization=util)
        rec = {"seed": seed, "util": util, "schedulable": r.schedulable,
               "max_wcrt_over_bound": round(r.max_ratio, 4),
               "max_kernel_span_over_lemma4": round(r.max_kernel_ratio, 4),
               "all_within_bound": r.all_within_bound, "allocation": r.allocation}
        out.append(rec)
        print(json.dumps(rec), flush=True)
ok = [x for x in out if x["schedulable"]]
print(json.dumps({"runs": len(out), "schedulable": len(ok),
                  "violations": sum(not x["all_within_bound"] for x in ok),
                  "worst_wcrt_ratio": max(x["max_wcrt_over_bound"] for x in ok),
                  "worst_kernel_ratio": max(x["max_kernel_span_over_lemma4"] for x in ok)}))
