"""Executor robustness: measured WCRT / R_k and kernel span / GR_up over
many seeds and load levels.  One JSON line per run, then a summary line.

    python scripts/wcrt_robustness.py [--wide] [--seeds N] [--horizon-s S]

--wide: partitions of several to tens of SMs (wcrt_experiment width mode,
three target-width ranges as the load levels); default: the utilisation
mode (2.5 / 3.0 / 4.0)."""
import argparse
import json
import sys

sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--wide", action="store_true")
ap.add_argument("--seeds", type=int, default=8)
ap.add_argument("--horizon-s", type=float, default=1.0)
ap.add_argument("--seed-list", default="", help="comma-separated seeds (overrides --seeds)")
args = ap.parse_args()
levels = [(8, 16), (16, 28), (28, 40)] if args.wide else [2.5, 3.0, 4.0]
seeds = [int(x) for x in args.seed_list.split(",") if x] or list(range(1, args.seeds + 1))
out = []
for seed in seeds:
    for lv in levels:
        kw = dict(width=lv) if args.wide else dict(utilization=lv)
        try:
            r = ex.wcrt_experiment(n_tasks=4, m=3, horizon_us=args.horizon_s * 1e6, seed=seed, **kw)
        except ValueError as exc:  # e.g. the analysis' partitions exceed the GPU's SMs
            print(json.dumps({"seed": seed, "level": lv, "skipped": str(exc)}), flush=True)
            continue
        rec = {"seed": seed, "level": lv, "schedulable": r.schedulable,
               "max_wcrt_over_bound": round(r.max_ratio, 4),
               "max_kernel_span_over_lemma4": round(r.max_kernel_ratio, 4),
               "all_within_bound": r.all_within_bound, "kernels_within_bound": r.kernels_within_bound,
               "allocation_vsm": r.allocation, "sms_used": r.sms_used,
               "jobs": [t["jobs"] for t in r.tasks], "note": r.note,
               "blocks_per_launch_vs_2g": [(t["blocks_per_launch"], 2 * t["sms"]) for t in r.tasks],
               "kernel_span_vs_gr_up": [t["kernel_span_us_vs_gr_up"] for t in r.tasks],
               "worst_launch": [t["worst_launch"] for t in r.tasks],
               "smsp_max_warps": max((t["smsp_max_warps"] for t in r.tasks), default=0),
               "launch_ratio_pcts": r.launch_ratio_pcts, "overruns": r.overruns,
               "stalls": r.stalls, "max_kernel_ratio_net_of_stalls": r.max_kernel_ratio_net,
               "kernels_within_bound_net_of_stalls": r.kernels_within_bound_net}
        out.append(rec)
        print(json.dumps(rec), flush=True)
ok = [x for x in out if x["schedulable"]]
print(json.dumps({"summary": True, "runs": len(out), "schedulable": len(ok),
                  "jobs_over_bound_runs": sum(not x["all_within_bound"] for x in ok),
                  "kernel_overrun_runs": sum(not x["kernels_within_bound"] for x in ok),
                  "kernel_overrun_runs_net_of_stalls": sum(x["kernels_within_bound_net_of_stalls"] is False
                                                           for x in ok),
                  "runs_with_sentinel": sum(x["kernels_within_bound_net_of_stalls"] is not None for x in ok),
                  "worst_kernel_ratio_net_of_stalls": max((x["max_kernel_ratio_net_of_stalls"] or 0 for x in ok),
                                                          default=None),
                  "worst_wcrt_ratio": max((x["max_wcrt_over_bound"] for x in ok), default=None),
                  "worst_kernel_ratio": max((x["max_kernel_span_over_lemma4"] for x in ok), default=None),
                  "min_sms_used": min((x["sms_used"] for x in ok), default=None),
                  "max_sms_used": max((x["sms_used"] for x in ok), default=None)}), flush=True)
