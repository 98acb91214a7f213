"""Executor diagnostics on the GPU: measured WCRT vs bound per host
resource model (cpu_mode, bus_mode), with on-GPU kernel spans.
    python scripts/wcrt_modes.py [horizon_us]"""
import json
import sys

sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex  # noqa: E402

hz = float(sys.argv[1]) if len(sys.argv) > 1 else 1.5e6
out = []
for seed, util in [(1, 3.0), (3, 4.0), (3, 3.0)]:
    for cm, bm in [(0, 1), (1, 1)]:
        r = ex.wcrt_experiment(n_tasks=4, m=3, horizon_us=hz, seed=seed, utilization=util,
                               cpu_mode=cm, bus_mode=bm)
        rec = {"seed": seed, "util": util, "cpu_mode": cm, "bus_mode": bm,
               "applied": [r.cpu_mode, r.bus_mode], "max_ratio": round(r.max_ratio, 4),
               "max_kernel_ratio": round(r.max_kernel_ratio, 4), "ok": r.all_within_bound,
               "cal": r.calibration,
               "tasks": [{k: t[k] for k in ("task", "sms", "jobs", "ratio", "kernel_span_us_vs_gr_up",
                                            "kernel_event_us", "kernel_wall_us", "worst_launch", "min_sm_mhz", "max_copy_us", "max_bus_wait_us")}
                         for t in r.tasks]}
        print(json.dumps(rec), flush=True)
        out.append(rec)
json.dump(out, open("gpurun_out/wcrt_modes.json", "w"), indent=1)
