import json, sys
sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex
for seed, util in ((5, 2.5), (8, 4.0), (5, 3.0)):
    r = ex.wcrt_experiment(n_tasks=4, m=3, horizon_us=1.0e6, seed=seed, utilization=util)
    print(seed, util, r.max_ratio, r.max_kernel_ratio)
    for t in r.tasks:
        print("   ", t["task"], t["sms"], t["kernel_span_us_vs_gr_up"], t["kernel_event_us"], t["kernel_wall_us"], t["worst_launch"], t["min_sm_mhz"])
    print("   cal", [(c["items"], c["t1_us"], c["t2_us"], c["alpha"], c["gw_hi_us"]) for c in r.calibration])
