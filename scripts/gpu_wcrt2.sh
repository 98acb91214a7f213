timeout 600 python - <<'PY'
import json
from paper_2101_10463_b200.executor import wcrt_experiment
for u in (3.0,):
    r = wcrt_experiment(n_tasks=4, m=3, horizon_us=1.5e6, seed=3, utilization=u)
    print(u, r.schedulable, r.all_within_bound, r.kernels_within_bound, round(r.max_ratio,3), r.allocation)
    for t in r.tasks: print("   ", t["task"], t["sms"], t["blocks_per_launch"], t["kernel_span_us_vs_gr_up"], t["ratio"])
PY
bash scripts/gpu_bench_prof.sh fast tests
