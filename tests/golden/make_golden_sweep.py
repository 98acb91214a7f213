"""Golden acceptance sweeps produced by the REFERENCE (needs /root/reference).

    python tests/golden/make_golden_sweep.py

Runs gpusched.workbench.acceptance_sweep on small configurations and stores
the CSV text.  The baselines need the three missing imports injected (see
make_golden.py); that is recorded in the file."""
import json
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import _ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sweep_golden.json")

CONFIGS = [
    {"params": {"n_tasks": 3, "n_subtasks": 3, "physical_sms": 4}, "dimension": "none",
     "utilizations": ["1/2", "1", "3/2"], "mem_models": ["two_copy", "one_copy"],
     "tasksets_per_point": 12, "seed": 7},
    {"params": {"n_tasks": 3, "n_subtasks": 2, "physical_sms": 6}, "dimension": "physical_sms",
     "values": [3, 5], "utilizations": ["1/2", "1"], "methods": ["rtgpu", "busywait"],
     "tasksets_per_point": 10, "seed": 3},
    {"params": {"n_tasks": 4, "n_subtasks": 3}, "dimension": "length_scale",
     "values": ["1/2", "2"], "utilizations": ["2/5", "4/5"], "methods": ["rtgpu", "selfsusp"],
     "tasksets_per_point": 8, "seed": 11},
]


def main():
    g = _ref()
    import gpusched.workbench as wb
    out = []
    for cfg in CONFIGS:
        sc = wb.sweep_config_from_dict(cfg)
        rows = wb.acceptance_sweep(sc)
        out.append({"config": cfg, "csv": wb.sweep_to_csv(rows)})
        print(wb.sweep_to_csv(rows))
    with open(OUT, "w") as fh:
        json.dump({"source": "reference gpusched acceptance_sweep (baseline imports injected)",
                   "sweeps": out}, fh, indent=1)


if __name__ == "__main__":
    main()
