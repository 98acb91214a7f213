# GPU pass: tests, lattice A/B, one wide-partition executor trial.
# Usage (repo root, under gpurun): bash scripts/gpu_mixed.sh TAG [variants...]
TAG=${1:-mx}
shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu_$TAG.log
bash scripts/gpu_lat_ab.sh $TAG "$@" | tail -16
timeout 600 python - <<'PY' > gpurun_out/exec_wide_$TAG.log 2>&1
import json, sys
sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex
for width in ((12, 24), (24, 36)):
    r = ex.wcrt_experiment(n_tasks=4, m=3, horizon_us=1.0e6, seed=1, width=width)
    print(json.dumps({"width": width, "schedulable": r.schedulable, "note": r.note, "alloc": r.allocation,
                      "sms_used": r.sms_used, "max_ratio": r.max_ratio, "max_kernel_ratio": r.max_kernel_ratio,
                      "calibration": r.calibration, "tasks": r.tasks}), flush=True)
PY
echo "exec rc=$?"; cut -c1-700 gpurun_out/exec_wide_$TAG.log
