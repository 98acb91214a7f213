mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2j | tail -4
timeout 3000 python scripts/wcrt_robustness.py --wide --seeds 24 --horizon-s 1.0 > gpurun_out/exec_wide_robust_r2j.jsonl 2>&1; echo "robust rc=$?"
tail -1 gpurun_out/exec_wide_robust_r2j.jsonl
