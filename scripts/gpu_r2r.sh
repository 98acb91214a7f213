# r2r: executor launch log over wide-partition seeds (is an overrun one
# partition's or GPU-wide?)
mkdir -p gpurun_out
timeout 3000 python scripts/wcrt_robustness.py --wide --seeds 16 --horizon-s 1.0 > gpurun_out/wcrt_r2r.jsonl 2>&1; echo "wcrt rc=$?"; tail -1 gpurun_out/wcrt_r2r.jsonl
