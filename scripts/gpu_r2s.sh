# r2s: executor robustness with the stall sentinel; lattice CTA-shape A/B
mkdir -p gpurun_out
timeout 2400 python scripts/wcrt_robustness.py --wide --seeds 16 --horizon-s 1.0 > gpurun_out/wcrt_r2s.jsonl 2>&1; echo "wcrt rc=$?"; tail -1 gpurun_out/wcrt_r2s.jsonl
bash scripts/gpu_lat_ab.sh r2s t128m3 t128m5 t128m4
