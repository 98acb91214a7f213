# r2y: header fields in shared memory + per-lane slot setup hoisted out of the
# fixed-point iterations (default) vs the committed build (c1) vs r2w (head).
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2y c1 head
