# r2zo: reciprocal floor division in the all-minimum passes (default) vs 64-bit division (c6).
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zo c6
