# r2zq: one report call site in the lattice kernel (default) vs HEAD (c7).
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zq c7
