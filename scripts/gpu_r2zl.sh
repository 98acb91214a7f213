# r2zl: lattice next-task L1 prefetch (default) vs without (nopf).
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zl nopf
