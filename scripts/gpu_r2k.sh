mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2k | tail -4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2k.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu_r2k.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
    -o gpurun_out/prof_r2k_sweep16x9 python scripts/lat_ab.py 1 sweep16x9 > gpurun_out/ncu_r2k.log 2>&1; echo "ncu rc=$?"
