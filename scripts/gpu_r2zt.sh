# r2zt: lattice setup in shared memory / lane-parallel (default) vs HEAD (c8); GPU tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zt c8
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2zt_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2zt_pytest_gpu.log
