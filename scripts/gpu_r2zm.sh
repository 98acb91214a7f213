# r2zm: set-level all-minimum quick pass (default) vs HEAD (c4); GPU tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zm c4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2zm_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2zm_pytest_gpu.log
