# r2zh: cycle-bound checks in the quick passes (default) vs without
# (nocycle, same tree) vs HEAD (c3); GPU tests of the paths.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zh nocycle c3
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2zh_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2zh_pytest_gpu.log
