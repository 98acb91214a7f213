# r2zc: fast-path quick pass (default) vs without (fnoquick) vs c1; GPU tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zc fnoquick c1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2zc_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2zc_pytest_gpu.log
