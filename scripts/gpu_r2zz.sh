# r2zz: largest count first in the exact search (default) vs HEAD (c11); GPU tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zz c11
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2zz_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2zz_pytest_gpu.log
