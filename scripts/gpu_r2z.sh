# r2z: fast_verdict search state in shared memory (default) vs the committed
# build (c1); full GPU test suite; one bench line.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2z c1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2z_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2z_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2z_bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/r2z_bench.log
