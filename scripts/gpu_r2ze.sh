# r2ze: packed task records (header word 7 = 2) in the bench workloads:
# GPU tests (incl. tests/test_rec32.py) and one bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2ze_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2ze_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-wcrt --no-sim > gpurun_out/r2ze_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2ze_bench.log | cut -c1-700
