# quick loop: GPU tests (optional), bench, one full ncu capture of the stage-0 kernel
TAG=${1:-x}
if [ "$2" = "tests" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log; fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_$TAG.log | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --flags bounds --no-cpu-baseline > gpurun_out/bench_bounds_$TAG.log 2>&1; cut -c1-300 gpurun_out/bench_bounds_$TAG.log | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:front_kernel -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sets-per-point 2000 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
