set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
timeout 600 python bench.py --steps 5 --warmup 3 --flags bounds --no-cpu-baseline > gpurun_out/bench_bounds.log 2>&1; tail -2 gpurun_out/bench_bounds.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:analyze_kernel -s 3 -c 1 -o gpurun_out/prof_stage0 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sets-per-point 2000 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -5 gpurun_out/ncu_full.log
