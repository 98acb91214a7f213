# r2t: executor with the fixed stall sentinel (tests + robustness), lattice
# micro variant A/B, e2e with the result copies queued before the host check
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu -q > gpurun_out/pytest_exec_r2t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exec_r2t.log
timeout 1800 python scripts/wcrt_robustness.py --wide --seeds 16 --horizon-s 1.0 > gpurun_out/wcrt_r2t.jsonl 2>&1; echo "wcrt rc=$?"; tail -1 gpurun_out/wcrt_r2t.jsonl
bash scripts/gpu_lat_ab.sh r2t micro
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sim --no-wcrt --sub '' > gpurun_out/bench_r2t_$i.log 2>&1; tail -1 gpurun_out/bench_r2t_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; done
