# r2q: array-path GPU parity + bench with the drop-in section + executor
# placement diagnostics on the seeds that overran in r2j.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_arrays.py tests/test_executor_gpu.py -m gpu -x -q > gpurun_out/pytest_r2q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2q.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sim --sub '' > gpurun_out/bench_r2q.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_r2q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value']); print(json.dumps(d.get('dropin'))); print(json.dumps(d.get('wcrt_vs_bound'))[:1500])"
timeout 2400 python scripts/wcrt_robustness.py --wide --seed-list 7,17,5,9,18,21,19 --horizon-s 1.0 > gpurun_out/wcrt_r2q.jsonl 2>&1; echo "wcrt rc=$?"; tail -1 gpurun_out/wcrt_r2q.jsonl
