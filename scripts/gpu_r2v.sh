mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2v.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r2v.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2v.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_r2v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value']); print({k:v.get('value') for k,v in d['workloads'].items()}); print(d['wcrt_vs_bound'].get('max_kernel_over_lemma4'), d['wcrt_vs_bound'].get('max_kernel_over_lemma4_net_of_stalls'), d['wcrt_vs_bound'].get('gpu_stalls')); print(d.get('dropin'))"
