for v in default variants/lib_minb3.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/$v; fi
  echo "== $v"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-wcrt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), 'sets/s e2e', round(d['e2e']['value']), 'stages', [round(x,3) for x in d['roofline']['stage_ms']], d['roofline']['stage_sets'])"
done
unset RTGPU_LIB
for w in sweep16x9 alloc64; do
  echo "== workload $w"
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-wcrt > gpurun_out/bench_$w.log 2>&1; tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'sets/s', d['ms_per_step'], [round(x,3) for x in d['roofline']['stage_ms']], d['roofline']['stage_sets'], d['acceptance_rtgpu'])"
done
