# workloads (configs[2] / configs[4] shapes): default vs variants/lib_f64first.so
for w in sweep16x9 alloc64; do
for v in default variants/lib_f64first.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/$v; fi
  echo "== $w $v"
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim > gpurun_out/bench_$w.log 2>&1; tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'sets/s e2e', round(d['e2e']['value']), d['ms_per_step'], [round(x,3) for x in d['roofline']['stage_ms']], d['roofline']['stage_sets'], d['acceptance_rtgpu'])"
done
done
unset RTGPU_LIB
