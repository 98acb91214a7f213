# A/B of library variants on the benchmark (bench only, no extras)
for v in default variants/lib_head.so default variants/lib_head.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/$v; fi
  echo "== $v"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), 'sets/s e2e', round(d['e2e']['value']), 'stages', [round(x,3) for x in d['roofline']['stage_ms']], d['roofline']['stage_sets'])"
done
unset RTGPU_LIB
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -x -q 2>&1 | tail -1
