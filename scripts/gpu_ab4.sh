# A/B: verdict and bounds modes, default vs variants/lib_head.so
for v in default variants/lib_head.so default variants/lib_head.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/$v; fi
  echo "== $v"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), 'sets/s e2e', round(d['e2e']['value']), 'stages', [round(x,3) for x in d['roofline']['stage_ms']], d['roofline']['stage_sets'])"
  timeout 300 python bench.py --steps 5 --warmup 3 --flags bounds --no-cpu-baseline --no-wcrt --no-sim | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bounds', round(d['value']), 'sets/s', [round(x,3) for x in d['roofline']['stage_ms']])"
done
unset RTGPU_LIB
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py tests/test_blocks.py -x -q 2>&1 | tail -1
