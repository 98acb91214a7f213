# A/B of library variants: default build vs variants/*.so, bench only (+ one ncu of default)
for v in default variants/lib_minb3.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/$v; fi
  echo "== $v"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), 'sets/s', 'k0_ms', round(d['roofline']['kernel_ms'],2), d['clocks'])"
  timeout 300 python bench.py --steps 5 --warmup 3 --flags bounds --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bounds', round(d['value']), 'sets/s')"
done
unset RTGPU_LIB
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:analyze_kernel -s 3 -c 1 -o gpurun_out/prof_${1:-ab} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sets-per-point 2000 > gpurun_out/ncu_ab.log 2>&1; echo "ncu rc=$?"
