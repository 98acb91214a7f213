# r2zx: fast-path all-minimum pass ahead of the range checks (default) vs HEAD (c10):
# the configs[1] bench workload (stage tail) and fast-path GPU tests.
mkdir -p gpurun_out
for lib in default c10; do
  if [ $lib = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/variants/lib_$lib.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim --sub '' \
    > gpurun_out/r2zx_main_$lib.log 2>&1; echo "bench $lib rc=$?"
  tail -1 gpurun_out/r2zx_main_$lib.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['e2e']['value'], d['roofline'].get('stage_ms'), d['roofline'].get('stage_sets'))"
done
unset RTGPU_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_rec32.py tests/test_fullsize.py tests/test_ood.py -m gpu -x -q > gpurun_out/r2zx_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2zx_pytest.log
