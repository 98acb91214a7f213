# r2zv: all-minimum pass ahead of the FP64 range check (default) vs HEAD (c9):
# the configs[4] bench workload (its range escalations) and the A/B shapes.
mkdir -p gpurun_out
for lib in default c9; do
  if [ $lib = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/variants/lib_$lib.so; fi
  timeout 600 python bench.py --workload alloc64 --steps 5 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim --sub '' \
    > gpurun_out/r2zv_alloc64_$lib.log 2>&1; echo "bench $lib rc=$?"
  tail -1 gpurun_out/r2zv_alloc64_$lib.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['roofline'].get('stage_ms'), d['roofline'].get('stage_sets'))"
done
unset RTGPU_LIB
timeout 900 python -m pytest tests/test_lattice.py tests/test_fullsize.py tests/test_adversarial.py -m gpu -x -q > gpurun_out/r2zv_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2zv_pytest.log
