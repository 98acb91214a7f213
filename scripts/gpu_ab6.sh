# L2 evict-first hint on batch words (RTGPU_BLOB_EVICT_FIRST): default vs variants/lib_evict.so
# bench value + DRAM bytes of one fast_kernel launch for each
for v in default variants/lib_evict.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; tag=def; else export RTGPU_LIB=$PWD/$v; tag=ef; fi
  echo "== $v"
  for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim > gpurun_out/bench_ab6_$tag.log 2>&1; tail -1 gpurun_out/bench_ab6_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'sets/s; e2e', round(d['e2e']['value']), d['ms_per_step'], round(d['roofline']['kernel_ms'],3))"
  done
  RTGPU_NO_STREAM=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fast_kernel -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
unset RTGPU_LIB
