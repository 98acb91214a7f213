mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2l noguess nodcheck neither | tail -16
for v in default bps16; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/variants/lib_$v.so; fi
  timeout 900 python scripts/wcrt_robustness.py --wide --seeds 3 --horizon-s 1.0 > gpurun_out/exec_diag_${v}_r2l.jsonl 2>&1
  echo "== $v"; tail -1 gpurun_out/exec_diag_${v}_r2l.jsonl
done
unset RTGPU_LIB
