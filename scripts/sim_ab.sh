# simulator A/B: default vs variants/lib_head.so, plus the simulator GPU tests
for v in default variants/lib_head.so; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/$v; fi
  echo "== $v"; timeout 300 python scripts/sim_speed.py 3000 2>&1 | tail -2
done
unset RTGPU_LIB
timeout 600 python -m pytest tests/test_sim_gpu.py -x -q 2>&1 | tail -1
