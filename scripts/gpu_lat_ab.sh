# A/B of lattice-kernel builds (variants/lib_*.so) on the 148-SM shapes.
# Usage (repo root, under gpurun): bash scripts/gpu_lat_ab.sh TAG [variants...]
TAG=${1:-ab}
shift
mkdir -p gpurun_out
for v in default "$@"; do
  if [ "$v" = default ]; then unset RTGPU_LIB; else export RTGPU_LIB=$PWD/variants/lib_$v.so; fi
  timeout 600 python scripts/lat_ab.py 3 >> gpurun_out/lat_ab_$TAG.log 2>&1
done
unset RTGPU_LIB
cat gpurun_out/lat_ab_$TAG.log
