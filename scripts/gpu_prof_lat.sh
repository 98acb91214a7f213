# ncu captures of the lattice kernel on the 148-SM workloads (configs[2] and
# configs[4]).  Usage (repo root, under gpurun): bash scripts/gpu_prof_lat.sh TAG
TAG=${1:-lat}
mkdir -p gpurun_out
for wl in sweep16x9 alloc64; do
  RTGPU_NO_STREAM=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:lattice_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG}_$wl \
    python bench.py --workload $wl --sub '' --steps 1 --warmup 1 --no-cpu-baseline --no-wcrt --no-sim \
    > gpurun_out/ncu_${TAG}_$wl.log 2>&1; echo "ncu $wl rc=$?"
  tail -2 gpurun_out/ncu_${TAG}_$wl.log | cut -c1-300
done
