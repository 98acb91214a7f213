# ncu captures of the lattice kernel via scripts/lat_ab.py shapes.
# Usage (repo root, under gpurun): bash scripts/gpu_prof_lat2.sh TAG shape[,shape]
TAG=${1:-lat}
SHAPES=${2:-sweep16x9,bounds8x5}
mkdir -p gpurun_out
for sh in ${SHAPES//,/ }; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_$sh python scripts/lat_ab.py 1 $sh > gpurun_out/ncu_${TAG}_$sh.log 2>&1
  echo "ncu $sh rc=$?"
done
