# r2za: memory-guess variants of the lattice path (guess1: hp-count-scaled
# 1.4 k/(k-1); guess2: 2x) against the default; ncu of the lattice kernel.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2za guess1 guess2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
  -o gpurun_out/prof_r2za_sweep16x9 python scripts/lat_ab.py 1 sweep16x9 > gpurun_out/ncu_r2za.log 2>&1
echo "ncu rc=$?"
