# r2w: lattice A/B baseline on this box + source-level ncu of the lattice kernel
# (configs[2] and configs[4] shapes).  Usage (repo root, under gpurun).
mkdir -p gpurun_out
timeout 600 python scripts/lat_ab.py 3 > gpurun_out/r2w_lat_ab.log 2>&1; echo "lat_ab rc=$?"
cat gpurun_out/r2w_lat_ab.log
for sh in sweep16x9 alloc64; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
    -o gpurun_out/prof_r2w_$sh python scripts/lat_ab.py 1 $sh > gpurun_out/ncu_r2w_$sh.log 2>&1
  echo "ncu $sh rc=$?"
done
