# r2zj: source-level ncu of the lattice kernel after the cycle bounds.
mkdir -p gpurun_out
for sh in alloc64 sweep16x9; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
    -o gpurun_out/prof_r2zj_$sh python scripts/lat_ab.py 1 $sh > gpurun_out/ncu_r2zj_$sh.log 2>&1
  echo "ncu $sh rc=$?"
done
