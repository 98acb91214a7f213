# One GPU pass: tests, smoke, bench (both arms), launch list, full ncu
# captures of the dominant kernels (fast kernel on configs[1]; the lattice
# kernel on configs[2] / configs[4] and on the bounds run).
# Usage (from repo root, under gpurun): bash scripts/gpu_round.sh TAG
# Under ncu the e2e verdict path runs unstreamed (RTGPU_NO_STREAM=1): ncu serialises
# kernels, so a persistent kernel waiting on copies queued behind it would time out.
# Then on the CPU box:
#   python scripts/make_profiles.py gpurun_out/prof_TAG.ncu-rep gpurun_out/launches_TAG.csv \
#       --tag TAG --key fast_kernel --sets 100000 --lib-sha $(cat gpurun_out/lib_sha_TAG.txt)
#   python scripts/make_profiles.py gpurun_out/prof_TAG_sweep16x9.ncu-rep --tag TAG_sweep16x9 \
#       --key lattice_kernel:sweep16x9 --sets 1000000 --lib-sha ...   (alloc64: 100000, bounds8x5: 100000)
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import bench; print(bench.lib_sha())" > gpurun_out/lib_sha_$TAG.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
RTGPU_NO_STREAM=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim --sub '' > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-launch rc=$?"
RTGPU_NO_STREAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel" -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim --sub '' > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
for wl in sweep16x9 alloc64; do
  RTGPU_NO_STREAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_$wl python bench.py --workload $wl --steps 1 --warmup 1 --no-cpu-baseline --no-wcrt --no-sim --sub '' \
    > gpurun_out/ncu_${TAG}_$wl.log 2>&1; echo "ncu $wl rc=$?"
done
RTGPU_NO_STREAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_bounds8x5 python bench.py --flags bounds --steps 1 --warmup 1 --no-cpu-baseline --no-wcrt --no-sim --sub '' \
  > gpurun_out/ncu_${TAG}_bounds8x5.log 2>&1; echo "ncu bounds8x5 rc=$?"
python - <<'PY' > gpurun_out/h2d_$TAG.txt 2>&1
import torch
x = torch.empty(192 << 20, dtype=torch.uint8, pin_memory=True)
y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); [y.copy_(x, non_blocking=True) for _ in range(10)]; e.record(); torch.cuda.synchronize()
print("H2D GB/s", 10 * x.numel() / (s.elapsed_time(e) * 1e-3) / 1e9)
PY
cat gpurun_out/h2d_$TAG.txt
