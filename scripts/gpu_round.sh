# One GPU pass: tests, smoke, bench (both arms), launch list, full ncu capture of the
# dominant kernel.  Usage (from repo root, under gpurun): bash scripts/gpu_round.sh TAG
# Under ncu the e2e verdict path runs unstreamed (RTGPU_NO_STREAM=1): ncu serialises
# kernels, so a persistent kernel waiting on copies queued behind it would time out.
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
RTGPU_NO_STREAM=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-launch rc=$?"
RTGPU_NO_STREAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel|front_kernel" -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-wcrt --no-sim > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
python - <<'PY' > gpurun_out/h2d_$TAG.txt 2>&1
import torch, time
x = torch.empty(192 << 20, dtype=torch.uint8, pin_memory=True)
y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); [y.copy_(x, non_blocking=True) for _ in range(10)]; e.record(); torch.cuda.synchronize()
print("H2D GB/s", 10 * x.numel() / (s.elapsed_time(e) * 1e-3) / 1e9)
PY
cat gpurun_out/h2d_$TAG.txt
