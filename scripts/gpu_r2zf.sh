# r2zf: fast path's exact fallback out of line (default) vs inlined (c2).
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zf c2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_rec32.py -m gpu -x -q > gpurun_out/r2zf_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2zf_pytest.log
