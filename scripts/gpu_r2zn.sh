# r2zn: fast-path all-minimum pass (default) vs HEAD (c5); fast-path GPU tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zn c5
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_rec32.py tests/test_fullsize.py -m gpu -x -q > gpurun_out/r2zn_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2zn_pytest.log
