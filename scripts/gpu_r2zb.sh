# r2zb: lattice quick pass at the minimum count (default) vs without
# (noquick) vs the committed build (c1); lattice GPU parity tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2zb noquick c1
timeout 900 python -m pytest tests/test_lattice.py tests/test_adversarial.py tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -x -q \
  > gpurun_out/r2zb_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2zb_pytest.log
