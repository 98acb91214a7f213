# r2x: lattice search state in shared memory -- same-box A/B against the
# previous build (variants/lib_head.so), then the lattice GPU tests.
mkdir -p gpurun_out
bash scripts/gpu_lat_ab.sh r2x head
timeout 900 python -m pytest tests/test_lattice.py tests/test_adversarial.py tests/test_gpu_parity.py -m gpu -x -q \
  > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2x_pytest.log
