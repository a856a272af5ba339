# compute-sanitizer over one GPU test: bash scripts/sanitize_test.sh <pytest -k expression>
timeout 900 /usr/local/cuda/bin/compute-sanitizer --print-limit 4 python -m pytest tests/test_gpu_parity.py -m gpu -q \
    -p no:cacheprovider -x -k "$1" > gpurun_out/sanitize.log 2>&1
echo rc=$?
grep -E "Invalid|at 0x|by thread|Address|passed|failed" gpurun_out/sanitize.log | head -20
