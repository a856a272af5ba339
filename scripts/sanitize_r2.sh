# compute-sanitizer memcheck over the round-2 kernels' tests
S="/usr/local/cuda/bin/compute-sanitizer --print-limit 4"
timeout 1200 $S python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x \
  -k "projection_gemm_shapes or bf16_regular_forward_dense or fp16 or c1_ or edge_shapes or bf16_parity" > gpurun_out/san1.log 2>&1; echo rc1=$?
grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/san1.log | head -8
timeout 1200 $S python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -x -k "tied" > gpurun_out/san2.log 2>&1; echo rc2=$?
grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/san2.log | head -8
