MCA_K3_DENSE=1 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_dense.log 2>&1; echo dense_tests_rc=$?; tail -4 gpurun_out/gpu_tests_dense.log
MCA_K3_DENSE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dense.json 2> gpurun_out/bench_dense.err; echo bench_rc=$?
MCA_K3_DENSE=1 timeout 300 python scripts/alpha_sweep.py --seeds 2 > gpurun_out/alpha_dense.log 2>&1
