MCA_K3_TILE=1 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_tile.log 2>&1; echo tile_tests_rc=$?; tail -4 gpurun_out/gpu_tests_tile.log
MCA_K3_TILE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tile.json 2> gpurun_out/bench_tile.err; echo bench_rc=$?
MCA_K3_TILE=1 timeout 300 python scripts/alpha_sweep.py --seeds 2 > gpurun_out/alpha_tile.log 2>&1
