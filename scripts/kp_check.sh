timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -x -k "projection or c3 or graph" > gpurun_out/t.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t.log
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 14 --csv --log-file gpurun_out/kp.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1; echo rc=$?
python scripts/launches_summary.py gpurun_out/kp.csv
