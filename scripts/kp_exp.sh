for v in 0 1; do
KP_DBG=$v ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:kp_project -c 4 --csv --log-file gpurun_out/kp_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1; echo rc=$?
python scripts/launches_summary.py gpurun_out/kp_$v.csv
done
