# ncu launch lists (per-kernel device time, cold cache, serialised) of the default bench and c4
for c in c2 c4; do
python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/plain_$c.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/ncu_$c.log 2>&1; echo ${c}_ncu_rc=$?
python scripts/launches_summary.py gpurun_out/launches_$c.csv
done
