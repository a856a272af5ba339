# ncu launch lists (per-kernel device time, cold cache, serialised) of the fp32 configurations: C2 fp32 and C1
python bench.py --dtype f32 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/plain_f32.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c2_f32.csv python bench.py --dtype f32 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/ncu_f32.log 2>&1; echo f32_ncu_rc=$?
python scripts/launches_summary.py gpurun_out/launches_c2_f32.csv
python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/plain_c1.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/ncu_c1.log 2>&1; echo c1_ncu_rc=$?
python scripts/launches_summary.py gpurun_out/launches_c1.csv
