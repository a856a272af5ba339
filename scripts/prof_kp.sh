python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --set full --clock-control none --import-source on -k regex:"kp_project_tc" -s 3 -c 1 -o gpurun_out/prof_kp python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/ncu_kp.log 2>&1; echo ncu_rc=$?
