# Round profile (scripts/profile_round.sh): launch list of the default bench
# (cold-cache, serialised) + one ncu --set full capture of every kernel of one
# forward. Run each only after the plain command exited 0.
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
ncu --nvtx --nvtx-include "mca_step/" --set full --clock-control none --import-source on -k regex:"kp_project_tc|k12_fused_tc|k2_scan|k3_encode_sampled|k3b_exact_tc|k4_apply_tc" -c 7 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
