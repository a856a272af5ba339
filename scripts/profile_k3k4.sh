python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3_encode_sampled|k3b_encode_exact|k4_apply_tc|k1_scores_tc" -s 8 -c 5 -o gpurun_out/prof_r1b python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu_rc=$?
