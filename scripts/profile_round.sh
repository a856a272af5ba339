# Launch list of the default bench (cold-cache, serialised) + one full ncu capture of the hot kernels.
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
ncu --nvtx --nvtx-include "mca_step/" --set full --clock-control none --import-source on -k regex:"k12_fused_tc|k2_scan|k2_scatter|k3_encode_sampled|k3b_exact_tc|k4_apply_tc" -s 10 -c 5 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
