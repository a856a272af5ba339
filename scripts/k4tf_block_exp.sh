# K4 tf32: product (32-key blocks, 2 stages, 4 O accumulators) vs the round-2 first version's
# (lib_exp/lib64.so is built from git show b72c506:paper_2201_12854_b200/csrc/k4_apply_tf32.cu with the
# whole-warp MMA issue ported in; it is not part of the tree.)
# 64-key single-buffered blocks with the whole-warp MMA issue (lib_exp/lib64.so)
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libk4p.so
for rep in 1 2; do for v in p 64; do
  if [ $v = p ]; then cp /tmp/libk4p.so paper_2201_12854_b200/lib/libmca_b200.so; else cp paper_2201_12854_b200/lib_exp/lib64.so paper_2201_12854_b200/lib/libmca_b200.so; fi
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k4_apply_tf32 -c 3 --csv --log-file gpurun_out/k4b$v.csv python bench.py --dtype f32 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo "$v $(python scripts/launches_summary.py gpurun_out/k4b$v.csv | tail -1)"
done; done
cp /tmp/libk4p.so paper_2201_12854_b200/lib/libmca_b200.so
