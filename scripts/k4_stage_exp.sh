# K4 bf16 ring depth: s0 = product (4 stages), s6, s3
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libs0.so
for v in 0 6 3; do
  cp /tmp/libs0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libs$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k4_apply_tc -c 3 --csv --log-file gpurun_out/k4s$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo e$v; python scripts/launches_summary.py gpurun_out/k4s$v.csv | tail -1
done
cp /tmp/libs0.so paper_2201_12854_b200/lib/libmca_b200.so
