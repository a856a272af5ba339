# K4 bf16 split: e0 = product, e1 = no exponentials, e2 = no MMAs
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libe0.so
for v in 0 1 2; do
  cp /tmp/libe0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libe$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k4_apply_tc -c 3 --csv --log-file gpurun_out/k4e$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo e$v; python scripts/launches_summary.py gpurun_out/k4e$v.csv | tail -1
done
cp /tmp/libe0.so paper_2201_12854_b200/lib/libmca_b200.so
