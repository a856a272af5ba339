# K4 tf32 split experiment: v0 = product, v1 = no softmax P stores, v2 = no MMAs
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libv0.so
for v in 0 1 2 3; do
  cp /tmp/libv0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libv$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k4_apply -c 3 --csv --log-file gpurun_out/k4v$v.csv python bench.py --dtype f32 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo v$v; python scripts/launches_summary.py gpurun_out/k4v$v.csv | tail -1
done
cp /tmp/libv0.so paper_2201_12854_b200/lib/libmca_b200.so
