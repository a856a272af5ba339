# KP CTA-pair ring depth: p0 = product (4 stages), p6, p3
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libp0.so
for v in 0 6 3; do
  cp /tmp/libp0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libk2s$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:kp_project -c 6 --csv --log-file gpurun_out/kp2s$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo p$v; python scripts/launches_summary.py gpurun_out/kp2s$v.csv | tail -2 | head -1
done
cp /tmp/libp0.so paper_2201_12854_b200/lib/libmca_b200.so
