# K1a (row statistics, n > 768) FMA-pipe exp2 share at C4 (n = 4096): q0 = MUFU only, qN = N of 32 pairs per chunk
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libq0.so
for v in 0 6 10 14; do
  cp /tmp/libq0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libq$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k1_scores_tc -c 4 --csv --log-file gpurun_out/k1q$v.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo q$v; python scripts/launches_summary.py gpurun_out/k1q$v.csv | tail -2
  true
done
cp /tmp/libq0.so paper_2201_12854_b200/lib/libmca_b200.so
