# K3 bf16 with / without the X-row L1 prefetch (A/B on one box, twice)
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libpf.so
for rep in 1 2; do for v in pf np; do
  if [ $v = pf ]; then cp /tmp/libpf.so paper_2201_12854_b200/lib/libmca_b200.so; else cp paper_2201_12854_b200/lib_exp/libnp.so paper_2201_12854_b200/lib/libmca_b200.so; fi
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k3_encode_sampled -c 3 --csv --log-file gpurun_out/k3$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo $v; python scripts/launches_summary.py gpurun_out/k3$v.csv | tail -1
done; done
cp /tmp/libpf.so paper_2201_12854_b200/lib/libmca_b200.so
