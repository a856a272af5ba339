# K3 bf16 split: k0 = product, k1 = draws only (no accumulation), k2 = accumulation only (no draws)
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libk0.so
for v in 0 1 2; do
  cp /tmp/libk0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libk$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k3_encode_sampled -c 3 --csv --log-file gpurun_out/k3s$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo k$v; grep "inst_executed" gpurun_out/k3s$v.csv | head -1 | awk -F'","' '{print $NF}'; grep "gpu__time_duration" gpurun_out/k3s$v.csv | head -1 | awk -F'","' '{print $NF}'
done
cp /tmp/libk0.so paper_2201_12854_b200/lib/libmca_b200.so
