# K3 bf16 micro-variants A/B on one box: 0 = product, A = __frcp_rn(r), B = count samples per token,
# (The MCA_K3_FRCP / MCA_K3_CNT_TOKEN switches were removed after this measurement: no gain,
# DESIGN.md §5. MCA_K3_STEAL remains.)
# C / D = head-stealing threshold 256 / 1024 list entries (product 512)
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/lib30.so
for rep in 1 2; do for v in 0 A B C D; do
  cp /tmp/lib30.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/lib3$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k3_encode_sampled -c 3 --csv --log-file gpurun_out/k3m$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo "$v $(python scripts/launches_summary.py gpurun_out/k3m$v.csv | tail -1)"
done; done
cp /tmp/lib30.so paper_2201_12854_b200/lib/libmca_b200.so
