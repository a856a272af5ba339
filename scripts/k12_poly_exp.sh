# K12 FMA-pipe exp2 share: p0 = product (MUFU only), pN = N of 16 pairs per chunk on the polynomial
# (The MCA_K12_POLY switch and ex2_poly5x2 in k12 were removed after this measurement: slower at
# every share, DESIGN.md §4. ex2_poly5x2 lives on in K1a, MCA_K1_POLY.)
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libp0.so
for v in 0 4 6 8; do
  cp /tmp/libp0.so paper_2201_12854_b200/lib/libmca_b200.so
  [ $v != 0 ] && cp paper_2201_12854_b200/lib_exp/libp$v.so paper_2201_12854_b200/lib/libmca_b200.so
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k12_fused -c 3 --csv --log-file gpurun_out/k12p$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo p$v; python scripts/launches_summary.py gpurun_out/k12p$v.csv | tail -1
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "bf16_parity or stage_budgets or c2_full or fused" 2>&1 | tail -1
done
cp /tmp/libp0.so paper_2201_12854_b200/lib/libmca_b200.so
