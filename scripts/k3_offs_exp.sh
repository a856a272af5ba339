# K3 bf16: per-round row offsets + coefficient words (new) vs packed (row | coef) words (old), A/B twice
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libnew.so
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then cp /tmp/libnew.so paper_2201_12854_b200/lib/libmca_b200.so; else cp paper_2201_12854_b200/lib_exp/libk3old.so paper_2201_12854_b200/lib/libmca_b200.so; fi
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k3_encode_sampled -c 3 --csv --log-file gpurun_out/k3$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo $v; grep -o '"smsp__inst_executed.sum","inst","[0-9,]*"\|"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/k3$v.csv | tail -2
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v bench', round(d['ms_per_step'],4), round(d['stages_ms']['encode'],4))"
done; done
cp /tmp/libnew.so paper_2201_12854_b200/lib/libmca_b200.so
