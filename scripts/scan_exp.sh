# k2_scan_scatter: budget loads issued before the histogram scan (new) vs after (old), A/B twice
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libnew.so
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then cp /tmp/libnew.so paper_2201_12854_b200/lib/libmca_b200.so; else cp paper_2201_12854_b200/lib_exp/libscanold.so paper_2201_12854_b200/lib/libmca_b200.so; fi
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:k2_scan_scatter -c 3 --csv --log-file gpurun_out/scan$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1
  echo $v; grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/scan$v.csv | tail -1
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v bench', round(d['ms_per_step'],4), round(d['stages_ms']['budgets'],4))"
done; done
cp /tmp/libnew.so paper_2201_12854_b200/lib/libmca_b200.so
