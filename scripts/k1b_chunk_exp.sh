# K1b: chunk maximum by FFMA2 + 3-input max, argmax located only when the chunk wins (new)
# vs per-element compare/select (old): C4 (n = 4096) and C2 fp32, A/B twice
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libnew.so
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then cp /tmp/libnew.so paper_2201_12854_b200/lib/libmca_b200.so; else cp paper_2201_12854_b200/lib_exp/libk1old.so paper_2201_12854_b200/lib/libmca_b200.so; fi
  python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c4', round(d['ms_per_step'],4), round(d['stages_ms']['score'],4), d['budget_mismatch_vs_fp64']['count'] if d.get('budget_mismatch_vs_fp64') else None)"
  python bench.py --dtype f32 --steps 10 --warmup 3 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c2f32', round(d['ms_per_step'],4), round(d['stages_ms']['score'],4))"
done; done
cp /tmp/libnew.so paper_2201_12854_b200/lib/libmca_b200.so
