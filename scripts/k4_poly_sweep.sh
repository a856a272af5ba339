# K4: pairs per thread and block exponentiated on the FMA pipe (of 16) vs MUFU
for k in 0 4 7 10; do
  make -s -B -C paper_2201_12854_b200/csrc EXTRA=-DMCA_K4_POLY=$k >/dev/null 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/k4poly_$k.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/k4poly_$k.json'));print('poly', $k, round(d['value']), round(d['stages_ms']['apply']*1e3,1), 'us apply')"
done
make -s -B -C paper_2201_12854_b200/csrc >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "bf16_parity or theorem or c2_full" 2>&1 | tail -2
