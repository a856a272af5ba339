# K4 with / without an L2 prefetch of the next tile's K / H~ (A/B twice), then the per-block timeline.
# Measured 94.7 (prefetch) vs 83.8 us; the prefetch (MCA_K4_L2PF, cp.async.bulk.prefetch.tensor) was removed after it.
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libpf.so
for rep in 1 2; do for v in pf nopf; do
  if [ $v = pf ]; then cp /tmp/libpf.so paper_2201_12854_b200/lib/libmca_b200.so; else cp paper_2201_12854_b200/lib_exp/libk4nopf.so paper_2201_12854_b200/lib/libmca_b200.so; fi
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['stages_ms']['apply']*1e3,1))"
done; done
cp /tmp/libpf.so paper_2201_12854_b200/lib/libmca_b200.so
bash scripts/k4_timeline.sh
