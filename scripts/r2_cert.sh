timeout 800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t.log
grep -E "mismatches|re-derived" gpurun_out/t.log | head -5
for c in c2 c4; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 2 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo ${c}_rc=$?; tail -2 gpurun_out/b_$c.err
python - <<PY
import json; d=json.loads(open('gpurun_out/b_$c.json').read())
print('$c', 'ms %.4f'%d['ms_per_step'], {k:round(v,4) for k,v in d['stages_ms'].items()}, d['budget_mismatch_vs_fp64'])
PY
done
