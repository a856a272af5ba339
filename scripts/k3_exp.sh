timeout 800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fp16 or bf16_parity or graph" > gpurun_out/t.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/t.log
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
(cd _old && python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', round(d['ms_per_step'],4), round(d['stages_ms']['encode'],4))")
done
