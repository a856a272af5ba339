# e2e vs HostPipeline chunk count, both input modes (no CPU baseline)
for inp in x qkx; do for c in 2 4 8; do
timeout 300 python bench.py --inputs $inp --e2e-chunks $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bc_${inp}_$c.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/bc_${inp}_$c.json'));print('$inp', $c, round(d['value']), round(d['e2e']['value']))"
done; done
