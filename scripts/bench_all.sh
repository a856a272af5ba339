# Round measurements: every config + the alpha sweep + the reference arm.
set -x
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --dtype f32 --steps 10 --warmup 3 --cpu-seconds 3 > gpurun_out/bench_c2_f32.json 2> gpurun_out/bench_c2_f32.err
timeout 300 python scripts/alpha_sweep.py --out gpurun_out/alpha_sweep.jsonl > gpurun_out/alpha_sweep.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for f in gpurun_out/bench_*.json; do echo "== $f"; cut -c1-400 $f; done
tail -n 3 gpurun_out/*.err
