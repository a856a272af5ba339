# Every config's bench line (one B200) into gpurun_out/bench_<cfg>.json
for c in c2 c1 c4 c3; do
  steps=20; [ $c = c3 ] && steps=5
  timeout 600 python bench.py --config $c --steps $steps --warmup 5 --cpu-seconds 8 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo ${c}_rc=$?
done
timeout 300 python bench.py --steps 20 --warmup 5 --certify --no-cpu-baseline > gpurun_out/bench_c2_certify.json 2> gpurun_out/bench_c2_certify.err; echo c2cert_rc=$?
timeout 600 python bench.py --dtype f32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_f32.json 2> gpurun_out/bench_c2_f32.err; echo c2f32_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
