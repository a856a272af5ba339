# CUDA-graph replay of repeated forwards (MCA_GRAPHS=1): GPU tests, then C1 / C2 with and without
MCA_GRAPHS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_mcam_cli.py -m gpu -q -p no:cacheprovider -x > gpurun_out/graphs_tests.log 2>&1; echo graph_tests_rc=$?; tail -3 gpurun_out/graphs_tests.log
for g in 0 1; do for c in c1 c2; do
  MCA_GRAPHS=$g timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_$c.json 2>gpurun_out/g_$c.err
  python -c "import json;d=json.load(open('gpurun_out/g_$c.json'));print('graphs=$g', '$c', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']/1e6,3), d['gpu_launches'])" || tail -3 gpurun_out/g_$c.err
done; done
