# round-2 check: GPU tests, default bench, c1 (fp32), c3 (24 layers), c4, and --gpus 2 on a 1-GPU box
#timeout 800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t.log
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 3 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; echo c2_rc=$?; tail -2 gpurun_out/b_c2.err
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --cpu-seconds 3 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo c1_rc=$?; tail -2 gpurun_out/b_c1.err
timeout 400 python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; echo c3_rc=$?; tail -2 gpurun_out/b_c3.err
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --cpu-seconds 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo c4_rc=$?; tail -2 gpurun_out/b_c4.err
timeout 60 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/b_g2.json 2> gpurun_out/b_g2.err; echo g2_rc=$?; tail -2 gpurun_out/b_g2.err
