# C2 in both input modes (q, k, x given / x only with device projections)
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 4 > gpurun_out/bench_qkx.json 2> gpurun_out/bench_qkx.err; echo qkx_rc=$?
timeout 300 python bench.py --inputs x --steps 10 --warmup 3 --cpu-seconds 4 > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err; echo x_rc=$?
tail -2 gpurun_out/bench_x.err
