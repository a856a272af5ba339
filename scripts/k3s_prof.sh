# per-head CTA exit spread of the sampled encoder at C2 (+ per-head sample counts): profiling build, run, normal build
make -s -B -C paper_2201_12854_b200/csrc EXTRA=-DMCA_K3S_PROF=1 && \
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-chunks 1 > /dev/null 2> gpurun_out/k3sprof.err; echo rc=$?; grep "k3s heads" gpurun_out/k3sprof.err | tail -1 | tr '|' '\n'
make -s -B -C paper_2201_12854_b200/csrc
