# timeline of K4's first CTA (softmax thread 0) at C2: profiling build, run, normal build
make -s -B -C paper_2201_12854_b200/csrc EXTRA=-DMCA_K4_PROF=1 && \
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-chunks 1 > gpurun_out/k4prof.json 2> gpurun_out/k4prof.err; echo rc=$?; grep "k4 CTA0" gpurun_out/k4prof.err | tail -2
make -s -B -C paper_2201_12854_b200/csrc
