# timeline of K3b's CTA (0, 0) at C2: profiling build, run, normal build
make -s -B -C paper_2201_12854_b200/csrc EXTRA=-DMCA_K3B_PROF=1 && \
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-chunks 1 > /dev/null 2> gpurun_out/k3bprof.err; echo rc=$?; grep "k3b CTA0" gpurun_out/k3bprof.err | tail -2
make -s -B -C paper_2201_12854_b200/csrc
