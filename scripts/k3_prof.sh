# phase clocks of the tile-GEMM encoder (k3t, CTA 0) at C2: a profiling build, then the normal one
make -s -B -C paper_2201_12854_b200/csrc EXTRA=-DMCA_K3T_PROF=1 && \
MCA_K3_PROF=1 MCA_K3_TILE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/k3prof.json 2> gpurun_out/k3prof.err; echo rc=$?; grep "k3t CTA0" gpurun_out/k3prof.err | tail -3
make -s -B -C paper_2201_12854_b200/csrc
