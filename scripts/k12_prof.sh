# timeline of the fused score + budget kernel at C2 (CTA 0's blocks, every CTA's SM / start / end):
# profiling build, run, normal build
make -s -B -C paper_2201_12854_b200/csrc EXTRA=-DMCA_K12_PROF=1 && \
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-chunks 1 > gpurun_out/k12prof.json 2> gpurun_out/k12prof.err; echo rc=$?; grep "k12 CTA0" gpurun_out/k12prof.err | tail -4
python scripts/k12_ctas.py gpurun_out/k12prof.err
make -s -B -C paper_2201_12854_b200/csrc
