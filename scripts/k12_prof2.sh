# K12 timeline at C2 (768 items): CTA 0's blocks and the per-CTA spread
make -s -B -C paper_2201_12854_b200/csrc EXTRA="-DMCA_K12_PROF=1 $1"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-chunks 1 > /dev/null 2> gpurun_out/k12prof_c2.err
grep "k12 CTA0" gpurun_out/k12prof_c2.err | tail -2 | cut -c1-900; python scripts/k12_ctas.py gpurun_out/k12prof_c2.err > gpurun_out/k12ctas_c2.txt; head -6 gpurun_out/k12ctas_c2.txt
make -s -B -C paper_2201_12854_b200/csrc
