# K4 per-block timeline of CTA 0's second tile (MCA_K4_PROF build): clocks relative to kernel start
cp paper_2201_12854_b200/lib/libmca_b200.so /tmp/libmain.so
cp paper_2201_12854_b200/lib_exp/libk4prof.so paper_2201_12854_b200/lib/libmca_b200.so
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular 2>&1 >/dev/null | grep "k4 CTA0" | tail -2
cp /tmp/libmain.so paper_2201_12854_b200/lib/libmca_b200.so
