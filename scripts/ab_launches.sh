# Launch-list A/B of compile-time switches on one box (ncu serialised kernel times):
#   bash scripts/ab_launches.sh "-DFOO=0" "-DFOO=1"
for v in "$@" "$@"; do
  make -s -B -C paper_2201_12854_b200/csrc EXTRA="$v" >/dev/null
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
      --log-file gpurun_out/ab_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "== $v"; python scripts/launches_summary.py gpurun_out/ab_launches.csv | tail -7
done
make -s -B -C paper_2201_12854_b200/csrc >/dev/null
