# usage: bash scripts/profile_one.sh <kernel-regex> <tag> [launches-to-skip (default 2)]
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "mca_step/" --set full --clock-control none --import-source on -k regex:"$1" -s "${3:-2}" -c 1 -o gpurun_out/prof_$2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$2.log 2>&1; echo ncu_rc=$?
