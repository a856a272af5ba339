# A/B of a k12 compile-time switch on one box: bash scripts/k12_ab.sh "-DMCA_K12_POLL=0" "-DMCA_K12_POLL=1"
for v in "$@" "$@"; do
  make -s -B -C paper_2201_12854_b200/csrc EXTRA="$v" >/dev/null
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})"
done
make -s -B -C paper_2201_12854_b200/csrc >/dev/null
