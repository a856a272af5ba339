for hint in 0 1 2; do
make -s -C paper_2201_12854_b200/csrc EXTRA="-DKP_STORE_HINT=$hint" > /dev/null 2>&1 || { echo build_fail; continue; }
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -c 14 --csv --log-file gpurun_out/kp.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1; echo "hint=$hint rc=$?"
python scripts/launches_summary.py gpurun_out/kp.csv | grep -E "kp_|k12"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-regular 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],4))"
touch paper_2201_12854_b200/csrc/kp_project_tc.cu
done
