for cfg in "4 2" "3 4" "3 3"; do set -- $cfg
make -s -C paper_2201_12854_b200/csrc EXTRA="-DKP_STAGES_256=$1 -DKP_OUTBUFS_256=$2" > /dev/null 2>&1 || { echo build_fail; continue; }
ncu --nvtx --nvtx-include "mca_step/" --metrics gpu__time_duration.sum --clock-control none -k regex:kp_project -c 4 --csv --log-file gpurun_out/kp.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-regular > /dev/null 2>&1; echo "stages=$1 outbufs=$2 rc=$?"
python scripts/launches_summary.py gpurun_out/kp.csv | tail -1
touch paper_2201_12854_b200/csrc/kp_project_tc.cu
done
