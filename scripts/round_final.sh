# Round-end evidence: every config's bench line, the launch list + ncu full capture of the default
# bench, the alpha sweep; outputs in gpurun_out/ (copied to profiles/r2 by hand)
bash scripts/bench_all.sh
python scripts/alpha_sweep.py --out gpurun_out/alpha_sweep.jsonl > gpurun_out/as.log 2>&1; echo sweep_rc=$?
bash scripts/profile_round.sh
bash scripts/launch_lists_fp32.sh > gpurun_out/ll_fp32.log 2>&1; echo fp32_lists_rc=$?
