"""Summarise a multi-kernel `ncu --set full` report (scripts/profile_round.sh):
writes the markdown table for profiles/<round>/ncu_full_summary.md and the
per-stage DRAM traffic bench.py reports as roofline.traffic.

  python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/r1/ncu_full_summary.md profiles/traffic.json
"""
import csv
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time (us)", 1e6),      # scales apply to SI base values (s, bytes, counts)
    ("dram__bytes_read.sum", "DRAM read (MB)", 1e-6),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %", 1),
    ("smsp__inst_executed.sum", "warp instr (M)", 1e-6),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts (M)", 1e-6),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
]
UNIT = {"second": 1.0, "s": 1.0, "msecond": 1e-3, "ms": 1e-3, "usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9, "byte": 1.0, "Kbyte": 1e3,
        "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "inst": 1.0, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}
STAGE = {"k2c_certify": "budgets", "kp_project_tc": "projection", "k12_fused_tc": "score", "k1_scores_tc": "score", "k2_budgets": "budgets", "k2_scan": "budgets", "k2_scatter": "budgets", "k3_encode_sampled": "encode", "k3t_encode_tc": "encode",
         "k3b_exact_tc": "encode_exact", "k4_apply_tc": "apply"}


def main(rep, md_out, traffic_out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _, _ in METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    col = {m: hdr.index(m) for m, _, _ in METRICS if m in hdr}
    lines = ["| kernel | " + " | ".join(t for _, t, _ in METRICS) + " |", "|---" * (len(METRICS) + 1) + "|"]
    traffic = {}
    per_kernel = {}
    for r in rows[2:]:   # row 1 holds units
        if len(r) <= name_i:
            continue
        name = r[name_i].split("(")[0].replace("mca_dev::", "").replace("void ", "")
        vals = []

        def si(m):
            return float(r[col[m]].replace(",", "")) * UNIT.get(units[col[m]], 1.0)
        for m, _, scale in METRICS:
            try:
                f = si(m) * scale
                vals.append(f"{f:.0f}" if float(f).is_integer() or abs(f) >= 1e5 else f"{f:.1f}")
            except (ValueError, KeyError):
                vals.append("")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        base = name.split("<")[0]
        stage = next((v for k, v in STAGE.items() if base.startswith(k)), None)
        if stage and "dram__bytes_read.sum" in col:
            b = si("dram__bytes_read.sum") + si("dram__bytes_write.sum")
            tot, cnt = per_kernel.get((stage, base), (0.0, 0))
            per_kernel[(stage, base)] = (tot + b, cnt + 1)
    # per launch: a kernel captured several times (one per profiled step) is
    # averaged over its launches, then a stage sums its distinct kernels
    for (stage, _), (tot, cnt) in per_kernel.items():
        traffic[stage] = traffic.get(stage, 0.0) + tot / cnt
    with open(md_out, "w") as f:
        f.write("# ncu --set full summary (C2 bf16, one launch of each kernel of one step; cold-cache, serialised)\n\n")
        f.write(f"Source: `{rep.split('/')[-1]}` from scripts/profile_round.sh.\n\n")
        f.write("\n".join(lines) + "\n")
    with open(traffic_out, "w") as f:
        json.dump({k: traffic[k] for k in sorted(traffic)}, f, indent=1)
    print("\n".join(lines))
    print(json.dumps(traffic))


if __name__ == "__main__":
    main(*sys.argv[1:4])
