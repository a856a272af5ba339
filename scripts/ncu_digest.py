"""Print the headline metrics of an ncu report: python scripts/ncu_digest.py rep.ncu-rep"""
import csv, subprocess, sys

KEYS = ("Duration", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy", "SM Busy", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Achieved Occupancy", "Registers Per Thread",
        "No Eligible", "One or More Eligible", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Dynamic Shared Memory Per Block")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mn, mu, mv = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
seen = set()
for r in rows[1:]:
    if len(r) <= mv or r[mn] in seen:
        continue
    if any(k == r[mn] for k in KEYS):
        seen.add(r[mn])
        print(f"{r[mn]:40s} {r[mv]:>14s} {r[mu]}")
