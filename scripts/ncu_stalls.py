"""Per-kernel warp-stall breakdown (share of sampled stall reasons) from an
`ncu --set full` report: python scripts/ncu_stalls.py rep.ncu-rep > profiles/r1/ncu_stalls.md"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki = hdr.index("Kernel Name")
cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
print("# Warp-stall reasons per kernel (share of PC samples; C2 bf16, one launch each)\n")
print("| kernel | top reasons |")
print("|---|---|")
seen = set()
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("mca_dev::", "").replace("void ", "")
    if name in seen or len(r) <= max(cols):
        continue
    seen.add(name)
    vals = []
    for i in cols:
        try:
            vals.append((float(r[i].replace(",", "")), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    tot = sum(v for v, _ in vals) or 1.0
    top = sorted(vals, reverse=True)[:6]
    print(f"| {name} | " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top) + " |")
