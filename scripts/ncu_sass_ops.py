"""Executed warp-instructions per SASS opcode (and top source lines) of an ncu
report: python scripts/ncu_sass_ops.py rep.ncu-rep [samples_per_launch]"""
import collections, csv, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
st = hdr.index("Warp Stall Sampling (All Samples)")
tot = 0
byop, stall = collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    byop[op] += n
    tot += n
    try:
        stall[op] += int(r[st])
    except ValueError:
        pass
per = float(sys.argv[2]) if len(sys.argv) > 2 else 0
print("total warp instructions", tot, f"per unit {tot / per:.2f}" if per else "")
for op, n in byop.most_common(30):
    print(f"{op:12s} {n:12d} {n / tot * 100:5.1f}%  stall samples {stall[op]}")
