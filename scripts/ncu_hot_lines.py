"""Top SASS lines of an ncu report by warp-stall samples, with CUDA source
line when available: python scripts/ncu_hot_lines.py rep.ncu-rep [N]"""
import csv, subprocess, sys

N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr, start = r, i + 1
        break
src, st, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows[start:]:
    try:
        lines.append((int(r[st]), int(r[ie] or 0), r[src][:110], r[0][:60]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in lines)
for s, n, text, addr in sorted(lines, reverse=True)[:N]:
    print(f"{s:7d} {s / max(tot, 1) * 100:5.1f}% {n:11d}  {addr:>8s}  {text}")
