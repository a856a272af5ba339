"""Warp-stall samples (with the top stall reasons) and executed instructions
per CUDA source line of an ncu report (needs -lineinfo + --import-source):
  python scripts/ncu_cuda_lines.py rep.ncu-rep [N]"""
import csv, subprocess, sys

N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, res = "?", None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    st, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    reasons = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
    try:
        rs = sorted(((int(r[i] or 0), c[6:]) for i, c in reasons), reverse=True)[:3]
        res.append((int(r[st] or 0), int(r[ie] or 0), f"{fname}:{r[0]}", r[1].strip()[:70], rs))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in res) or 1
print("total stall samples", tot, "instructions", sum(x[1] for x in res))
for s, n, where, text, rs in sorted(res, key=lambda x: -x[0])[:N]:
    why = " ".join(f"{c}:{v}" for v, c in rs if v)
    print(f"{s:6d} {s / tot * 100:5.1f}% {n:10d} {where:26s} {text:70s} {why}")
