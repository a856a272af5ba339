"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: mean
device time per kernel (cold-cache, serialised launches: compare shares)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3,
              "second": v * 1e6, "s": v * 1e6}.get(unit, v)
        name = r[ki].split("(")[0].replace("void ", "")[:48]
        d.setdefault(name, []).append(us)
# everything inside the NVTX "mca_step" range is the forward; K0 is one-time
# weight preparation (outside the range). A kernel launched twice per step with
# very different durations (kp_project_tc: the q / k GEMM and the dense-exact
# GEMM that exits at once unless K2's exact fraction >= 12%) is split into
# "(long)" and "(exit)" rows so the means stay per launch.
per_forward = lambda k: "k0_" not in k and "elementwise" not in k
rows = OrderedDict()
for k, v in d.items():
    short = [x for x in v if x < 5.0]
    if short and len(short) < len(v):
        rows[k + " (long)"] = [x for x in v if x >= 5.0]
        rows[k + " (exit)"] = short
    else:
        rows[k] = v
tot = sum(sum(v) / len(v) * (len(v) / max(len(d[next(iter(d))]), 1)) for k, v in rows.items() if per_forward(k))
steps = min(len(v) for k, v in rows.items() if per_forward(k))
tot = sum(sum(v) / steps for k, v in rows.items() if per_forward(k))   # device time per step
print(f"{'kernel':56s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
for k, v in rows.items():
    m = sum(v) / len(v)
    share = (sum(v) / steps) / tot if per_forward(k) else 0
    print(f"{k:56s} {len(v):8d} {m:9.1f} {share:6.1%}")
