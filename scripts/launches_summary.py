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
# everything inside the NVTX "mca_step" range is the forward (ours + the cuBLAS
# projection GEMM); K0 is one-time weight preparation (outside the range)
per_forward = lambda k: "k0_" not in k and "elementwise" not in k
tot = sum(sum(v) / len(v) for k, v in d.items() if per_forward(k))
print(f"{'kernel':50s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
for k, v in d.items():
    m = sum(v) / len(v)
    share = m / tot if per_forward(k) else 0
    print(f"{k:50s} {len(v):8d} {m:9.1f} {share:6.1%}")
