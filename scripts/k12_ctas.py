"""Summarise the per-CTA timeline a MCA_K12_PROF build prints ("k12 CTAS" lines)."""
import statistics
import sys
from collections import defaultdict

line = [l for l in open(sys.argv[1]) if l.startswith("k12 CTAS")][-1]
ctas = [tuple(int(v) for v in t.split(":")) for t in line.split()[2:]]
span = max(c[2] for c in ctas)
dur = [c[2] - c[1] for c in ctas]
cyc = [c[3] for c in ctas]
per_sm = defaultdict(list)
for i, c in enumerate(ctas):
    per_sm[c[0]].append(c)
gaps, busy = [], []
for sm, lst in per_sm.items():
    lst.sort(key=lambda c: c[1])
    busy.append(sum(c[2] - c[1] for c in lst))
    for x, y in zip(lst, lst[1:]):
        gaps.append(y[1] - x[2])
q = lambda v, f: sorted(v)[int(f * (len(v) - 1))]  # noqa: E731
print(f"CTAs {len(ctas)} on {len(per_sm)} SMs; kernel span {span / 1e3:.1f} us")
print(f"CTA ns: min {min(dur)} p10 {q(dur, .1)} med {statistics.median(dur):.0f} p90 {q(dur, .9)} max {max(dur)}")
print(f"CTA cycles: min {min(cyc)} med {statistics.median(cyc):.0f} max {max(cyc)}")
cnt = defaultdict(int)
for lst in per_sm.values():
    cnt[len(lst)] += 1
print("CTAs per SM:", dict(sorted(cnt.items())))
print(f"inter-CTA gap ns: med {statistics.median(gaps):.0f} p90 {q(gaps, .9)} max {max(gaps)}" if gaps else "")
print(f"SM busy fraction of span: mean {statistics.mean(busy) / span:.3f} min {min(busy) / span:.3f}")
starts = sorted(c[1] for c in ctas)
print("first-wave start spread ns:", starts[147] - starts[0], " last start", starts[-1], " last end", span)
for w in range(0, len(ctas), 148):
    seg = sorted(ctas, key=lambda c: c[1])[w:w + 148]
    print(f"wave {w // 148}: start {min(c[1] for c in seg) / 1e3:.1f}-{max(c[1] for c in seg) / 1e3:.1f} us,"
          f" end {min(c[2] for c in seg) / 1e3:.1f}-{max(c[2] for c in seg) / 1e3:.1f} us")
