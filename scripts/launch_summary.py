"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    n = re.sub(r"\(.*", "", d["Kernel Name"])[:60]
    v = float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(t for _, t in agg.values())
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:60s} {c:6d} calls {t / div:10.1f} us/iter {t / c:8.2f} us/call {100 * t / tot:5.1f}%")
print(f"total {tot / div:.1f} us/iter")
