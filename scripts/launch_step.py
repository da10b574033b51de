"""Cut one training step out of an ncu --csv launch list (gpu__time_duration.sum) of
`scripts/kprof_step.py --no-prof` (eager steps, each ending with one adam_kernel):
the launches after the (n-1)-th adam_kernel up to the n-th, written as a csv, and a
per-kernel summary with each kernel's share of the step.

    python scripts/launch_step.py launches.csv step.csv [n]
"""
import collections
import csv
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
rows = list(csv.reader(open(src)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[hdr]
ki, mi, vi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
data = [r for r in rows[hdr + 1:] if len(r) == len(H) and r[mi] == "gpu__time_duration.sum"]
ends = [i for i, r in enumerate(data) if "adam_kernel" in r[ki]]
step = data[ends[n - 2] + 1:ends[n - 1] + 1]
with open(dst, "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(H)
    w.writerows(step)
unit_ms = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[step[0][H.index("Metric Unit")]]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in step:
    k = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", "")) * unit_ms
tot = sum(t for _, t in agg.values())
print(f"{len(step)} kernel launches, {tot:.2f} ms of serialised kernel time")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{k[:62]:62s} {c:5d} calls {t * 1e3:10.1f} us {t / c * 1e3:9.2f} us/call {100 * t / tot:5.1f}%")
