"""Summarize an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel.

    python scripts/summarize_launches.py gpurun_out/launches.csv [--skip-first N]
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    m = re.search(r"(\w+_kernel|\w+Kernel|\w+_kernel<[^>]*>)", name)
    n = m.group(1) if m else name[:60]
    t = re.search(r"<([^>]*)>", name)
    return n + (f"<{t.group(1)}>" if t and "<" not in n else "")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0] != "ID"]
    per = defaultdict(lambda: defaultdict(float))
    launches = {}
    for r in rows:
        lid, name, metric, val = r[0], r[4], r[12], r[14]
        try:
            v = float(val.replace(",", ""))
        except ValueError:
            continue
        launches[lid] = name
        per[lid][metric] = v
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for lid, name in launches.items():
        k = short(name)
        a = agg[k]
        a[0] += 1
        a[1] += per[lid].get("gpu__time_duration.sum", 0.0)
        a[2] += per[lid].get("dram__bytes_read.sum", 0.0) + per[lid].get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | total ms | share | mean us/launch | DRAM MB/launch |")
    print(f"|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t / 1e6:.3f} | {t / total * 100:.1f}% | {t / n / 1e3:.1f} | {b / n / 1e6:.1f} |")
    print(f"\ntotal kernel time {total / 1e6:.3f} ms over {len(launches)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
