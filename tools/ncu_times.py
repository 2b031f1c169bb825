"""Per-kernel durations from an `ncu --metrics gpu__time_duration.sum --csv`
log: python tools/ncu_times.py log.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
acc = defaultdict(list)
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    acc[r[ki].split("(")[0][:60]].append(v * scale)
for k, v in acc.items():
    print(f"{k:60s} n={len(v):3d} mean {sum(v) / len(v):9.2f} us  min {min(v):9.2f}")
