"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, mean, share."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > vi:
        d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) / 1e6)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):4d} mean={sum(v) / len(v):9.4f} ms share={sum(v) / tot:.3f}")
