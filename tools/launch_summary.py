"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    u = r[unit_i] if unit_i is not None else "ns"
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
    name = r[ki].split("(")[0][:90]
    agg[name][0] += 1
    agg[name][1] += v * scale
    total += v * scale
print(f"{'kernel':90s} {'launches':>9s} {'ms':>10s} {'share':>7s}")
for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:90s} {n:9d} {ms:10.3f} {100 * ms / total:6.1f}%")
print(f"{'TOTAL':90s} {sum(v[0] for v in agg.values()):9d} {total:10.3f}")
