"""Bucket an ncu launch list (gpu__time_duration.sum + launch__grid_size) by kernel kind and grid size."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ID, K, M, V = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
L = {}
for r in rows[hi + 1:]:
    if len(r) <= V:
        continue
    d = L.setdefault(r[ID], {"k": r[K].split("(")[0]})
    d[r[M]] = float(r[V].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for d in L.values():
    g = int(d.get("launch__grid_size", 0))
    t = d["gpu__time_duration.sum"] / 1e6  # ns -> ms
    k = d["k"]
    kind = "leaf" if "leaf" in k else "small" if "small" in k else "gemm64" if "64, 64" in k else \
        "gemm128" if "128, 128" in k else k.split("::")[-1][:30]
    b = "g<=37" if g <= 37 else "g<=148" if g <= 148 else "g<=592" if g <= 592 else "big"
    agg[(kind, b)][0] += 1
    agg[(kind, b)][1] += t
    tot += t
for (kind, b), (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{kind:32s} {b:7s} {n:6d} {ms:9.2f} ms  avg {1000 * ms / n:8.1f} us")
print(f"total {tot:.2f} ms, {len(L)} launches")
