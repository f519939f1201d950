"""Join an ncu launch list (gpu__time_duration.sum) with CGGM_GEMM_LOG lines: per-launch FP64
efficiency of every TMA GEMM launch, bucketed by grid size and tile."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ID, K, M, V = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
L = {}
for r in rows[hi + 1:]:
    if len(r) <= V:
        continue
    d = L.setdefault(int(r[ID]), {"k": r[K]})
    d[r[M]] = float(r[V].replace(",", ""))
dmma = [L[i] for i in sorted(L) if "gemm_dmma_kernel" in L[i]["k"]]
logs = [l for l in open(sys.argv[2]) if l.startswith("GEMMLOG")][-len(dmma):]
assert len(logs) == len(dmma), (len(logs), len(dmma))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot_t = tot_f = 0.0
worst = []
for d, l in zip(dmma, logs):
    kv = dict(re.findall(r"(\w+)=([\w.+\-x]+)", l))
    t = d["gpu__time_duration.sum"] * 1e-9
    f = float(kv["exec_flops"])
    g = int(kv["grid"])
    b = "g<=148" if g <= 148 else "g<=592" if g <= 592 else "g<=2048" if g <= 2048 else "big"
    key = (kv["tile"], b)
    agg[key][0] += 1
    agg[key][1] += t
    agg[key][2] += f
    tot_t += t
    tot_f += f
    worst.append((t * (1 - (f / t / 37.1e12)), t, f / t / 1e12, l.strip()[8:]))
print(f"{'tile':8s} {'grid':8s} {'n':>5s} {'ms':>9s} {'TF/s':>7s}")
for (tile, b), (n, t, f) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{tile:8s} {b:8s} {n:5d} {1e3 * t:9.2f} {f / t / 1e12:7.2f}")
print(f"TOTAL {1e3 * tot_t:.2f} ms, {tot_f / tot_t / 1e12:.2f} TF/s")
print("largest losses vs 37.1 TF/s (ms lost, ms, TF/s, launch):")
for w in sorted(worst, reverse=True)[:15]:
    print(f"  {1e3 * w[0]:7.2f} {1e3 * w[1]:8.2f} {w[2]:6.2f}  {w[3]}")
print("largest losses among the non-'big' launches (grid <= 2048 CTAs):")
small = [w for w in worst if "grid=" in w[3] and int(re.search(r"grid=(\d+)", w[3]).group(1)) <= 2048]
for w in sorted(small, reverse=True)[:25]:
    print(f"  {1e3 * w[0]:7.2f} {1e3 * w[1]:8.2f} {w[2]:6.2f}  {w[3]}")
