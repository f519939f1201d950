"""Windowed view of a timeline CSV (tools/timeline.py --out): per W-ms window, each stream's busy
fraction and its dominant tag, plus the fraction of the window in which only kernels shorter
than 0.2 ms are in flight (latency-bound stretches)."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.csv"
W = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
rows = list(csv.DictReader(open(path)))
t_end = max(float(r["end_ms"]) for r in rows)
streams = sorted({r["stream"] for r in rows}, key=lambda s: min(float(r["start_ms"]) for r in rows if r["stream"] == s))
sid = {s: i for i, s in enumerate(streams)}
nb = int(t_end / W) + 1
busy = [[0.0] * nb for _ in streams]
tagt = [[collections.Counter() for _ in range(nb)] for _ in streams]
bin_ms = 0.02
nfine = int(t_end / bin_ms) + 1
big = [False] * nfine
anyk = [False] * nfine
for r in rows:
    a, b, s, tag = float(r["start_ms"]), float(r["end_ms"]), sid[r["stream"]], r["tag"]
    for w in range(int(a / W), min(nb, int(b / W) + 1)):
        lo, hi = max(a, w * W), min(b, (w + 1) * W)
        if hi > lo:
            busy[s][w] += hi - lo
            tagt[s][w][tag] += hi - lo
    for i in range(int(a / bin_ms), min(nfine, int(b / bin_ms) + 1)):
        anyk[i] = True
        if b - a >= 0.2:
            big[i] = True
print(f"span {t_end:.1f} ms, {len(rows)} launches, streams in order of first launch: {len(streams)}")
hdr = "window(ms)  " + "  ".join(f"s{i:<2}          " for i in range(len(streams))) + " short-only"
print(hdr)
for w in range(nb):
    cells = []
    for s in range(len(streams)):
        f = busy[s][w] / W
        top = tagt[s][w].most_common(1)
        cells.append(f"{f:4.2f} {top[0][0][:9]:9s}" if top else " " * 14)
    lo, hi = int(w * W / bin_ms), min(nfine, int((w + 1) * W / bin_ms))
    so = sum(1 for i in range(lo, hi) if anyk[i] and not big[i]) * bin_ms / W
    idle = sum(1 for i in range(lo, hi) if not anyk[i]) * bin_ms / W
    print(f"{w * W:6.0f}-{(w + 1) * W:<5.0f} " + " ".join(cells) + f"  {so:4.2f} idle {idle:4.2f}")
