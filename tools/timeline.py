"""Timeline of one composite Newton-iteration evaluation (per-launch CUDA events on every stream,
cggm_test_profile_dump), summarised per stream: span, busy time, and the time in which each stream
is the only one with a kernel in flight.  Profiling events perturb the schedule slightly."""
import argparse
import collections
import csv
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, colmajor_empty, newton_evaluation, to_device_colmajor  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
ap.add_argument("--out", default="gpurun_out/timeline.csv")
args = ap.parse_args()
P = make_problem(args.config)
label, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
ctx = Context(0, dtype=args.dtype)
dt = torch.float32 if args.dtype == "f32" else torch.float64
X, Y = to_device_colmajor(P.X, dtype=dt), to_device_colmajor(P.Y, dtype=dt)
L, T = DeviceCsc.from_host(lam, dtype=dt), DeviceCsc.from_host(th, dtype=dt)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
q = P.q
bufs = {}
try:  # two-call pattern: the first call reports the list sizes
    newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
except Exception:
    pass
mL, mT = ctx.last_active_sizes
for k, c in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT)):
    bufs[k] = torch.empty(int(c) + 1024, dtype=torch.int32, device="cuda")
for _ in range(2):
    newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
torch.cuda.synchronize()
ctx.profile(True)
newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
torch.cuda.synchronize()
if os.environ.get("CGGM_GRAPH_PROF") == "1":   # second profiled call captures a graph with the events
    ctx.profile(True)
    newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
    torch.cuda.synchronize()
ctx._check(ctx.lib.cggm_test_profile_dump(ctx.h, args.out.encode()))
ctx.profile(False)

rows = list(csv.DictReader(open(args.out)))
by = collections.defaultdict(list)
for r in rows:
    by[int(r["stream"])].append((float(r["start_ms"]), float(r["end_ms"]), r["tag"]))
t_end = max(e for v in by.values() for _, e, _ in v)
print(f"step span {t_end:.2f} ms, {len(rows)} launches")
# 0.05 ms bins: which streams are busy
nb = int(t_end / 0.05) + 1
busy = {s: [False] * nb for s in by}
for s, v in by.items():
    for a, b, _ in v:
        for i in range(int(a / 0.05), min(nb, int(b / 0.05) + 1)):
            busy[s][i] = True
for s, v in sorted(by.items()):
    tags = collections.Counter(t for _, _, t in v)
    alone = sum(1 for i in range(nb) if busy[s][i] and not any(busy[o][i] for o in by if o != s)) * 0.05
    print(f"stream {s}: {len(v)} launches, span {min(a for a, _, _ in v):.2f}-{max(b for _, b, _ in v):.2f} ms, "
          f"busy {sum(busy[s]) * 0.05:.2f} ms, alone {alone:.2f} ms, tags {dict(tags.most_common(4))}")
idle = sum(1 for i in range(nb) if not any(busy[s][i] for s in by)) * 0.05
print(f"no kernel in flight: {idle:.2f} ms")
# short-kernel-only time: bins where every in-flight kernel is shorter than 0.2 ms
short = [True] * nb
anyk = [False] * nb
for s, v in by.items():
    for a, b, _ in v:
        for i in range(int(a / 0.05), min(nb, int(b / 0.05) + 1)):
            anyk[i] = True
            if b - a >= 0.2:
                short[i] = False
print(f"only short (<0.2 ms) kernels in flight: {sum(1 for i in range(nb) if anyk[i] and short[i]) * 0.05:.2f} ms")
