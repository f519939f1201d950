"""Time sharded.DistributedInverse on ONE GPU (world size 1: the same blocked algorithm and
building-block calls a rank runs, without the exchanges) at a config's Lambda, next to the
single-call cggm_invert_logdet.  The per-rank time at G ranks is about this / G + the exchanges."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc  # noqa
from paper_1509_04681_b200.sharded import CudaBackend, DistributedInverse  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--blocks", default="1024,2048,4096")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
P = make_problem(args.config)
lam = [pt for pt in P.points if pt[0] == "truth"][0][1]
ctx = Context(0)
L = DeviceCsc.from_host(lam)
q = P.q
res = {"config": args.config, "q": q}


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / args.reps * 1e3, out


ms, r1 = timed(lambda: ctx.cggm_invert_logdet(L))
res["invert_logdet_ms"] = round(ms, 2)
for b in (int(v) for v in args.blocks.split(",")):
    di = DistributedInverse(CudaBackend(ctx), block=b)
    ms, r = timed(lambda: di.invert(L))
    S, ld, pd, _ = r
    err = float((S - r1[0]).abs().max() / r1[0].abs().max())
    res[f"distributed_b{b}_ms"] = round(ms, 2)
    res[f"distributed_b{b}_tflops"] = round(4.0 / 3.0 * q ** 3 / ms / 1e9, 2)
    res[f"distributed_b{b}_maxrel_vs_single"] = err
    res[f"distributed_b{b}_logdet_diff"] = abs(ld - r1[1])
print(json.dumps(res))
