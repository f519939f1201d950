"""FP32 variant of one Newton-iteration evaluation (ctx dtype f32: SIMT FFMA GEMM engine, fp32
factorisation) at a config: ms per evaluation, and agreement of the objective / log-det with fp64."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, newton_evaluation, to_device_colmajor  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", default="", help="f32 or f64: time one dtype only")
args = ap.parse_args()
P = make_problem(args.config)
_, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
out = {"config": args.config}
for dt, tdt in (("f32", torch.float32), ("f64", torch.float64)):
    if args.only and dt != args.only:
        continue
    ctx = Context(0, dtype=dt)
    X, Y = to_device_colmajor(P.X, dtype=tdt), to_device_colmajor(P.Y, dtype=tdt)
    L, T = DeviceCsc.from_host(lam, dtype=tdt), DeviceCsc.from_host(th, dtype=tdt)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    bufs = {}
    try:
        newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
    except Exception:
        pass
    mL, mT = ctx.last_active_sizes
    for k, c in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT)):
        bufs[k] = torch.empty(int(c) + 1024, dtype=torch.int32, device="cuda")
    for _ in range(2):   # eager, then the graph capture: the timed calls replay it
        r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
    e1.record()
    torch.cuda.synchronize()
    out[dt] = {"ms": round(e0.elapsed_time(e1) / args.reps, 2), "f": r["objective"]["f"], "logdet": r["logdet"],
               "m_L": r["active"]["m_L"], "m_T": r["active"]["m_T"]}
    del ctx, X, Y, L, T, Syy, bufs, r
    torch.cuda.empty_cache()
if not args.only:
    out["f_rel_diff"] = abs(out["f32"]["f"] - out["f64"]["f"]) / abs(out["f64"]["f"])
print(json.dumps(out))
