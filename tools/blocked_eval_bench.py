"""NEXT-4 measurement: cggm_newton_eval_blocked (no dense Sigma / Psi / gradients) at a config, per
block width: ms per evaluation and the device memory the evaluation holds (cudaMemGetInfo after a
warm call, i.e. inputs + the library's workspace), next to the dense composite evaluation.  One
JSON line."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, colmajor_empty, to_device_colmajor  # noqa
from paper_1509_04681_b200.api import newton_evaluation  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--blocks", default="2048,4096")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--dense", type=int, default=1)
args = ap.parse_args()
P = make_problem(args.config)
_, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
free0, total = torch.cuda.mem_get_info()
res = {"config": args.config, "n": P.n, "p": P.p, "q": P.q, "device_total_gb": round(total / 2**30, 1)}


def used_gb():
    f, t = torch.cuda.mem_get_info()
    return round((t - f) / 2**30, 2)


for b in (int(v) for v in args.blocks.split(",")):
    ctx = Context(0)
    bufs = {k: torch.empty(0, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")}
    try:
        ctx.cggm_newton_eval_blocked(X, Y, L, T, P.lam_L, P.lam_T, block=b, bufs=bufs)
    except Exception as exc:
        if getattr(exc, "status", None) != 6:
            raise
    mL, mT = ctx.last_active_sizes
    for k, cap in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT)):
        bufs[k] = torch.empty(int(cap) + 1024, dtype=torch.int32, device="cuda")
    r = ctx.cggm_newton_eval_blocked(X, Y, L, T, P.lam_L, P.lam_T, block=b, bufs=bufs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        r = ctx.cggm_newton_eval_blocked(X, Y, L, T, P.lam_L, P.lam_T, block=b, bufs=bufs)
    torch.cuda.synchronize()
    res[f"blocked_b{b}_ms"] = round((time.perf_counter() - t0) / args.reps * 1e3, 1)
    res[f"blocked_b{b}_device_used_gb"] = used_gb()
    res[f"blocked_b{b}_f"] = r["objective"]["f"]
    res[f"blocked_b{b}_m"] = [r["active"]["m_L"], r["active"]["m_T"]]
    ctx.close()
    del bufs
    torch.cuda.empty_cache()
def dense_leg():
    ctx = Context(0)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    mk = next(k for k in res if k.endswith("_m"))
    mL, mT = res[mk]
    bufs = {k: torch.empty(int(c) + 1024, dtype=torch.int32, device="cuda")
            for k, c in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT))}
    r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
    torch.cuda.synchronize()
    res["dense_ms"] = round((time.perf_counter() - t0) / args.reps * 1e3, 1)
    res["dense_device_used_gb"] = used_gb()
    res["dense_f"] = r["objective"]["f"]
    res["dense_m"] = [r["active"]["m_L"], r["active"]["m_T"]]


if args.dense:
    try:
        dense_leg()
    except Exception as exc:   # the dense evaluation beyond one GPU's capacity
        res["dense_error"] = f"{type(exc).__name__}: {str(exc)[:200]}"
print(json.dumps(res))
