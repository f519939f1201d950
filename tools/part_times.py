"""Time each ABI call of one Newton-iteration evaluation alone (CUDA events on the launching
stream, after warm-up), next to the composite cggm_newton_eval, to locate the latency-bound
parts of the step.  Prints one JSON line."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, colmajor_empty, newton_evaluation, to_device_colmajor  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--parts", default="")
args = ap.parse_args()

P = make_problem(args.config)
label, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
ctx = Context(0)
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
q = P.q
Sigma = colmajor_empty(q, q)
r0 = ctx.cggm_psi_grad(X, Y, T, ctx.cggm_invert_logdet(L, Sigma=Sigma)[0], Syy=Syy)
cnt = ctx.cggm_active_set(r0["GradL"], r0["GradT"], L, T, P.lam_L, P.lam_T)
bufs = {"Sigma": Sigma, "Psi": r0["Psi"], "GradL": r0["GradL"], "GradT": r0["GradT"]}
for k, c in (("L_row", cnt["m_L"]), ("L_col", cnt["m_L"]), ("T_row", cnt["m_T"]), ("T_col", cnt["m_T"])):
    bufs[k] = torch.empty(int(c) + 1024, dtype=torch.int32, device="cuda")

parts = {
    "invert": lambda: ctx.cggm_invert_logdet(L, Sigma=Sigma),
    "invert_nosigma": lambda: ctx.cggm_invert_logdet(L),
    "psi_grad": lambda: ctx.cggm_psi_grad(X, Y, T, Sigma, Syy=Syy, out=bufs),
    "active": lambda: ctx.cggm_active_set(bufs["GradL"], bufs["GradT"], L, T, P.lam_L, P.lam_T,
                                          cap_L=int(cnt["m_L"]) + 1024, cap_T=int(cnt["m_T"]) + 1024),
    "objective": lambda: ctx.cggm_objective(X, Y, L, T, P.lam_L, P.lam_T),
    "newton_eval": lambda: newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs),
}
res = {}
for name, fn in parts.items():
    if args.parts and name not in args.parts.split(","):
        continue
    try:
        fn()
        fn()
    except TypeError as e:  # binding signature differs: skip the part
        res[name] = f"skipped: {e}"
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(e0.elapsed_time(e1) / args.reps, 3)
print(json.dumps({"config": args.config, "ms": res}))
