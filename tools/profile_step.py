"""Run exactly one Newton-iteration evaluation of a config inside cudaProfilerStart/Stop, after
warm-up, for `ncu --profile-from-start off` launch lists and captures.  Also prints the step's
wall time measured with CUDA events (no profiling events inside the library)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, colmajor_empty, newton_evaluation, to_device_colmajor  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--part", default="all", choices=["all", "invert", "psi", "objective", "active"])
ap.add_argument("--no-grad-theta", action="store_true", help="GradT = NULL (K01: S_Theta selected in the X^T E epilogue)")
args = ap.parse_args()

P = make_problem(args.config)
label, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
ctx = Context(0, dtype=args.dtype)
dt = torch.float32 if args.dtype == "f32" else torch.float64
X, Y = to_device_colmajor(P.X, dtype=dt), to_device_colmajor(P.Y, dtype=dt)
L, T = DeviceCsc.from_host(lam, dtype=dt), DeviceCsc.from_host(th, dtype=dt)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
q, p = P.q, P.p
Sigma = colmajor_empty(q, q, dtype=dt)
r0 = ctx.cggm_psi_grad(X, Y, T, ctx.cggm_invert_logdet(L, Sigma=Sigma)[0], Syy=Syy)
cnt = ctx.cggm_active_set(r0["GradL"], r0["GradT"], L, T, P.lam_L, P.lam_T)
bufs = {"Sigma": Sigma, "Psi": r0["Psi"], "GradL": r0["GradL"], "GradT": r0["GradT"]}
for k, c in (("L_row", cnt["m_L"]), ("L_col", cnt["m_L"]), ("T_row", cnt["m_T"]), ("T_col", cnt["m_T"])):
    bufs[k] = torch.empty(int(c) + 1024, dtype=torch.int32, device="cuda")


def step():
    if args.part == "all":
        newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=args.no_grad_theta)
    elif args.part == "invert":
        ctx.cggm_invert_logdet(L, Sigma=Sigma)
    elif args.part == "psi":
        ctx.cggm_psi_grad(X, Y, T, Sigma, Syy=Syy, out=bufs)
    elif args.part == "active":
        ctx.cggm_active_set(bufs["GradL"], bufs["GradT"], L, T, P.lam_L, P.lam_T,
                            cap_L=int(cnt["m_L"]) + 1024, cap_T=int(cnt["m_T"]) + 1024)
    else:
        ctx.cggm_objective(X, Y, L, T, P.lam_L, P.lam_T)


for _ in range(args.warmup):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
l0 = ctx.launch_count()
torch.cuda.profiler.start()
e0.record()
for _ in range(args.steps):
    step()
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"part={args.part} ms_per_step={e0.elapsed_time(e1) / args.steps:.2f} launches_per_step="
      f"{(ctx.launch_count() - l0) / args.steps:.0f}")
