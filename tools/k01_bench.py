"""grad_Theta forms of the composite evaluation at a config: stored (p x q), not stored with S_Theta
selected in the X^T E epilogue (K01, the FP64 default for GradT = NULL), and -- with CGGM_K01=0 in the
environment -- not stored, streamed in 2048-column chunks through the scan.  ms per evaluation
(CUDA events around `reps` graph replays) and the list sizes / statistic of each."""
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
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
P = make_problem(args.config)
_, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
ctx = Context(0)
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
q, p = P.q, P.p
bufs = {"Sigma": colmajor_empty(q, q), "Psi": colmajor_empty(q, q), "GradL": colmajor_empty(q, q)}
for k in ("L_row", "L_col", "T_row", "T_col"):
    bufs[k] = torch.empty(0, dtype=torch.int32, device="cuda")
try:
    newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=True)
except Exception:
    pass
mL, mT = ctx.last_active_sizes
for k, c in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT)):
    bufs[k] = torch.empty(int(c * 1.1) + 1024, dtype=torch.int32, device="cuda")
out = {"config": args.config, "k01_env": os.environ.get("CGGM_K01", "1")}
for name, streamed in (("not_stored", True), ("stored", False)):
    if not streamed:
        bufs["GradT"] = colmajor_empty(p, q)
    for _ in range(2):
        r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=streamed)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=streamed)
    e1.record()
    torch.cuda.synchronize()
    a = r["active"]
    out[name] = {"ms": round(e0.elapsed_time(e1) / args.reps, 3), "m_L": a["m_L"], "m_T": a["m_T"],
                 "ties_T": a["ties_T"], "subgrad_l1": a["subgrad_l1"], "f": r["objective"]["f"]}
print(json.dumps(out))
