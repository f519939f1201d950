"""Print FP32-variant errors against the fp64 oracle (for DESIGN.md)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cggm_oracle as O  # noqa
from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor  # noqa
from paper_1509_04681_b200.api import newton_evaluation  # noqa
from synth.cggm_inputs import make_problem  # noqa

ctx = Context(0, dtype="f32")
for name, k in (("tiny", 1), ("small", 1), ("medium", 0)):
    P = make_problem(name)
    _, lam, th = P.points[k]
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, ld, _, _ = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    f32 = torch.float32
    X, Y = to_device_colmajor(P.X, dtype=f32), to_device_colmajor(P.Y, dtype=f32)
    Lg, Tg = DeviceCsc.from_host(lam, dtype=f32), DeviceCsc.from_host(th, dtype=f32)
    S32, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    bufs = {key: torch.empty(4_000_000, dtype=torch.int32, device="cuda") for key in ("L_row", "L_col", "T_row", "T_col")}
    g = newton_evaluation(ctx, X, Y, S32, Lg, Tg, P.lam_L, P.lam_T, True, bufs)
    rel = lambda a, b: float(np.linalg.norm(a.double().cpu().numpy() - b) / np.linalg.norm(b))
    print(name, k, {"Sigma": rel(g["Sigma"], Sig), "Psi": rel(g["Psi"], r["Psi"]), "GradL": rel(g["GradL"], r["GradL"]),
                    "GradT": rel(g["GradT"], r["GradT"]), "f": abs(g["objective"]["f"] - ob["f"]) / abs(ob["f"]),
                    "logdet": abs(g["logdet"] - ld)})
