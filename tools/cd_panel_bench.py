"""Time the full blocked Lambda direction sweep at a config (default `large`) in the right-looking
form (CGGM_CD_PANEL=0: incremental U, Z row updates) and in the left-looking panel form at the given
panel widths, and report the agreement of the directions.  Prints one JSON object per variant.
usage: tools/cd_panel_bench.py [config] [widths, comma separated: 0,512,...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor  # noqa: E402
from synth.cggm_inputs import make_problem  # noqa: E402


def ctx_with(env):
    for k, v in env.items():
        os.environ[k] = v
    try:
        return Context(0)
    finally:
        for k in env:
            os.environ.pop(k, None)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "large"
    widths = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,512").split(",")]
    P = make_problem(name)
    label, lam, th = P.points[0]
    c0 = ctx_with({"CGGM_CD_BLOCK": "1", "CGGM_CD_PANEL": "0"})
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, Sxy = c0.cggm_covariances(X, Y)
    Sigma, _, _, _ = c0.cggm_invert_logdet(Lg)
    cap_l, cap_t = P.q * (P.q + 1) // 2, 8_000_000
    spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=1,
                L_row=torch.empty(cap_l, dtype=torch.int32, device="cuda"),
                L_col=torch.empty(cap_l, dtype=torch.int32, device="cuda"),
                T_row=torch.empty(cap_t, dtype=torch.int32, device="cuda"),
                T_col=torch.empty(cap_t, dtype=torch.int32, device="cuda"))
    r = c0.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Sxy=Sxy, Lam=Lg, fused=spec)
    act = r["active"]
    del r["GradT"]
    Lr, Lc = act["L_row"], act["L_col"]
    m = int(Lr.numel())
    base = None
    for w in widths:
        c = c0 if w == 0 else ctx_with({"CGGM_CD_BLOCK": "1", "CGGM_CD_PANEL": str(w)})
        c.cggm_lambda_direction(Sigma, r["Psi"], r["GradL"], Lg, Lr[:1000], Lc[:1000], P.lam_L, True, 1)  # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        D, delta, _ = c.cggm_lambda_direction(Sigma, r["Psi"], r["GradL"], Lg, Lr, Lc, P.lam_L, True, 1)
        torch.cuda.synchronize()
        t = time.perf_counter() - t
        Dh = D.cpu().numpy().copy()
        out = {"config": name, "m_L": m, "panel": w, "lambda_sweep_s": t, "us_per_update": 1e6 * t / max(m, 1),
               "delta": delta}
        if base is None:
            base = Dh
        else:
            out["rel_diff_vs_first"] = float(np.linalg.norm(Dh - base) / max(np.linalg.norm(base), 1e-300))
        print(json.dumps(out), flush=True)
        del c


if __name__ == "__main__":
    main()
