"""Time the NEXT-1 / NEXT-2 coordinate sweeps at a config (default `large`): the column walk
(CGGM_CD_BLOCK=0) against the entry-blocked sweep (csrc/cd.cu k_sweep_blk) on the entries of the
last `window` columns of the active lists (the column walk needs ~14 us per update at large), agreement of the two on that prefix,
and the blocked sweep over the whole lists.  Prints one JSON object."""
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


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "large"
    window = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    full = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
    P = make_problem(name)
    label, lam, th = P.points[0]
    cb = ctx_with({"CGGM_CD_BLOCK": "1"})
    cw = ctx_with({"CGGM_CD_BLOCK": "0"})
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, Sxy = cb.cggm_covariances(X, Y)
    Sigma, _, _, _ = cb.cggm_invert_logdet(Lg)
    cap_l, cap_t = P.q * (P.q + 1) // 2, 8_000_000
    spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=1,
                L_row=torch.empty(cap_l, dtype=torch.int32, device="cuda"),
                L_col=torch.empty(cap_l, dtype=torch.int32, device="cuda"),
                T_row=torch.empty(cap_t, dtype=torch.int32, device="cuda"),
                T_col=torch.empty(cap_t, dtype=torch.int32, device="cuda"))
    r = cb.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Sxy=Sxy, Lam=Lg, fused=spec)
    act = r["active"]
    del r["GradT"]
    Lr, Lc, Tr, Tc = act["L_row"], act["L_col"], act["T_row"], act["T_col"]
    out = {"config": name, "m_L": int(Lr.numel()), "m_T": int(Tr.numel())}
    lc = Lc.cpu().numpy()
    tc = Tc.cpu().numpy()
    aL = int(np.searchsorted(lc, P.q - window))
    aT = int(np.searchsorted(tc, P.q - 20 * window))
    mL, mT = Lr.numel() - aL, Tr.numel() - aT
    out["prefix"] = {"last_columns_lambda": window, "last_columns_theta": 20 * window, "m_L": mL, "m_T": mT}

    def lam_dir(c, m):
        a = Lr.numel() - m
        return c.cggm_lambda_direction(Sigma, r["Psi"], r["GradL"], Lg, Lr[a:], Lc[a:], P.lam_L, True, 1)

    for tag, c in (("walk", cw), ("blocked", cb)):
        lam_dir(c, min(mL, 1000))   # warm-up (workspaces, attributes)
        (D, delta, _), t = timed(lambda: lam_dir(c, mL))
        out["prefix"][f"lambda_{tag}_s"] = t
        out["prefix"][f"lambda_{tag}_us_per_update"] = 1e6 * t / max(mL, 1)
        out["prefix"][f"_D_{tag}"] = D.cpu().numpy()
    Dw, Db = out["prefix"].pop("_D_walk"), out["prefix"].pop("_D_blocked")
    out["prefix"]["lambda_rel_diff"] = float(np.linalg.norm(Dw - Db) / max(np.linalg.norm(Dw), 1e-300))
    cols, xmap = cb.cggm_gram_rows(X, Tr)

    def th_sweep(c, m):
        a = Tr.numel() - m
        return c.cggm_theta_cd_rows(Sigma, cols, xmap, Sxy, Tg, Tr[a:], Tc[a:], P.lam_T, 1)

    for tag, c in (("walk", cw), ("blocked", cb)):
        th_sweep(c, min(mT, 1000))
        (Tn, _), t = timed(lambda: th_sweep(c, mT))
        out["prefix"][f"theta_{tag}_s"] = t
        out["prefix"][f"theta_{tag}_us_per_update"] = 1e6 * t / max(mT, 1)
        out["prefix"][f"_T_{tag}"] = Tn.val.cpu().numpy()
    Tw, Tb = out["prefix"].pop("_T_walk"), out["prefix"].pop("_T_blocked")
    out["prefix"]["theta_rel_diff"] = float(np.linalg.norm(Tw - Tb) / max(np.linalg.norm(Tw), 1e-300))
    print(json.dumps(out), flush=True)
    if full:
        (_, _, _), t = timed(lambda: lam_dir(cb, Lr.numel()))
        out["full_lambda_blocked_s"] = t
        out["full_lambda_us_per_update"] = 1e6 * t / Lr.numel()
        print(json.dumps(out), flush=True)
        (_, _), t = timed(lambda: th_sweep(cb, Tr.numel()))
        out["full_theta_blocked_s"] = t
        out["full_theta_us_per_update"] = 1e6 * t / Tr.numel()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
