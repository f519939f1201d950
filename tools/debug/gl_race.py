"""Debug: composite vs separate GradT under CGGM_GL_OVERLAP (which differs, where, by how much)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor  # noqa
from paper_1509_04681_b200.api import newton_evaluation  # noqa
from synth.cggm_inputs import make_problem  # noqa

P = make_problem(sys.argv[1] if len(sys.argv) > 1 else "medium")
label, lam, th = P.points[0]
ctx = Context(0)
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
cap = 4_000_000
def bufs():
    return {k: torch.empty(cap, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")}
res = {}
for comp in (False, True, False, True):
    r = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), composite=comp)
    torch.cuda.synchronize()
    res.setdefault(comp, []).append(r["GradT"].clone())
ref = (2.0 / P.n) * (X.t() @ (Y + (X @ torch.from_numpy(th.to_dense()).cuda()) @ res[False][0].new_tensor(0) if False else Y))
for comp, lst in res.items():
    for i, g in enumerate(lst):
        d = (g - res[False][0]).abs()
        nz = torch.nonzero(d > 0)
        print(f"composite={comp} run {i}: max|diff| vs separate run 0 = {float(d.max()):.3e}, n_diff = {nz.shape[0]}")
        if nz.shape[0]:
            rows = torch.unique(nz[:, 0]).tolist()
            tiles = sorted({(int(r) // 128, int(c) // 64) for r, c in nz.tolist()})
            print("   rows:", rows[:40], "n_rows", len(rows), "tiles (128x64):", tiles[:20], "n_tiles", len(tiles))
            r0 = rows[0]
            cs = nz[nz[:, 0] == r0][:, 1].tolist()
            print("   row", r0, "cols", cs[:8], "...", cs[-4:], "n", len(cs))
            g0 = res[False][0]
            print("   sample good/bad", float(g0[r0, cs[0]]), float(g[r0, cs[0]]))
