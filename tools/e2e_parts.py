"""Decompose the end-to-end evaluation: device composite (graph / eager), the host-buffer entry point,
and the host entry point with S_yy excluded (computed on device inputs), ms per call."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import (Context, DeviceCsc, HostCsc, _abi, colmajor_empty, host_colmajor,  # noqa
                                   newton_evaluation, to_device_colmajor)
from synth.cggm_inputs import make_problem  # noqa

P = make_problem("large")
_, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
ctx = Context(0)
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
bufs = {k: torch.empty(110_000_000 if k[0] == "L" else 6_000_000, dtype=torch.int32, device="cuda")
        for k in ("L_row", "L_col", "T_row", "T_col")}
Xh, Yh = host_colmajor(P.X), host_colmajor(P.Y)
Lh, Th = HostCsc.from_host(lam), HostCsc.from_host(th)
Syy_e = colmajor_empty(P.q, P.q)


def timed(fn, reps=3):
    fn()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 2)


res = {}
res["device_graph"] = timed(lambda: newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs))
ctx.set_option(_abi.CGGM_OPT_GRAPHS, 0)
res["device_eager"] = timed(lambda: newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs))
ctx.set_option(_abi.CGGM_OPT_GRAPHS, 1)
res["host_api"] = timed(lambda: ctx.cggm_newton_eval_host(Xh, Yh, Lh, Th, P.lam_L, P.lam_T, True, bufs=bufs, Syy=Syy_e))
res["syy_alone"] = timed(lambda: ctx.cggm_covariances(X, Y, want_sxy=False, Syy=Syy_e))
res["h2d_xy_alone"] = timed(lambda: (X.copy_(Xh, non_blocking=True), Y.copy_(Yh, non_blocking=True)))
print(json.dumps(res))
