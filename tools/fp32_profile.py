"""Per-phase launch times of one FP32-variant evaluation (CGGM_F32 context; separate calls, lookahead
off, CUDA events around every library launch) at a config: where the FP32 step's time goes."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, _abi, to_device_colmajor  # noqa
from paper_1509_04681_b200.api import newton_evaluation  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
args = ap.parse_args()
P = make_problem(args.config)
_, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
ctx = Context(0, dtype="f32")
f32 = torch.float32
X, Y = to_device_colmajor(P.X, dtype=f32), to_device_colmajor(P.Y, dtype=f32)
L, T = DeviceCsc.from_host(lam, dtype=f32), DeviceCsc.from_host(th, dtype=f32)
Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
bufs = {k: torch.empty(0, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")}
try:
    newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
except Exception:
    pass
mL, mT = ctx.last_active_sizes
for k, c in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT)):
    bufs[k] = torch.empty(int(c * 1.1) + 1024, dtype=torch.int32, device="cuda")
newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, composite=False)
ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, 0)
newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, composite=False)
torch.cuda.synchronize()
ctx.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs, composite=False)
e1.record()
torch.cuda.synchronize()
prof = ctx.profile_read()
print(json.dumps({"config": args.config, "serial_ms": e0.elapsed_time(e1),
                  "phases": {k: {"ms": round(v[0], 3), "launches": v[1]} for k, v in prof.items() if v[1]}}))
