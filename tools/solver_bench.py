"""Time Algorithm 1 (paper_1509_04681_b200/solver.py) on a config: wall time per ABI call kind
(each call ends in a host read of its scalars, so wall time is its GPU time) over a few outer
iterations from (I, 0).  One JSON line."""
import argparse
import collections
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, to_device_colmajor  # noqa
from paper_1509_04681_b200.solver import ancd_fit  # noqa
from synth.cggm_inputs import make_problem  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="medium")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--tol", type=float, default=0.01)
args = ap.parse_args()
P = make_problem(args.config)
ctx = Context(0)
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
acc = collections.defaultdict(lambda: [0, 0.0])
for name in ("cggm_covariances", "cggm_gram", "cggm_invert_logdet", "cggm_psi_grad", "cggm_lambda_direction",
             "cggm_lambda_step", "cggm_objective", "cggm_theta_cd"):
    fn = getattr(ctx, name)

    def wrap(*a, _fn=fn, _n=name, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = _fn(*a, **k)
        torch.cuda.synchronize()
        acc[_n][0] += 1
        acc[_n][1] += time.perf_counter() - t0
        return r

    setattr(ctx, name, wrap)
t0 = time.perf_counter()
res = ancd_fit(ctx, X, Y, P.lam_L, P.lam_T, max_iter=args.iters, tol=args.tol)
wall = time.perf_counter() - t0
print(json.dumps({"config": args.config, "iters": res.iters, "converged": res.converged, "wall_s": round(wall, 3),
                  "f": res.f, "history": res.history,
                  "calls": {k: {"n": v[0], "s": round(v[1], 4)} for k, v in acc.items()}}))
