"""Time Algorithm 1 (paper_1509_04681_b200/solver.py) on a config: wall time per ABI call kind
(each call ends in a host read of its scalars, so wall time is its GPU time) over a few outer
iterations from (I, 0), or warm-started at the generating point (--warm: Lambda*, Theta*).  One JSON
line (also written to --out)."""
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
ap.add_argument("--warm", action="store_true", help="start at (Lambda*, Theta*) instead of (I, 0)")
ap.add_argument("--sxx", default="rows", choices=["rows", "dense"])
ap.add_argument("--out", default=None)
args = ap.parse_args()
P = make_problem(args.config)
ctx = Context(0)
X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
acc = collections.defaultdict(lambda: [0, 0.0])
for name in ("cggm_covariances", "cggm_gram", "cggm_gram_rows", "cggm_invert_logdet", "cggm_psi_grad",
             "cggm_lambda_direction", "cggm_lambda_step", "cggm_objective", "cggm_objective_given_inverse",
             "cggm_theta_cd", "cggm_theta_cd_rows", "cggm_densify", "cggm_chol_inverse_dense", "cggm_gemm"):
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
kw = {}
if args.warm:
    from paper_1509_04681_b200 import DeviceCsc
    kw = dict(Lam0=DeviceCsc.from_host(P.lam_star), Theta0=DeviceCsc.from_host(P.theta_star))
t0 = time.perf_counter()
res = ancd_fit(ctx, X, Y, P.lam_L, P.lam_T, max_iter=args.iters, tol=args.tol, sxx=args.sxx, **kw)
wall = time.perf_counter() - t0
line = json.dumps({"config": args.config, "start": "generating point" if args.warm else "(I, 0)", "sxx": args.sxx,
                   "iters": res.iters, "converged": res.converged, "wall_s": round(wall, 3), "f": res.f,
                   "history": res.history, "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                   "calls": {k: {"n": v[0], "s": round(v[1], 4)} for k, v in acc.items()}})
print(line)
if args.out:
    with open(args.out, "w") as f:
        f.write(line + "\n")
