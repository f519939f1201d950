"""One complete oracle evaluation at a config (default `large`) on the host cores, timed per phase,
beside the bench's flop-extrapolated estimate from sub-blocks of two sizes (validate the
cpu_baseline extrapolation).  Writes a JSON record (profiles/r02_oracle_full_<config>.json).

    python tools/oracle_full_eval.py [--config large] [--out profiles/r02_oracle_full_large.json]

The oracle is test infrastructure; this tool only measures it (like bench.py's cpu_baseline leg)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-full", action="store_true")
    args = ap.parse_args()
    from bench import alg_flops, blas_threads, oracle_eval_seconds, oracle_sample
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem

    P = make_problem(args.config)
    lam, th = P.lam_star, P.theta_star
    _, full = alg_flops(P.n, P.p, P.q, th.nnz)
    rec = {"config": args.config, "n": P.n, "p": P.p, "q": P.q, "cores": blas_threads(),
           "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}
    ext = []
    for qs, ps in ((3000, 6000), (5000, 10000)):
        X, Y, ls, ts = oracle_sample(P, qs, ps)
        secs, _ = oracle_eval_seconds(X, Y, ls, ts, P.lam_L, P.lam_T)
        _, samp = alg_flops(P.n, ps, qs, ts.nnz)
        ext.append({"qs": qs, "ps": ps, "sample_s": secs, "extrapolated_s": secs * full / samp,
                    "factor": full / samp})
        print(ext[-1], flush=True)
    rec["extrapolations"] = ext
    if not args.skip_full:
        ph = {}
        t = time.perf_counter
        t0 = t()
        Syy, _ = O.covariances(P.X, P.Y)
        ph["covariances_setup"] = t() - t0
        t0 = t()
        L, ok, fc = O.cholesky(lam.to_dense())
        ph["cholesky"] = t() - t0
        t0 = t()
        ld = O.logdet_from_cholesky(L)
        Sig = O.inverse_from_cholesky(L)
        ph["inverse"] = t() - t0
        del L
        t0 = t()
        r = O.psi_grad(P.X, P.Y, th, Sig, Syy, None)
        ph["psi_grad"] = t() - t0
        t0 = t()
        a = O.active_set(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T)
        sub = O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T)
        ph["active_set_subgrad"] = t() - t0
        del r, Sig
        t0 = t()
        ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, W=None)
        ph["objective"] = t() - t0
        total = sum(v for k, v in ph.items() if k != "covariances_setup")
        rec["full"] = {"phases_s": ph, "evaluation_s": total, "evals_per_s": 1.0 / total,
                       "f": ob["f"], "logdet": ld, "m_L": a["m_L"], "m_T": a["m_T"], "subgrad_l1": sub}
        rec["extrapolation_over_full"] = [e["extrapolated_s"] / total for e in ext]
        print(rec["full"], flush=True)
    out = args.out or os.path.join(ROOT, "profiles", f"r02_oracle_full_{args.config}.json")
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
