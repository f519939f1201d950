"""Per-phase host timing of the plain-C oracle (oracle/c/cggm_oracle_c.c: loop nests, no BLAS) for one
evaluation of a config -- SURVEY.md §8(d)'s oracle timing, at OMP_NUM_THREADS threads (set it in the
environment).  Test/measurement infrastructure: prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import c_oracle as C  # noqa: E402
from synth.cggm_inputs import make_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="medium")
args = ap.parse_args()
t0 = time.time()
P = make_problem(args.config)
label, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
gen_s = time.time() - t0
r = C.timed_evaluation(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
cpu = ""
try:
    cpu = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
r.update(config=args.config, threads=os.environ.get("OMP_NUM_THREADS", str(os.cpu_count())), host_cores=os.cpu_count(),
         cpu_model=cpu, generator_s=round(gen_s, 2),
         evaluation_s=round(sum(v for k, v in r["seconds"].items() if k != "covariances"), 3))
print(json.dumps(r))
