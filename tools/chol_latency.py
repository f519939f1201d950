"""Latency of the recursive Cholesky (+ triangular inverse) on dense SPD matrices of growing size
(cggm_test_chol_dense): per-size milliseconds, the achieved FP64 rate, and launches per call.
Locates the latency-bound recursion levels.  One JSON line per size."""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, colmajor_empty, ld_of  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="64,128,256,512,1024,2048,4096")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--potrf-only", action="store_true")
args = ap.parse_args()
ctx = Context(0)
for q in [int(v) for v in args.sizes.split(",")]:
    g = torch.Generator(device="cpu").manual_seed(q)
    M = torch.randn(q, q, generator=g, dtype=torch.float64) / q ** 0.5
    A0 = colmajor_empty(q, q)
    A0.copy_((M @ M.T + torch.eye(q, dtype=torch.float64)).cuda())
    A = colmajor_empty(q, q)
    X = colmajor_empty(q, q)
    full = 0 if args.potrf_only else 1

    def run():
        A.copy_(A0)
        st = ctx.lib.cggm_test_chol_dense(ctx.h, ctypes.c_void_p(A.data_ptr()), ld_of(A), q,
                                          ctypes.c_void_p(X.data_ptr()), ld_of(X), full, None, None)
        assert st == 0, ctx.lib.cggm_last_error(ctx.h)

    ctx._sync_stream()
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    c0.record()
    for _ in range(args.reps):
        A.copy_(A0)
    e0.record()
    for _ in range(args.reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(e0) / args.reps
    ms = e0.elapsed_time(e1) / args.reps - copy_ms
    flops = (2.0 / 3.0 if full else 1.0 / 3.0) * q ** 3
    print(json.dumps({"q": q, "mode": "full_inverse" if full else "potrf", "ms": round(ms, 4),
                      "tflops": round(flops / ms / 1e9, 3),
                      "launches": (ctx.launch_count() - l0) / args.reps}), flush=True)
