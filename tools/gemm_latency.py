"""Per-call latency of small FP64 GEMMs (cggm_test_gemm) issued back to back on one stream, the
shapes at the bottom of the Cholesky recursion.  One JSON line per shape."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, colmajor_empty, ld_of  # noqa

ctx = Context(0)
reps = 500
for (M, N, K, flags) in [(64, 64, 64, 0), (64, 64, 64, 4), (128, 128, 128, 0), (256, 256, 256, 0), (128, 64, 64, 0),
                         (512, 512, 512, 0), (1024, 1024, 1024, 0), (192, 128, 128, 0)]:
    A = colmajor_empty(M, K)
    A.copy_(torch.randn(M, K, dtype=torch.float64))
    B = colmajor_empty(N, K)
    B.copy_(torch.randn(N, K, dtype=torch.float64))
    C = colmajor_empty(M, N, zero=True)
    ctx._sync_stream()

    def run():
        st = ctx.lib.cggm_test_gemm(ctx.h, 0, 1, M, N, K, ctypes.c_void_p(A.data_ptr()), ld_of(A),
                                    ctypes.c_void_p(B.data_ptr()), ld_of(B), ctypes.c_void_p(C.data_ptr()), ld_of(C),
                                    1.0, 1.0, flags)
        assert st == 0

    for _ in range(10):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = 1000 * e0.elapsed_time(e1) / reps
    print(json.dumps({"M": M, "N": N, "K": K, "flags": flags, "us": round(us, 2),
                      "tflops": round(2 * M * N * K / us / 1e6, 3)}), flush=True)
