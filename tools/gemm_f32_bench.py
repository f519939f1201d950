"""FP32 GEMM engines (cggm_test_gemm_f32: 3xTF32 tcgen05 and SIMT FFMA) on hot-path shapes: TFLOP/s."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context  # noqa
from paper_1509_04681_b200.api import colmajor_empty, ld_of  # noqa

ctx = Context(0, dtype="f32")
for eng, (tA, tB, M, N, K) in [(e, s) for e in (2, 4, 1) for s in [
        (1, 0, 8192, 8192, 8192), (0, 1, 8192, 8192, 8192), (0, 0, 8192, 8192, 8192), (1, 1, 8192, 8192, 8192),
        (1, 0, 40000, 20000, 1000), (0, 0, 1000, 20000, 20000)]]:
    ctx._check(ctx.lib.cggm_test_set_f32_engine(ctx.h, eng))
    A = colmajor_empty(K, M, dtype=torch.float32) if tA else colmajor_empty(M, K, dtype=torch.float32)
    B = colmajor_empty(N, K, dtype=torch.float32) if tB else colmajor_empty(K, N, dtype=torch.float32)
    C = colmajor_empty(M, N, dtype=torch.float32)
    for t in (A, B, C):
        t.normal_()
    args = (ctx.h, tA, tB, M, N, K, ctypes.c_void_p(A.data_ptr()), ld_of(A), ctypes.c_void_p(B.data_ptr()), ld_of(B),
            ctypes.c_void_p(C.data_ptr()), ld_of(C), 1.0, 0.0, 0)
    ctx._check(ctx.lib.cggm_test_gemm_f32(*args))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.lib.cggm_test_gemm_f32(*args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{({1: 'ffma', 2: 'tf32x3', 3: 'tf32x3_ldg', 4: 'tf32x3_ts'})[eng]} tA={tA} tB={tB} {M}x{N}x{K}: {ms:.3f} ms {2.0 * M * N * K / ms / 1e9:.2f} TFLOP/s", flush=True)
