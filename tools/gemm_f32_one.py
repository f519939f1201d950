"""One FP32 GEMM through cggm_test_gemm_f32 on the ctx's engine (for ncu captures):
tools/gemm_f32_one.py tA tB M N K [engine (4 = 3xTF32 TS form)] [reps]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context  # noqa
from paper_1509_04681_b200.api import colmajor_empty, ld_of  # noqa

tA, tB, M, N, K = (int(x) for x in sys.argv[1:6])
eng = int(sys.argv[6]) if len(sys.argv) > 6 else 4
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
ctx = Context(0, dtype="f32")
ctx._check(ctx.lib.cggm_test_set_f32_engine(ctx.h, eng))
A = colmajor_empty(K, M, dtype=torch.float32) if tA else colmajor_empty(M, K, dtype=torch.float32)
B = colmajor_empty(N, K, dtype=torch.float32) if tB else colmajor_empty(K, N, dtype=torch.float32)
C = colmajor_empty(M, N, dtype=torch.float32)
for t in (A, B, C):
    t.normal_()
for _ in range(reps):
    ctx._check(ctx.lib.cggm_test_gemm_f32(ctx.h, tA, tB, M, N, K, ctypes.c_void_p(A.data_ptr()), ld_of(A),
                                          ctypes.c_void_p(B.data_ptr()), ld_of(B), ctypes.c_void_p(C.data_ptr()),
                                          ld_of(C), 1.0, 0.0, 0))
torch.cuda.synchronize()
print("ok")
