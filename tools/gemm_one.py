"""One FP64 GEMM through cggm_test_gemm (for ncu captures): tools/gemm_one.py tA tB M N K [tile] [reps] [flags]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context  # noqa
from paper_1509_04681_b200.api import colmajor_empty, ld_of  # noqa

tA, tB, M, N, K = (int(x) for x in sys.argv[1:6])
tile = int(sys.argv[6]) if len(sys.argv) > 6 else 0
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
flags = int(sys.argv[8]) if len(sys.argv) > 8 else 0
ctx = Context(0)
ctx._check(ctx.lib.cggm_test_set_tile(ctx.h, tile))
A = colmajor_empty(K, M) if tA else colmajor_empty(M, K)
B = colmajor_empty(N, K) if tB else colmajor_empty(K, N)
C = colmajor_empty(M, N)
for t in (A, B, C):
    t.normal_()
for _ in range(reps):
    ctx._check(ctx.lib.cggm_test_gemm(ctx.h, tA, tB, M, N, K, ctypes.c_void_p(A.data_ptr()), ld_of(A),
                                      ctypes.c_void_p(B.data_ptr()), ld_of(B), ctypes.c_void_p(C.data_ptr()),
                                      ld_of(C), 1.0, 0.0, flags))
torch.cuda.synchronize()
print("ok")
