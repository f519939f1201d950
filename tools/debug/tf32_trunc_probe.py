"""How the tcgen05 kind::tf32 MMA reads the 13 low mantissa bits of a 32-bit operand (truncation or
rounding): with CGGM_TF32_DEBUG=2 the TS form passes every operand's raw fp32 bits as hi (lo = 0), so
C = A B with A(0, 0) = 1 + f ulp_tf32, B(0, 0) = 1 shows what the tensor core multiplied."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1509_04681_b200 import Context  # noqa
from paper_1509_04681_b200.api import colmajor_empty, ld_of  # noqa

assert os.environ.get("CGGM_TF32_DEBUG") == "2", "run with CGGM_TF32_DEBUG=2"
ctx = Context(0, dtype="f32")
ctx._check(ctx.lib.cggm_test_set_tile(ctx.h, 1))   # no small-shape routing: the tensor-core engine
M = N = 256
K = 256
ulp = 2.0 ** -10
for frac in (0.25, 0.49, 0.51, 0.75, -0.25, -0.75):
    A = np.zeros((M, K), np.float32)
    B = np.zeros((K, N), np.float32)
    a = np.float32(1.0 + frac * ulp) if frac > 0 else np.float32(2.0 - (1 + frac) * ulp)  # frac < 0: just below 2
    A[0, 0] = a
    B[0, 0] = 1.0
    dA = colmajor_empty(M, K, dtype=torch.float32)
    dB = colmajor_empty(K, N, dtype=torch.float32)
    dC = colmajor_empty(M, N, dtype=torch.float32)
    dA.copy_(torch.from_numpy(A))
    dB.copy_(torch.from_numpy(B))
    ctx._check(ctx.lib.cggm_test_gemm_f32(ctx.h, 0, 0, M, N, K, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                          ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(dC.data_ptr()),
                                          ld_of(dC), 1.0, 0.0, 0))
    torch.cuda.synchronize()
    c = float(dC[0, 0])
    base = 1.0 if frac > 0 else 2.0 - ulp
    print(f"a = {float(a):.10f} ({'1 +' if frac > 0 else '2 - ulp +'} {frac if frac > 0 else 1 + frac:.2f} ulp): "
          f"MMA saw {c:.10f} = base + {(c - base) / ulp:+.3f} ulp")
