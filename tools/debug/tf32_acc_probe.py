"""Error of the 3xTF32 engine against an fp64 product as K grows, per accumulator mode (CGGM_TF32_ACC)
and the FFMA engine (CGGM_TF32_CHUNK: k-tiles per drained partial); mean signed relative error shows accumulation bias."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1509_04681_b200 import Context
from paper_1509_04681_b200.api import colmajor_empty, ld_of

rng = np.random.default_rng(1)
M = N = 256
for K in (32, 256, 1024, 4096, 16384):
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = np.abs(rng.standard_normal((K, N))).astype(np.float32)   # positive B: sums grow, bias visible
    ref = A.astype(np.float64) @ B.astype(np.float64)
    row = []
    for mode, eng in (("chunk0", 0), ("chunk4", 0), ("chunk8", 0), ("chunk16", 0), ("ffma", 1)):
        if mode.startswith("chunk"):
            os.environ["CGGM_TF32_CHUNK"] = mode[5:]
        ctx = Context(0, dtype="f32")
        ctx._check(ctx.lib.cggm_test_set_f32_engine(ctx.h, eng))
        dA = colmajor_empty(M, K, dtype=torch.float32); dA.copy_(torch.from_numpy(A))
        dB = colmajor_empty(K, N, dtype=torch.float32); dB.copy_(torch.from_numpy(B))
        dC = colmajor_empty(M, N, dtype=torch.float32)
        ctx._check(ctx.lib.cggm_test_gemm_f32(ctx.h, 0, 0, M, N, K, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                              ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(dC.data_ptr()),
                                              ld_of(dC), 1.0, 0.0, 0))
        torch.cuda.synchronize()
        C = dC.double().cpu().numpy()
        relf = np.linalg.norm(C - ref) / np.linalg.norm(ref)
        bias = float(np.mean((C - ref) * np.sign(ref)) / np.mean(np.abs(ref)))
        row.append(f"{mode}: relF {relf:.2e} bias {bias:+.2e}")
    print(f"K={K}: " + " | ".join(row), flush=True)
