"""Probe the 3xTF32 engine on structured inputs (debugging aid): prints errors and value mappings."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1509_04681_b200 import Context
from paper_1509_04681_b200.api import colmajor_empty, ld_of

ctx = Context(0, dtype="f32")


def run(tA, tB, A, B, M, N, K, eng=int(os.environ.get('TF32_ENGINE', '0'))):
    ctx._check(ctx.lib.cggm_test_set_f32_engine(ctx.h, eng))
    ts = []
    for a in (A, B, np.zeros((M, N))):
        t = colmajor_empty(a.shape[0], a.shape[1], dtype=torch.float32)
        t.copy_(torch.from_numpy(np.asfortranarray(a)).float())
        ts.append(t)
    dA, dB, dC = ts
    ctx._check(ctx.lib.cggm_test_gemm_f32(ctx.h, int(tA), int(tB), M, N, K, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                          ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(dC.data_ptr()),
                                          ld_of(dC), 1.0, 0.0, 0))
    torch.cuda.synchronize()
    return dC.double().cpu().numpy()


rng = np.random.default_rng(0)
for tA in (0, 1):
    for tB in (0, 1):
        M = N = K = 128
        Ar = np.round(rng.standard_normal((M, K)) * 8) / 8   # exact in tf32
        I = np.eye(K)
        A = Ar.T if tA else Ar
        C = run(tA, tB, A, I, M, N, K)
        err = np.abs(C - Ar).max()
        print(f"tA={tA} tB={tB} A*I: max err {err:.3e}", flush=True)
        if err > 1e-6:
            # where did A[i,j] land?
            for (i, j) in [(0, 0), (0, 1), (1, 0), (5, 9), (37, 100)]:
                hits = np.argwhere(np.abs(C - Ar[i, j]) < 1e-9)
                print(f"   A[{i},{j}]={Ar[i,j]} found at {hits[:6].tolist()}")
            print("   C[0:4,0:4]=", C[:4, :4].round(3).tolist(), " A[0:4,0:4]=", Ar[:4, :4].tolist())
        Br = np.round(rng.standard_normal((K, N)) * 8) / 8
        B = Br.T if tB else Br
        C = run(tA, tB, (I.T if tA else I), B, M, N, K)
        err = np.abs(C - Br).max()
        print(f"tA={tA} tB={tB} I*B: max err {err:.3e}", flush=True)
        if err > 1e-6:
            for (i, j) in [(0, 0), (0, 1), (1, 0), (5, 9), (37, 100)]:
                hits = np.argwhere(np.abs(C - Br[i, j]) < 1e-9)
                print(f"   B[{i},{j}]={Br[i,j]} found at {hits[:6].tolist()}")
        # lo part: values with bits below tf32
        x = 1.0 + 2.0 ** -15
        C = run(0, 0, np.full((1, 1), x), np.full((1, 1), x), 1, 1, 1)
        print("   1x1 (1+2^-15)^2:", C[0, 0], "exact", x * x, "fp32", np.float32(x) * np.float32(x))
