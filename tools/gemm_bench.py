"""Time the FP64 DMMA GEMM engine (cggm_test_gemm) per variant / shape / flags; prints TFLOP/s
against the algorithmic flops of each call."""
import ctypes
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context  # noqa
from paper_1509_04681_b200.api import colmajor_empty, ld_of  # noqa

ctx = Context(0)
A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N, SYM_LOWER, SYM_MIRROR = 1, 2, 4, 8, 16, 32


def bench(tA, tB, M, N, K, flags=0, alg=None, reps=3, beta=0.0, tile=0):
    ctx._check(ctx.lib.cggm_test_set_tile(ctx.h, tile))
    A = colmajor_empty(K, M) if tA else colmajor_empty(M, K)
    B = colmajor_empty(N, K) if tB else colmajor_empty(K, N)
    C = colmajor_empty(M, N)
    for t in (A, B, C):
        t.normal_()
    args = lambda: (ctx.h, int(tA), int(tB), M, N, K, ctypes.c_void_p(A.data_ptr()), ld_of(A),
                    ctypes.c_void_p(B.data_ptr()), ld_of(B), ctypes.c_void_p(C.data_ptr()), ld_of(C), 1.0, beta, flags)
    ctx._check(ctx.lib.cggm_test_gemm(*args()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.lib.cggm_test_gemm(*args())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = alg if alg is not None else 2.0 * M * N * K
    print(f"tA={int(tA)} tB={int(tB)} M={M:6d} N={N:6d} K={K:6d} flags={flags:3d} tile={tile} beta={beta}: "
          f"{ms:9.3f} ms  {fl / ms / 1e9:7.2f} TFLOP/s", flush=True)


if __name__ != "__main__":
    pass
elif len(sys.argv) > 1 and sys.argv[1] == "tiles":
    for s_ in (1536, 2048, 3072, 4096, 6144):
        for tile in (1, 2):
            bench(False, True, s_, s_, s_, tile=tile, reps=5)
            bench(True, False, s_, s_, s_, tile=tile, reps=5)
    for tile in (1, 2):
        bench(True, False, 4000, 4000, 500, flags=SYM_LOWER | SYM_MIRROR, alg=4000 * 4001 * 500.0, tile=tile)
        bench(True, False, 10000, 4000, 500, tile=tile)
        bench(False, False, 500, 4000, 4000, tile=tile)
    sys.exit(0)
if __name__ == "__main__":
    n = 8192
    for tA in (False, True):
        for tB in (False, True):
            bench(tA, tB, n, n, n)
    bench(False, True, n, n, n, beta=1.0)
    bench(False, True, 10016, 10016, 9984, flags=SYM_LOWER, alg=10016 * 10017 * 9984.0, beta=1.0)
    bench(True, False, 10016, 10016, 9984, flags=SYM_LOWER, alg=10016 * 10017 * 9984.0)
    bench(False, True, 10016, 9984, 9984, flags=B_KLE_N, alg=10016 * 9984.0 * 9984)
    bench(False, False, 10016, 9984, 9984, flags=B_KGE_N, alg=10016 * 9984.0 * 9984)
    bench(False, False, 10016, 9984, 10016, flags=A_KLE_M, alg=10016 * 10016.0 * 9984)
    bench(True, False, 20000, 20000, 20000, flags=A_KGE_M | B_KGE_N | SYM_LOWER | SYM_MIRROR, alg=20000 ** 3 / 3.0, reps=1)
    bench(False, False, 1000, 20000, 20000)
    bench(True, False, 20000, 20000, 1000, flags=SYM_LOWER | SYM_MIRROR, alg=20000 * 20001 * 1000.0)
    bench(True, False, 40000, 20000, 1000)
    for s in (256, 512, 1024, 2048):
        for tile in (1, 2):
            bench(False, True, s, s, s, tile=tile, reps=10)
    for tile in (1, 2):
        bench(False, True, 1064, 64, 64, tile=tile, reps=20)
        bench(False, True, 1064 + 500, 500, 512, flags=SYM_LOWER, tile=tile, reps=20, alg=(500 * 501 / 2 + 1064 * 500) * 512 * 2.0)
