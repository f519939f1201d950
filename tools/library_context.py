"""Context numbers ("cuBLAS DGEMM/DSYRK/DTRSM, cuSOLVER DPOTRF/DPOTRI and cuSPARSE
SpMM at the same shapes on the same box"), through torch's bindings of the vendor libraries, next to
libcggm's kernels.  Not the bar -- the bar is the measured FP64 tensor peak.  One JSON line."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04681_b200 import Context, DeviceCsc, colmajor_empty, ld_of  # noqa
from synth.cggm_inputs import make_problem  # noqa


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
ctx = Context(0)
f64 = torch.float64
# GEMMs at the hot path's shapes: cuBLAS DGEMM (torch.matmul) vs cggm_test_gemm
for name, (tA, M, N, K) in {"XtE": (True, 40000, 20000, 1000), "WSigma": (False, 1000, 20000, 20000),
                            "sq8192": (False, 8192, 8192, 8192)}.items():
    A = torch.randn((K, M) if tA else (M, K), dtype=f64, device="cuda")
    B = torch.randn((K, N), dtype=f64, device="cuda")
    ms = timed(lambda: (A.t() if tA else A) @ B)
    res[f"cublas_dgemm_{name}_tflops"] = round(2.0 * M * N * K / ms / 1e9, 2)
    Ac = colmajor_empty(*(A.shape))
    Ac.copy_(A)
    Bc = colmajor_empty(*(B.shape))
    Bc.copy_(B)
    C = colmajor_empty(M, N)
    ms2 = timed(lambda: ctx.lib.cggm_test_gemm(ctx.h, int(tA), 0, M, N, K, ctypes.c_void_p(Ac.data_ptr()), ld_of(Ac),
                                                ctypes.c_void_p(Bc.data_ptr()), ld_of(Bc), ctypes.c_void_p(C.data_ptr()),
                                                ld_of(C), 1.0, 0.0, 0))
    res[f"cggm_gemm_{name}_tflops"] = round(2.0 * M * N * K / ms2 / 1e9, 2)
    del A, B, Ac, Bc, C
    torch.cuda.empty_cache()
# Sigma = Lambda^{-1} at large: cuSOLVER DPOTRF + DPOTRI (torch.linalg.cholesky + cholesky_inverse)
P = make_problem("large")
lam = [pt for pt in P.points if pt[0] == "truth"][0][1]
q = P.q
L = DeviceCsc.from_host(lam)
D = ctx.cggm_densify(L)
Dt = D.contiguous()
ms_potrf = timed(lambda: torch.linalg.cholesky(Dt), reps=2)
Lf = torch.linalg.cholesky(Dt)
ms_potri = timed(lambda: torch.cholesky_inverse(Lf), reps=2)
res["cusolver_potrf_ms"] = round(ms_potrf, 1)
res["cusolver_potri_ms"] = round(ms_potri, 1)
res["cusolver_inverse_total_ms"] = round(ms_potrf + ms_potri, 1)
res["cusolver_inverse_tflops"] = round(q ** 3 / (ms_potrf + ms_potri) / 1e9, 2)
ms_cggm = timed(lambda: ctx.cggm_invert_logdet(L), reps=2)
res["cggm_invert_logdet_ms"] = round(ms_cggm, 1)
res["cggm_invert_tflops"] = round(q ** 3 / ms_cggm / 1e9, 2)
# SpMM W = X Theta: cuSPARSE (torch.sparse.mm with Theta as CSR^T) vs k_spmm_x_theta2 (inside psi_grad; timed alone)
th = [pt for pt in P.points if pt[0] == "truth"][0][2]
Xd = torch.from_numpy(P.X).to("cuda")
Ts = torch.sparse_csr_tensor(torch.from_numpy(th.colptr), torch.from_numpy(th.rowidx.astype("int64")),
                             torch.from_numpy(th.val), size=(q, P.p), device="cuda")   # Theta^T in CSR
ms_sp = timed(lambda: torch.sparse.mm(Ts, Xd.t()))                                     # (X Theta)^T
res["cusparse_spmm_ms"] = round(ms_sp, 3)
print(json.dumps(res))
