"""Symmetric (SYM_LOWER) hot-path products on the current engine configuration (env selects variants):
the Sigma product (lauum shape, triangular k-ranges, mirrored) and a plain mirrored syrk."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import bench, SYM_LOWER, SYM_MIRROR, A_KGE_M, B_KGE_N  # noqa

q = 20000
bench(True, False, q, q, q, flags=A_KGE_M | B_KGE_N | SYM_LOWER | SYM_MIRROR, alg=q ** 3 / 3.0)   # Sigma = L^-T L^-1
bench(False, True, 10000, 10000, 2500, flags=SYM_LOWER | SYM_MIRROR, alg=10000 * 10000 * 2500.0)  # trailing update
