"""Hot-path GEMM shapes on the current engine configuration (env selects variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import bench, SYM_LOWER, SYM_MIRROR, B_KLE_N  # noqa

bench(True, False, 40000, 20000, 1000)                       # X^T E
bench(False, False, 1000, 20000, 20000)                      # W Sigma
bench(False, True, 11016, 2560, 2432, beta=1.0)              # objective panel update
bench(False, True, 11016, 2560, 2560, flags=B_KLE_N, alg=11016 * 2560.0 * 2560)   # block-inverse apply
for tA in (False, True):
    for tB in (False, True):
        bench(tA, tB, 8192, 8192, 8192)
