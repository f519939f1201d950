"""ctypes declarations of the libcggm C-ABI (include/cggm.h).  Marshalling only.

The shared library is built in-tree (paper_1509_04681_b200/lib/libcggm.so).  There is no CPU
fallback: if the library cannot be loaded, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CGGM_LIB: an alternative in-tree build of the same library (A/B kernel-variant measurements)
LIB_PATH = os.environ.get("CGGM_LIB") or os.path.join(_HERE, "lib", "libcggm.so")

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p
c_d = ctypes.c_double

STATUS = {
    0: "CGGM_OK", 1: "CGGM_ERR_INVALID_ARG", 2: "CGGM_ERR_SHAPE", 3: "CGGM_ERR_NOT_SYMMETRIC",
    4: "CGGM_ERR_BAD_SPARSE", 5: "CGGM_ERR_NONFINITE", 6: "CGGM_ERR_CAPACITY", 7: "CGGM_ERR_OOM",
    8: "CGGM_ERR_CUDA", 9: "CGGM_ERR_NCCL", 10: "CGGM_ERR_UNSUPPORTED",
}
CGGM_F64 = 0
CGGM_F32 = 1
CGGM_OPT_LOOKAHEAD_MIN = 0
CGGM_OPT_GRAPHS = 1
CGGM_OPT_FACTOR_REUSE = 2
CGGM_OPT_SIGMA_BLOCK = 3
# cggm_gemm structural flags
A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N, SYM_LOWER, SYM_MIRROR = 1, 2, 4, 8, 16, 32
PROF_NTAGS = 14


class cggm_csc(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i64), ("nnz", c_i64),
                ("colptr", c_vp), ("rowidx", c_vp), ("val", c_vp)]


class cggm_active_out(ctypes.Structure):
    _fields_ = [("lam_L", c_d), ("lam_T", c_d), ("penalize_diag", c_i32), ("tie_eps", c_d),
                ("cap_L", c_i64), ("cap_T", c_i64),
                ("L_row", c_vp), ("L_col", c_vp), ("T_row", c_vp), ("T_col", c_vp),
                ("m_L", c_i64), ("m_T", c_i64), ("ties_L", c_i64), ("ties_T", c_i64),
                ("subgrad_l1", c_d)]


class cggm_objective_out(ctypes.Structure):
    _fields_ = [("f", c_d), ("g", c_d), ("logdet", c_d), ("tr_syy_lam", c_d), ("tr_sxy_theta", c_d),
                ("tr_sigma_m", c_d), ("pen_L", c_d), ("pen_T", c_d), ("is_pd", c_i32), ("fail_col", c_i64)]


class cggm_eval_out(ctypes.Structure):
    _fields_ = [("logdet", c_d), ("is_pd", c_i32), ("fail_col", c_i64), ("obj", cggm_objective_out)]


# caller-provided collectives (cggm_comm_init_external)
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_vp, c_i64, c_i32)
BROADCAST_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_vp, c_i64, c_i32, c_i32)

# name -> (restype, argtypes); every symbol include/cggm.h declares
SIGNATURES = {
    "cggm_comm_unique_id": (c_i32, [c_vp]),
    "cggm_comm_init": (c_i32, [c_vp, c_vp, c_i32, c_i32]),
    "cggm_comm_init_external": (c_i32, [c_vp, c_i32, c_i32, ALLREDUCE_FN, BROADCAST_FN, c_vp]),
    "cggm_comm_destroy": (c_i32, [c_vp]),
    "cggm_device_alloc": (c_i32, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "cggm_device_free": (c_i32, [c_vp, c_vp]),
    "cggm_ipc_get_handle": (c_i32, [c_vp, c_vp, c_vp]),
    "cggm_ipc_open_handle": (c_i32, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "cggm_ipc_close_handle": (c_i32, [c_vp, c_vp]),
    "cggm_peer_allreduce": (c_i32, [c_vp, c_i32, c_i32, ctypes.POINTER(c_vp), c_i64]),
    "cggm_gemm": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i64, c_i64, c_d, c_vp, c_i64, c_vp, c_i64, c_d, c_vp, c_i64,
                          c_i32]),
    "cggm_chol_inverse_dense": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(c_d),
                                        ctypes.POINTER(c_i32), ctypes.POINTER(c_i64)]),
    "cggm_symmetrize": (c_i32, [c_vp, c_i64, c_vp, c_i64]),
    "cggm_objective_given_inverse": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                                             ctypes.POINTER(cggm_csc), ctypes.POINTER(cggm_csc), c_d, c_d, c_i32,
                                             c_vp, c_i64, c_vp, c_i64, c_d, ctypes.POINTER(cggm_objective_out)]),
    "cggm_densify": (c_i32, [c_vp, ctypes.POINTER(cggm_csc), c_vp, c_i64]),
    "cggm_psi_residual": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc),
                                  c_vp, c_i64, c_vp, c_i64, c_vp, c_i64]),
    "cggm_active_theta_block": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc), c_d, c_d,
                                        c_vp, c_vp, c_i64, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                        ctypes.POINTER(c_d)]),
    "cggm_comm_info": (c_i32, [c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "cggm_ctx_create": (c_i32, [ctypes.POINTER(c_vp), c_i32, c_i32, c_vp]),
    "cggm_ctx_destroy": (c_i32, [c_vp]),
    "cggm_ctx_set_stream": (c_i32, [c_vp, c_vp]),
    "cggm_ctx_set_validate": (c_i32, [c_vp, c_i32]),
    "cggm_ctx_set_option": (c_i32, [c_vp, c_i32, c_i64]),
    "cggm_ctx_launch_count": (c_i32, [c_vp, ctypes.POINTER(c_i64)]),
    "cggm_ctx_release_workspace": (c_i32, [c_vp]),
    "cggm_last_error": (ctypes.c_char_p, [c_vp]),
    "cggm_ctx_profile": (c_i32, [c_vp, c_i32]),
    "cggm_ctx_profile_read": (c_i32, [c_vp, ctypes.POINTER(c_d), ctypes.POINTER(c_i64), c_i32]),
    "cggm_profile_tag_name": (ctypes.c_char_p, [c_i32]),
    "cggm_version": (ctypes.c_char_p, []),
    "cggm_covariances": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                                 c_vp, c_i64, c_vp, c_i64]),
    "cggm_invert_logdet": (c_i32, [c_vp, ctypes.POINTER(cggm_csc), c_vp, c_i64, ctypes.POINTER(c_d),
                                   ctypes.POINTER(c_i32), ctypes.POINTER(c_i64)]),
    "cggm_psi_grad": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                              ctypes.POINTER(cggm_csc), c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                              c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                              ctypes.POINTER(cggm_csc), ctypes.POINTER(cggm_active_out)]),
    "cggm_grad_lambda": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64]),
    "cggm_active_set": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc),
                                ctypes.POINTER(cggm_csc), ctypes.POINTER(cggm_active_out)]),
    "cggm_newton_eval": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                 ctypes.POINTER(cggm_csc), ctypes.POINTER(cggm_csc), c_vp, c_i64, c_vp, c_i64,
                                 c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_active_out),
                                 ctypes.POINTER(cggm_eval_out)]),
    "cggm_newton_eval_blocked": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc),
                                         ctypes.POINTER(cggm_csc), c_i64, ctypes.POINTER(cggm_active_out),
                                         ctypes.POINTER(cggm_eval_out)]),
    "cggm_newton_eval_host": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc),
                                      ctypes.POINTER(cggm_csc), c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                      c_vp, c_i64, ctypes.POINTER(cggm_active_out), ctypes.POINTER(cggm_eval_out)]),
    "cggm_test_gemm": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                               c_d, c_d, c_i32]),
    "cggm_test_gemm_mir": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                   c_vp, c_d, c_i32]),
    "cggm_test_gemm_f32": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                   c_d, c_d, c_i32]),
    "cggm_test_set_tile": (c_i32, [c_vp, c_i32]),
    "cggm_test_set_f32_engine": (c_i32, [c_vp, c_i32]),
    "cggm_test_fp64_peak": (c_i32, [c_vp, c_d, ctypes.POINTER(c_d), ctypes.POINTER(c_d)]),
    "cggm_test_l2_peak": (c_i32, [c_vp, c_d, ctypes.POINTER(c_d), ctypes.POINTER(c_d)]),
    "cggm_test_profile_dump": (c_i32, [c_vp, ctypes.c_char_p]),
    "cggm_test_chol_dense": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_i32, ctypes.POINTER(c_d),
                                     ctypes.POINTER(c_i64)]),
    "cggm_gram": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64]),
    "cggm_lambda_direction": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc),
                                      c_vp, c_vp, c_i64, c_d, c_i32, c_i32, c_vp, ctypes.POINTER(c_d),
                                      ctypes.POINTER(c_d)]),
    "cggm_lambda_step": (c_i32, [c_vp, c_i64, ctypes.POINTER(cggm_csc), c_vp, c_vp, c_i64, c_vp, c_d,
                                 ctypes.POINTER(cggm_csc)]),
    "cggm_theta_cd": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.POINTER(cggm_csc),
                              c_vp, c_vp, c_i64, c_d, c_i32, ctypes.POINTER(cggm_csc), ctypes.POINTER(c_d)]),
    "cggm_gram_rows": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp,
                               ctypes.POINTER(c_i64)]),
    "cggm_theta_cd_rows": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                   ctypes.POINTER(cggm_csc), c_vp, c_vp, c_i64, c_d, c_i32, ctypes.POINTER(cggm_csc),
                                   ctypes.POINTER(c_d)]),
    "cggm_objective": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                               ctypes.POINTER(cggm_csc), ctypes.POINTER(cggm_csc), c_d, c_d, c_i32,
                               c_vp, c_i64, ctypes.POINTER(cggm_objective_out)]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libcggm.so and declare every exported symbol.  Raises OSError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"libcggm not built: {path} missing (run __graft_entry__.build()); "
                      "there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
