"""ctypes binding of the plain-C oracle (oracle/c/cggm_oracle_c.c) -- TEST INFRASTRUCTURE ONLY.

The second, independent form of the oracle's definitions: C loop nests in fp64 without BLAS /
LAPACK, built by `build()` (gcc -O2 -fopenmp, no fast-math).  Used by
tests/test_oracle_c.py to pin the numpy oracle against an implementation that shares none of its
code or library routines, and to time the plain definition per phase on the host."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "cggm_oracle_c.c")
LIB = os.path.join(HERE, "c", "libcggm_oracle_c.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", LIB, SRC, "-lm"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
    return _lib


_d = ctypes.c_double
_i64 = ctypes.c_int64


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _csc(m):
    return (np.ascontiguousarray(m.colptr, dtype=np.int64), np.ascontiguousarray(m.rowidx, dtype=np.int32),
            np.ascontiguousarray(m.val, dtype=np.float64))


def covariances(X, Y):
    X, Y = _f(X), _f(Y)
    n, p = X.shape
    q = Y.shape[1]
    Syy, Sxy = np.zeros((q, q), order="F"), np.zeros((p, q), order="F")
    lib().cggm_oracle_c_covariances(_i64(n), _i64(p), _i64(q), _p(X), _p(Y), _p(Syy), _p(Sxy))
    return Syy, Sxy


def invert_logdet(Lam, want_sigma=True):
    A = _f(Lam)
    q = A.shape[0]
    S = np.zeros((q, q), order="F") if want_sigma else None
    ld, pd, fc = _d(), ctypes.c_int(), _i64()
    lib().cggm_oracle_c_invert_logdet(_i64(q), _p(A), _p(S), ctypes.byref(ld), ctypes.byref(pd), ctypes.byref(fc))
    return (S if pd.value else None), ld.value, bool(pd.value), int(fc.value)


def psi_grad(X, Y, theta, Sigma, Syy):
    X, Y, Sigma, Syy = _f(X), _f(Y), _f(Sigma), _f(Syy)
    n, p = X.shape
    q = Y.shape[1]
    cp, ri, v = _csc(theta)
    Psi, GL, GT = np.zeros((q, q), order="F"), np.zeros((q, q), order="F"), np.zeros((p, q), order="F")
    lib().cggm_oracle_c_psi_grad(_i64(n), _i64(p), _i64(q), _p(X), _p(Y), _p(cp), _p(ri), _p(v), _p(Sigma),
                                 _p(Syy), _p(Psi), _p(GL), _p(GT))
    return dict(Psi=Psi, GradL=GL, GradT=GT)


def active_set(GradL, GradT, lam_csc, theta_csc, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
    GL, GT = _f(GradL), _f(GradT)
    q, p = GL.shape[0], GT.shape[0]
    lc, lr, lv = _csc(lam_csc)
    tc, tr, tv = _csc(theta_csc)
    mL, mT, tL, tT, sub = _i64(), _i64(), _i64(), _i64(), _d()
    args = [_i64(p), _i64(q), _p(GL), _p(GT), _p(lc), _p(lr), _p(lv), _p(tc), _p(tr), _p(tv), _d(lam_L), _d(lam_T),
            ctypes.c_int(int(bool(penalize_diag))), _d(tie_eps), ctypes.byref(mL), ctypes.byref(mT), ctypes.byref(tL),
            ctypes.byref(tT), ctypes.byref(sub)]
    lib().cggm_oracle_c_active_set(*args, None, None, None, None)   # sizes first
    Lr, Lc = np.zeros(mL.value, np.int32), np.zeros(mL.value, np.int32)
    Tr, Tc = np.zeros(mT.value, np.int32), np.zeros(mT.value, np.int32)
    lib().cggm_oracle_c_active_set(*args, _p(Lr), _p(Lc), _p(Tr), _p(Tc))
    return dict(L_row=Lr, L_col=Lc, T_row=Tr, T_col=Tc, m_L=mL.value, m_T=mT.value, ties_L=tL.value,
                ties_T=tT.value, subgrad_l1=sub.value)


def objective(X, Y, lam_csc, theta_csc, lam_L, lam_T, penalize_diag=True):
    X, Y = _f(X), _f(Y)
    n, p = X.shape
    q = Y.shape[1]
    lc, lr, lv = _csc(lam_csc)
    tc, tr, tv = _csc(theta_csc)
    f, ld, pd = _d(), _d(), ctypes.c_int()
    lib().cggm_oracle_c_objective(_i64(n), _i64(p), _i64(q), _p(X), _p(Y), _p(lc), _p(lr), _p(lv), _p(tc), _p(tr),
                                  _p(tv), _d(lam_L), _d(lam_T), ctypes.c_int(int(bool(penalize_diag))),
                                  ctypes.byref(f), ctypes.byref(ld), ctypes.byref(pd))
    return dict(f=f.value, logdet=ld.value, is_pd=bool(pd.value))


def timed_evaluation(X, Y, lam_csc, theta_csc, lam_L, lam_T, penalize_diag=True):
    """One evaluation in the plain-loop form; per-phase host seconds."""
    X, Y = _f(X), _f(Y)
    n, p = X.shape
    q = Y.shape[1]
    lc, lr, lv = _csc(lam_csc)
    tc, tr, tv = _csc(theta_csc)
    f, ld, sub, mL, mT = _d(), _d(), _d(), _i64(), _i64()
    secs = np.zeros(5)
    lib().cggm_oracle_c_eval(_i64(n), _i64(p), _i64(q), _p(X), _p(Y), _p(lc), _p(lr), _p(lv), _p(tc), _p(tr), _p(tv),
                             _d(lam_L), _d(lam_T), ctypes.c_int(int(bool(penalize_diag))), ctypes.byref(f),
                             ctypes.byref(ld), ctypes.byref(mL), ctypes.byref(mT), ctypes.byref(sub), _p(secs))
    return dict(f=f.value, logdet=ld.value, m_L=mL.value, m_T=mT.value, subgrad_l1=sub.value,
                seconds=dict(zip(("invert_logdet", "psi_grad", "active_set", "objective", "covariances"),
                                 secs.tolist())))
