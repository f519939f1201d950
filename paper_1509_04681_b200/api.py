"""Thin Python binding of libcggm with the ABI's names (argument marshalling only).

Matrices are torch CUDA tensors in COLUMN-MAJOR layout: shape (rows, cols) with stride
(1, ld).  `colmajor_empty` / `to_device_colmajor` create them.  Every step of the hot path
runs in libcggm's CUDA kernels; this module only passes pointers, sizes and the current stream.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math

import numpy as np
import torch

from . import _abi

__all__ = ["Context", "DeviceCsc", "HostCsc", "CggmError", "colmajor_empty", "to_device_colmajor", "ld_of",
           "host_colmajor"]


class CggmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_abi.STATUS.get(status, status)}: {msg}")
        self.status = status


def colmajor_empty(rows: int, cols: int, device="cuda", dtype=torch.float64, zero=False) -> torch.Tensor:
    """(rows, cols) column-major tensor with a leading dimension padded to 16 bytes (TMA-friendly)."""
    m = 16 // torch.empty(0, dtype=dtype).element_size()
    ld = max(m, (rows + m - 1) // m * m)
    f = torch.zeros if zero else torch.empty
    base = f((max(cols, 1), ld), device=device, dtype=dtype)
    return base.t()[:rows, :cols]


def to_device_colmajor(a: np.ndarray, device="cuda", dtype=torch.float64) -> torch.Tensor:
    a = np.asarray(a, dtype=np.float64)
    t = colmajor_empty(a.shape[0], a.shape[1], device=device, dtype=dtype)
    t.copy_(torch.from_numpy(np.asfortranarray(a)).to(dtype))
    return t


def ld_of(t: torch.Tensor) -> int:
    if t.dim() != 2:
        raise ValueError("expected a 2-D column-major tensor")
    rows, cols = t.shape
    if t.stride(0) != 1 and rows > 1:
        raise ValueError(f"tensor is not column-major (strides {t.stride()})")
    return max(int(t.stride(1)) if cols > 1 else rows, rows, 1)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


@dataclasses.dataclass
class DeviceCsc:
    nrows: int
    ncols: int
    colptr: torch.Tensor  # int64
    rowidx: torch.Tensor  # int32
    val: torch.Tensor     # float64

    @classmethod
    def from_host(cls, csc, device="cuda", dtype=torch.float64) -> "DeviceCsc":
        return cls(int(csc.nrows), int(csc.ncols),
                   torch.as_tensor(np.asarray(csc.colptr, dtype=np.int64), device=device),
                   torch.as_tensor(np.asarray(csc.rowidx, dtype=np.int32), device=device),
                   torch.as_tensor(np.asarray(csc.val, dtype=np.float64), device=device).to(dtype))

    @property
    def nnz(self) -> int:
        return int(self.rowidx.numel())

    def c_struct(self) -> _abi.cggm_csc:
        return _abi.cggm_csc(self.nrows, self.ncols, self.nnz, self.colptr.data_ptr(),
                             self.rowidx.data_ptr() if self.nnz else None,
                             self.val.data_ptr() if self.nnz else None)


@dataclasses.dataclass
class HostCsc:
    """A CSC in (page-locked) host memory, for cggm_newton_eval_host."""
    nrows: int
    ncols: int
    colptr: torch.Tensor  # int64, CPU
    rowidx: torch.Tensor  # int32, CPU
    val: torch.Tensor     # float64, CPU

    @classmethod
    def from_host(cls, csc, pin=True) -> "HostCsc":
        def t(a, dt):
            x = torch.as_tensor(np.ascontiguousarray(a, dtype=dt))
            return x.pin_memory() if pin else x
        return cls(int(csc.nrows), int(csc.ncols), t(csc.colptr, np.int64), t(csc.rowidx, np.int32),
                   t(csc.val, np.float64))

    @property
    def nnz(self) -> int:
        return int(self.rowidx.numel())

    def c_struct(self) -> _abi.cggm_csc:
        return _abi.cggm_csc(self.nrows, self.ncols, self.nnz, self.colptr.data_ptr(),
                             self.rowidx.data_ptr() if self.nnz else None, self.val.data_ptr() if self.nnz else None)


def host_colmajor(a: np.ndarray, pin=True) -> torch.Tensor:
    """(rows, cols) column-major fp64 host tensor (stride (1, rows)), page-locked by default."""
    a = np.asarray(a, dtype=np.float64)
    base = torch.empty((a.shape[1], a.shape[0]), dtype=torch.float64, pin_memory=pin)
    base.copy_(torch.from_numpy(np.ascontiguousarray(a.T)))
    return base.t()


class Context:
    """A libcggm context on one CUDA device, enqueuing on torch's current stream."""

    def __init__(self, device: int = 0, dtype: str = "f64", validate: int = 1):
        self.lib = _abi.load()
        self.device = device
        if dtype not in ("f64", "f32"):
            raise ValueError("dtype must be 'f64' or 'f32'")
        self.tdtype = torch.float64 if dtype == "f64" else torch.float32
        h = ctypes.c_void_p()
        stream = torch.cuda.current_stream(device).cuda_stream
        st = self.lib.cggm_ctx_create(ctypes.byref(h), device, _abi.CGGM_F64 if dtype == "f64" else _abi.CGGM_F32,
                                      ctypes.c_void_p(stream))
        if st != 0:
            raise CggmError(st, "cggm_ctx_create failed (is this an sm_100 GPU?)")
        self.h = h
        self.lib.cggm_ctx_set_validate(self.h, validate)

    def close(self):
        if getattr(self, "h", None):
            self.lib.cggm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise CggmError(st, self.lib.cggm_last_error(self.h).decode())

    def _sync_stream(self):
        self.lib.cggm_ctx_set_stream(self.h, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))

    def set_option(self, option: int, value: int):
        """Scheduling options (include/cggm.h cggm_ctx_set_option): _abi.CGGM_OPT_LOOKAHEAD_MIN,
        _abi.CGGM_OPT_GRAPHS."""
        self._check(self.lib.cggm_ctx_set_option(self.h, int(option), int(value)))

    def profile(self, enable: bool):
        self._check(self.lib.cggm_ctx_profile(self.h, int(bool(enable))))

    def profile_read(self) -> dict:
        n = _abi.PROF_NTAGS
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        self._check(self.lib.cggm_ctx_profile_read(self.h, ms, cnt, n))
        return {self.lib.cggm_profile_tag_name(i).decode(): (ms[i], int(cnt[i])) for i in range(n)}

    # ---------------------------------------------------------------- dense building blocks
    def cggm_gemm(self, C, A, B, transA=False, transB=False, alpha=1.0, beta=0.0, flags=0, M=None, N=None, K=None):
        """C = alpha op(A) op(B) + beta C on column-major views (include/cggm.h cggm_gemm)."""
        self._sync_stream()
        M = C.shape[0] if M is None else M
        N = C.shape[1] if N is None else N
        if K is None:
            K = A.shape[0] if transA else A.shape[1]
        self._check(self.lib.cggm_gemm(self.h, int(bool(transA)), int(bool(transB)), M, N, K, float(alpha), _ptr(A),
                                       ld_of(A), _ptr(B), ld_of(B), float(beta), _ptr(C), ld_of(C), int(flags)))
        return C

    def cggm_chol_inverse_dense(self, A, X=None):
        """X = L^{-1} of the dense SPD block A (A's storage is overwritten); returns X, logdet, is_pd,
        fail_col."""
        self._sync_stream()
        q = A.shape[0]
        if X is None:
            X = colmajor_empty(q, q, device=A.device, dtype=self.tdtype)
        ld, pd, fc = ctypes.c_double(), ctypes.c_int32(), ctypes.c_int64()
        self._check(self.lib.cggm_chol_inverse_dense(self.h, q, _ptr(A), ld_of(A), _ptr(X), ld_of(X), ctypes.byref(ld),
                                                     ctypes.byref(pd), ctypes.byref(fc)))
        return X, ld.value, bool(pd.value), int(fc.value)

    def cggm_symmetrize(self, S):
        self._sync_stream()
        self._check(self.lib.cggm_symmetrize(self.h, S.shape[0], _ptr(S), ld_of(S)))
        return S

    def cggm_densify(self, A: DeviceCsc, D=None):
        self._sync_stream()
        if D is None:
            D = colmajor_empty(A.nrows, A.ncols, device=A.colptr.device, dtype=self.tdtype)
        cs = A.c_struct()
        self._check(self.lib.cggm_densify(self.h, ctypes.byref(cs), _ptr(D), ld_of(D)))
        return D

    # ---------------------------------------------------------------- sample sharding
    def comm_init(self, group=None):
        """Attach an NCCL communicator inside the library (cggm_comm_init) spanning the ranks of the
        torch.distributed `group`; rank 0's unique id travels over that group.  Afterwards
        cggm_covariances / cggm_gram / cggm_invert_logdet / cggm_psi_grad / cggm_objective are
        collective (include/cggm.h, "sample sharding")."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (ctypes.c_char * 128)()
        if rank == 0:
            st = self.lib.cggm_comm_unique_id(buf)
            if st != 0:
                raise CggmError(st, "cggm_comm_unique_id failed (NCCL not loadable?)")
        dev = torch.device("cuda", self.device) if dist.get_backend(group) == "nccl" else torch.device("cpu")
        t = torch.frombuffer(bytearray(bytes(buf)), dtype=torch.uint8).to(dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        buf = (ctypes.c_char * 128).from_buffer_copy(bytes(t.cpu().tolist()))
        self._check(self.lib.cggm_comm_init(self.h, buf, rank, world))

    def comm_init_torch(self, group=None):
        """Attach the torch.distributed `group` itself as the library's collectives
        (cggm_comm_init_external): each all-reduce / broadcast the library issues runs as a
        torch.distributed call on a view of the library's device buffer (staged through host memory
        for gloo).  For transports NCCL cannot serve, e.g. several ranks sharing one GPU in tests."""
        import torch.distributed as dist
        host = dist.get_backend(group) == "gloo"
        device = torch.device("cuda", self.device)

        def view(ptr, count, dtype):
            class _Cai:
                __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8" if dtype == 0 else "<f4",
                                            "data": (int(ptr), False), "version": 3, "strides": None}
            return torch.as_tensor(_Cai(), device=device)

        def allreduce(_user, ptr, count, dtype):
            try:
                t = view(ptr, count, dtype)
                if host:
                    h = t.cpu()
                    dist.all_reduce(h, group=group)
                    t.copy_(h)
                else:
                    dist.all_reduce(t, group=group)
                torch.cuda.synchronize(device)
                return 0
            except Exception:   # noqa: BLE001 -- reported to the library as a collective failure
                return 1

        def broadcast(_user, ptr, count, dtype, root):
            try:
                t = view(ptr, count, dtype)
                src = dist.get_global_rank(group, root) if group is not None else root
                if host:
                    h = t.cpu()
                    dist.broadcast(h, src=src, group=group)
                    t.copy_(h)
                else:
                    dist.broadcast(t, src=src, group=group)
                torch.cuda.synchronize(device)
                return 0
            except Exception:   # noqa: BLE001
                return 1

        self._comm_cbs = (_abi.ALLREDUCE_FN(allreduce), _abi.BROADCAST_FN(broadcast))   # keep alive
        self._check(self.lib.cggm_comm_init_external(self.h, dist.get_rank(group), dist.get_world_size(group),
                                                     self._comm_cbs[0], self._comm_cbs[1], None))

    def comm_destroy(self):
        self._check(self.lib.cggm_comm_destroy(self.h))
        self._comm_cbs = None

    def comm_info(self) -> tuple[int, int]:
        r, w = ctypes.c_int32(), ctypes.c_int32()
        self._check(self.lib.cggm_comm_info(self.h, ctypes.byref(r), ctypes.byref(w)))
        return int(r.value), int(w.value)

    def launch_count(self) -> int:
        v = ctypes.c_int64()
        self._check(self.lib.cggm_ctx_launch_count(self.h, ctypes.byref(v)))
        return int(v.value)

    # ---------------------------------------------------------------- a1
    def cggm_covariances(self, X, Y, n_total=None, want_syy=True, want_sxy=True, Syy=None, Sxy=None):
        self._sync_stream()
        n, q = Y.shape
        p = X.shape[1] if X is not None else 0
        n_total = n if n_total is None else n_total
        if want_syy and Syy is None:
            Syy = colmajor_empty(q, q, device=Y.device, dtype=self.tdtype)
        if want_sxy and Sxy is None:
            Sxy = colmajor_empty(p, q, device=Y.device, dtype=self.tdtype)
        self._check(self.lib.cggm_covariances(
            self.h, n, n_total, p, q, _ptr(X), ld_of(X) if X is not None else 1, _ptr(Y), ld_of(Y),
            _ptr(Syy) if want_syy else None, ld_of(Syy) if want_syy else 1,
            _ptr(Sxy) if want_sxy else None, ld_of(Sxy) if want_sxy else 1))
        return (Syy if want_syy else None), (Sxy if want_sxy else None)

    # ---------------------------------------------------------------- a3
    def cggm_invert_logdet(self, Lam: DeviceCsc, want_sigma=True, Sigma=None):
        self._sync_stream()
        q = Lam.nrows
        if want_sigma and Sigma is None:
            Sigma = colmajor_empty(q, q, device=Lam.colptr.device, dtype=self.tdtype)
        ld, pd, fc = ctypes.c_double(), ctypes.c_int32(), ctypes.c_int64()
        cs = Lam.c_struct()
        self._check(self.lib.cggm_invert_logdet(self.h, ctypes.byref(cs), _ptr(Sigma) if want_sigma else None,
                                                ld_of(Sigma) if want_sigma else 1,
                                                ctypes.byref(ld), ctypes.byref(pd), ctypes.byref(fc)))
        return (Sigma if want_sigma else None), ld.value, bool(pd.value), int(fc.value)

    # ---------------------------------------------------------------- a2/a4/a5
    def cggm_psi_grad(self, X, Y, Theta: DeviceCsc, Sigma, Syy=None, Sxy=None, n_total=None,
                      want_gradL=True, want_gradT=True, Lam: DeviceCsc | None = None, fused: dict | None = None,
                      out=None):
        self._sync_stream()
        n, p = X.shape
        q = Y.shape[1]
        n_total = n if n_total is None else n_total
        out = dict(out or {})
        dev = X.device
        Psi = out.get("Psi")
        if Psi is None:
            Psi = colmajor_empty(q, q, device=dev, dtype=self.tdtype)
        GradL = out.get("GradL") if want_gradL else None
        if want_gradL and GradL is None:
            GradL = colmajor_empty(q, q, device=dev, dtype=self.tdtype)
        GradT = out.get("GradT") if want_gradT else None
        if want_gradT and GradT is None:
            GradT = colmajor_empty(p, q, device=dev, dtype=self.tdtype)
        ts = Theta.c_struct()
        ls = Lam.c_struct() if Lam is not None else None
        ao = None
        if fused is not None:
            ao = self._active_struct(fused)
        st = self.lib.cggm_psi_grad(
            self.h, n, n_total, p, q, _ptr(X), ld_of(X), _ptr(Y), ld_of(Y), ctypes.byref(ts),
            _ptr(Sigma), ld_of(Sigma), _ptr(Syy), ld_of(Syy) if Syy is not None else 1,
            _ptr(Sxy), ld_of(Sxy) if Sxy is not None else 1,
            _ptr(Psi), ld_of(Psi), _ptr(GradL), ld_of(GradL) if GradL is not None else 1,
            _ptr(GradT), ld_of(GradT) if GradT is not None else 1,
            ctypes.byref(ls) if ls is not None else None, ctypes.byref(ao) if ao is not None else None)
        if ao is not None:   # required list sizes, also under CGGM_ERR_CAPACITY (two-call pattern)
            self.last_active_sizes = (int(ao.m_L), int(ao.m_T))
        self._check(st)
        res = dict(Psi=Psi, GradL=GradL, GradT=GradT)
        if ao is not None:
            res["active"] = self._active_result(ao, fused)
        return res

    def cggm_grad_lambda(self, Syy, Sigma, Psi, GradL=None):
        self._sync_stream()
        q = Syy.shape[0]
        if GradL is None:
            GradL = colmajor_empty(q, q, device=Syy.device, dtype=self.tdtype)
        self._check(self.lib.cggm_grad_lambda(self.h, q, _ptr(Syy), ld_of(Syy), _ptr(Sigma), ld_of(Sigma),
                                              _ptr(Psi), ld_of(Psi), _ptr(GradL), ld_of(GradL)))
        return GradL

    def cggm_psi_residual(self, X, Y, Theta: DeviceCsc, Sigma, n_total=None, Psi=None, E=None):
        """Psi partial (all-reduced with a communicator) and the residual E = Y + X Theta Sigma
        (include/cggm.h, sample-sharded grad_Theta by column ranges)."""
        self._sync_stream()
        n, p = X.shape
        q = Y.shape[1]
        n_total = n if n_total is None else n_total
        if Psi is None:
            Psi = colmajor_empty(q, q, device=X.device, dtype=self.tdtype)
        if E is None:
            E = colmajor_empty(n, q, device=X.device, dtype=self.tdtype)
        ts = Theta.c_struct()
        self._check(self.lib.cggm_psi_residual(self.h, n, n_total, p, q, _ptr(X), ld_of(X), _ptr(Y), ld_of(Y),
                                               ctypes.byref(ts), _ptr(Sigma), ld_of(Sigma), _ptr(Psi), ld_of(Psi),
                                               _ptr(E), ld_of(E)))
        return Psi, E

    def cggm_active_theta_block(self, GradT_block, Theta: DeviceCsc, col0, lam_T, tie_eps, T_row, T_col):
        """S_Theta entries of the column block [col0, col0 + ncols) (global column indices) written
        into T_row / T_col from offset 0; returns (m, ties, subgrad_theta_part).  CGGM_ERR_CAPACITY
        carries the required size in the exception's `m`."""
        self._sync_stream()
        p, nc = GradT_block.shape
        ts = Theta.c_struct()
        m, ties, sub = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        st = self.lib.cggm_active_theta_block(self.h, p, int(col0), nc, _ptr(GradT_block), ld_of(GradT_block),
                                              ctypes.byref(ts), float(lam_T), float(tie_eps), _ptr(T_row), _ptr(T_col),
                                              int(T_row.numel()), ctypes.byref(m), ctypes.byref(ties),
                                              ctypes.byref(sub))
        if st == 6:
            err = CggmError(st, self.lib.cggm_last_error(self.h).decode())
            err.m = int(m.value)
            raise err
        self._check(st)
        return int(m.value), int(ties.value), float(sub.value)

    # ---------------------------------------------------------------- a6
    @staticmethod
    def _active_struct(spec: dict) -> _abi.cggm_active_out:
        ao = _abi.cggm_active_out()
        ao.lam_L = float(spec["lam_L"])
        ao.lam_T = float(spec["lam_T"])
        ao.penalize_diag = int(spec.get("penalize_diag", 1))
        ao.tie_eps = float(spec.get("tie_eps", 1e-9))
        for k in ("L_row", "L_col", "T_row", "T_col"):
            t = spec.get(k)
            setattr(ao, k, t.data_ptr() if t is not None and t.numel() > 0 else None)
        ao.cap_L = int(spec["L_row"].numel()) if spec.get("L_row") is not None else 0
        ao.cap_T = int(spec["T_row"].numel()) if spec.get("T_row") is not None else 0
        return ao

    @staticmethod
    def _active_result(ao, spec):
        m_L, m_T = int(ao.m_L), int(ao.m_T)
        r = dict(m_L=m_L, m_T=m_T, ties_L=int(ao.ties_L), ties_T=int(ao.ties_T), subgrad_l1=float(ao.subgrad_l1))
        if spec.get("L_row") is not None:
            r.update(L_row=spec["L_row"][:m_L], L_col=spec["L_col"][:m_L])
        if spec.get("T_row") is not None:
            r.update(T_row=spec["T_row"][:m_T], T_col=spec["T_col"][:m_T])
        return r

    def cggm_active_set(self, GradL, GradT, Lam: DeviceCsc, Theta: DeviceCsc, lam_L, lam_T, penalize_diag=True,
                        tie_eps=1e-9, cap_L=None, cap_T=None):
        """Two-call pattern: with cap None, first query the sizes, then allocate and fill."""
        self._sync_stream()
        q = GradL.shape[0]
        p = GradT.shape[0]
        dev = GradL.device
        spec = dict(lam_L=lam_L, lam_T=lam_T, penalize_diag=int(bool(penalize_diag)), tie_eps=tie_eps)
        if cap_L is None or cap_T is None:
            probe = self._active_struct(dict(spec))
            ls, ts = Lam.c_struct(), Theta.c_struct()
            st = self.lib.cggm_active_set(self.h, p, q, _ptr(GradL), ld_of(GradL), _ptr(GradT), ld_of(GradT),
                                          ctypes.byref(ls), ctypes.byref(ts), ctypes.byref(probe))
            if st not in (0, 6):
                self._check(st)
            cap_L, cap_T = int(probe.m_L), int(probe.m_T)
        spec.update(L_row=torch.empty(cap_L, dtype=torch.int32, device=dev),
                    L_col=torch.empty(cap_L, dtype=torch.int32, device=dev),
                    T_row=torch.empty(cap_T, dtype=torch.int32, device=dev),
                    T_col=torch.empty(cap_T, dtype=torch.int32, device=dev))
        ao = self._active_struct(spec)
        ls, ts = Lam.c_struct(), Theta.c_struct()
        self._check(self.lib.cggm_active_set(self.h, p, q, _ptr(GradL), ld_of(GradL), _ptr(GradT), ld_of(GradT),
                                             ctypes.byref(ls), ctypes.byref(ts), ctypes.byref(ao)))
        return self._active_result(ao, spec)

    # ---------------------------------------------------------------- a7
    def cggm_objective(self, X, Y, Lam: DeviceCsc, Theta: DeviceCsc, lam_L, lam_T, penalize_diag=True, W=None,
                       n_total=None):
        self._sync_stream()
        n, q = Y.shape
        p = Theta.nrows
        n_total = n if n_total is None else n_total
        o = _abi.cggm_objective_out()
        ls, ts = Lam.c_struct(), Theta.c_struct()
        self._check(self.lib.cggm_objective(
            self.h, n, n_total, p, q, _ptr(X), ld_of(X) if X is not None else 1, _ptr(Y), ld_of(Y),
            ctypes.byref(ls), ctypes.byref(ts), float(lam_L), float(lam_T), int(bool(penalize_diag)),
            _ptr(W), ld_of(W) if W is not None else 1, ctypes.byref(o)))
        return dict(f=o.f, g=o.g, logdet=o.logdet, tr_syy_lam=o.tr_syy_lam, tr_sxy_theta=o.tr_sxy_theta,
                    tr_sigma_m=o.tr_sigma_m, pen_L=o.pen_L, pen_T=o.pen_T, is_pd=bool(o.is_pd),
                    fail_col=int(o.fail_col))


    # ---------------------------------------------------------------- NEXT-1 / NEXT-2
    def cggm_objective_given_inverse(self, X, Y, Lam: DeviceCsc, Theta: DeviceCsc, lam_L, lam_T, Linv, logdet,
                                     penalize_diag=True, W=None, n_total=None):
        """The objective with the caller's L^{-1} and log-det (include/cggm.h)."""
        self._sync_stream()
        n, q = Y.shape
        p = Theta.nrows
        n_total = n if n_total is None else n_total
        o = _abi.cggm_objective_out()
        ls, ts = Lam.c_struct(), Theta.c_struct()
        self._check(self.lib.cggm_objective_given_inverse(
            self.h, n, n_total, p, q, _ptr(X), ld_of(X) if X is not None else 1, _ptr(Y), ld_of(Y), ctypes.byref(ls),
            ctypes.byref(ts), float(lam_L), float(lam_T), int(bool(penalize_diag)), _ptr(W),
            ld_of(W) if W is not None else 1, _ptr(Linv), ld_of(Linv), float(logdet), ctypes.byref(o)))
        return dict(f=o.f, g=o.g, logdet=o.logdet, tr_syy_lam=o.tr_syy_lam, tr_sxy_theta=o.tr_sxy_theta,
                    tr_sigma_m=o.tr_sigma_m, pen_L=o.pen_L, pen_T=o.pen_T, is_pd=bool(o.is_pd), fail_col=int(o.fail_col))

    def cggm_gram(self, X, n_total=None, Sxx=None):
        """S_xx = X^T X / n (p x p), for the Theta sweep."""
        self._sync_stream()
        n, p = X.shape
        n_total = n if n_total is None else n_total
        if Sxx is None:
            Sxx = colmajor_empty(p, p, device=X.device, dtype=self.tdtype)
        self._check(self.lib.cggm_gram(self.h, n, n_total, p, _ptr(X), ld_of(X), _ptr(Sxx), ld_of(Sxx)))
        return Sxx

    def cggm_lambda_direction(self, Sigma, Psi, GradL, Lam: DeviceCsc, L_row, L_col, lam_L, penalize_diag=True,
                              passes=1, D=None):
        """D_Lambda of Eq. (6) on the active list; returns (D, delta = tr(G^T D) + penalty change,
        ||Lambda||_1)."""
        self._sync_stream()
        q = Sigma.shape[0]
        m = int(L_row.numel())
        if D is None:
            D = torch.empty(max(m, 1), dtype=torch.float64, device=Sigma.device)
        dl = (ctypes.c_double * 2)()
        l1 = ctypes.c_double()
        cs = Lam.c_struct()
        self._check(self.lib.cggm_lambda_direction(
            self.h, q, _ptr(Sigma), ld_of(Sigma), _ptr(Psi), ld_of(Psi), _ptr(GradL), ld_of(GradL), ctypes.byref(cs),
            _ptr(L_row), _ptr(L_col), m, float(lam_L), int(bool(penalize_diag)), int(passes), _ptr(D), dl,
            ctypes.byref(l1)))
        return D[:m], dl[0] + dl[1], l1.value

    def cggm_lambda_step(self, Lam: DeviceCsc, L_row, L_col, D, alpha, out: DeviceCsc | None = None) -> DeviceCsc:
        """Lambda + alpha D as a symmetric CSC over the active list (and its mirror)."""
        self._sync_stream()
        q = Lam.nrows
        m = int(L_row.numel())
        dev = Lam.colptr.device
        if out is None or out.rowidx.numel() < 2 * m:
            out = DeviceCsc(q, q, torch.zeros(q + 1, dtype=torch.int64, device=dev),
                            torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev),
                            torch.empty(max(2 * m, 1), dtype=torch.float64, device=dev))
        oc = _abi.cggm_csc(q, q, int(out.rowidx.numel()), out.colptr.data_ptr(), out.rowidx.data_ptr(),
                           out.val.data_ptr())
        cs = Lam.c_struct()
        self._check(self.lib.cggm_lambda_step(self.h, q, ctypes.byref(cs), _ptr(L_row), _ptr(L_col), m, _ptr(D),
                                              float(alpha), ctypes.byref(oc)))
        return DeviceCsc(q, q, out.colptr, out.rowidx[:oc.nnz], out.val[:oc.nnz])

    def cggm_theta_cd(self, Sigma, Sxx, Sxy, Theta: DeviceCsc, T_row, T_col, lam_T, passes=1):
        """One (or `passes`) Theta sweeps of Eq. (7); returns (new Theta CSC, ||Theta||_1)."""
        self._sync_stream()
        p, q = Theta.nrows, Theta.ncols
        m = int(T_row.numel())
        dev = Sigma.device
        out = DeviceCsc(p, q, torch.zeros(q + 1, dtype=torch.int64, device=dev),
                        torch.empty(max(m, 1), dtype=torch.int32, device=dev),
                        torch.empty(max(m, 1), dtype=torch.float64, device=dev))
        oc = _abi.cggm_csc(p, q, m, out.colptr.data_ptr(), out.rowidx.data_ptr(), out.val.data_ptr())
        cs = Theta.c_struct()
        l1 = ctypes.c_double()
        self._check(self.lib.cggm_theta_cd(self.h, p, q, _ptr(Sigma), ld_of(Sigma), _ptr(Sxx), ld_of(Sxx), _ptr(Sxy),
                                           ld_of(Sxy), ctypes.byref(cs), _ptr(T_row), _ptr(T_col), m, float(lam_T),
                                           int(passes), ctypes.byref(oc), ctypes.byref(l1)))
        return DeviceCsc(p, q, out.colptr, out.rowidx[:m], out.val[:m]), l1.value

    def cggm_gram_rows(self, X, T_row, n_total=None, cache=None):
        """On-demand S_xx: the columns X^T X_i / n of the distinct rows i of the active list T_row
        (include/cggm.h).  Returns (Sxx_cols p x k, xmap int32 p); `cache` (a dict) keeps the buffers
        across calls (grown on CGGM_ERR_CAPACITY)."""
        self._sync_stream()
        n, p = X.shape
        n_total = n if n_total is None else n_total
        cache = {} if cache is None else cache
        if cache.get("xmap") is None or cache["xmap"].numel() != p:
            cache["xmap"] = torch.empty(p, dtype=torch.int32, device=X.device)
        while True:
            cols = cache.get("cols")
            cap = 0 if cols is None else cols.shape[1]
            k = ctypes.c_int64()
            st = self.lib.cggm_gram_rows(self.h, n, n_total, p, _ptr(X), ld_of(X), _ptr(T_row), int(T_row.numel()),
                                         _ptr(cols), ld_of(cols) if cols is not None else max(p, 1), cap,
                                         _ptr(cache["xmap"]), ctypes.byref(k))
            if st == 6:
                cache["cols"] = colmajor_empty(p, max(int(k.value), 1), device=X.device)
                continue
            self._check(st)
            return (cache["cols"][:, :int(k.value)] if cache.get("cols") is not None else None), cache["xmap"]

    def cggm_theta_cd_rows(self, Sigma, Sxx_cols, xmap, Sxy, Theta: DeviceCsc, T_row, T_col, lam_T, passes=1):
        """cggm_theta_cd on the on-demand S_xx columns of cggm_gram_rows."""
        self._sync_stream()
        p, q = Theta.nrows, Theta.ncols
        m = int(T_row.numel())
        dev = Sigma.device
        out = DeviceCsc(p, q, torch.zeros(q + 1, dtype=torch.int64, device=dev),
                        torch.empty(max(m, 1), dtype=torch.int32, device=dev),
                        torch.empty(max(m, 1), dtype=torch.float64, device=dev))
        oc = _abi.cggm_csc(p, q, m, out.colptr.data_ptr(), out.rowidx.data_ptr(), out.val.data_ptr())
        cs = Theta.c_struct()
        l1 = ctypes.c_double()
        k = 0 if Sxx_cols is None else int(Sxx_cols.shape[1])
        self._check(self.lib.cggm_theta_cd_rows(
            self.h, p, q, _ptr(Sigma), ld_of(Sigma), _ptr(Sxx_cols), ld_of(Sxx_cols) if k else 1, _ptr(xmap), k,
            _ptr(Sxy), ld_of(Sxy), ctypes.byref(cs), _ptr(T_row), _ptr(T_col), m, float(lam_T), int(passes),
            ctypes.byref(oc), ctypes.byref(l1)))
        return DeviceCsc(p, q, out.colptr, out.rowidx[:m], out.val[:m]), l1.value

    # ---------------------------------------------------------------- composite
    def cggm_newton_eval(self, X, Y, Syy, Lam: DeviceCsc, Theta: DeviceCsc, lam_L, lam_T, penalize_diag=True,
                         tie_eps=1e-9, bufs=None, stream_grad_theta=False):
        """One Newton-iteration evaluation in one call (objective overlapped on an internal stream).
        stream_grad_theta: do not store the p x q grad_Theta (it is compacted chunk by chunk)."""
        self._sync_stream()
        n, p = X.shape
        q = Y.shape[1]
        dev = X.device
        bufs = bufs if bufs is not None else {}
        shapes = [("Sigma", (q, q)), ("Psi", (q, q)), ("GradL", (q, q))]
        if not stream_grad_theta:
            shapes.append(("GradT", (p, q)))
        for k, shape in shapes:
            if bufs.get(k) is None:
                bufs[k] = colmajor_empty(*shape, device=dev, dtype=self.tdtype)
        if stream_grad_theta:
            bufs["GradT"] = None
        spec = dict(lam_L=lam_L, lam_T=lam_T, penalize_diag=int(bool(penalize_diag)), tie_eps=tie_eps,
                    L_row=bufs.get("L_row"), L_col=bufs.get("L_col"), T_row=bufs.get("T_row"), T_col=bufs.get("T_col"))
        ao = self._active_struct(spec)
        eo = _abi.cggm_eval_out()
        ls, ts = Lam.c_struct(), Theta.c_struct()
        self.last_active_sizes = None
        st = self.lib.cggm_newton_eval(
            self.h, n, p, q, _ptr(X), ld_of(X), _ptr(Y), ld_of(Y), _ptr(Syy), ld_of(Syy), ctypes.byref(ls),
            ctypes.byref(ts), _ptr(bufs["Sigma"]), ld_of(bufs["Sigma"]), _ptr(bufs["Psi"]), ld_of(bufs["Psi"]),
            _ptr(bufs["GradL"]), ld_of(bufs["GradL"]), _ptr(bufs["GradT"]),
            ld_of(bufs["GradT"]) if bufs["GradT"] is not None else 1, ctypes.byref(ao), ctypes.byref(eo))
        self.last_active_sizes = (int(ao.m_L), int(ao.m_T))
        self._check(st)
        o = eo.obj
        ob = dict(f=o.f, g=o.g, logdet=o.logdet, tr_syy_lam=o.tr_syy_lam, tr_sxy_theta=o.tr_sxy_theta,
                  tr_sigma_m=o.tr_sigma_m, pen_L=o.pen_L, pen_T=o.pen_T, is_pd=bool(o.is_pd), fail_col=int(o.fail_col))
        return dict(Sigma=bufs["Sigma"], logdet=eo.logdet, is_pd=bool(eo.is_pd), fail_col=int(eo.fail_col),
                    Psi=bufs["Psi"], GradL=bufs["GradL"], GradT=bufs["GradT"], active=self._active_result(ao, spec),
                    objective=ob)




    def cggm_newton_eval_blocked(self, X, Y, Lam: DeviceCsc, Theta: DeviceCsc, lam_L, lam_T, penalize_diag=True,
                                 tie_eps=1e-9, block=0, bufs=None):
        """NEXT-4: the evaluation without dense Sigma / Psi / gradients (include/cggm.h); bufs holds the
        active-list buffers (L_row, L_col, T_row, T_col; two-call pattern: last_active_sizes)."""
        self._sync_stream()
        n, p = X.shape
        q = Y.shape[1]
        bufs = bufs if bufs is not None else {}
        spec = dict(lam_L=lam_L, lam_T=lam_T, penalize_diag=int(bool(penalize_diag)), tie_eps=tie_eps,
                    L_row=bufs.get("L_row"), L_col=bufs.get("L_col"), T_row=bufs.get("T_row"), T_col=bufs.get("T_col"))
        ao = self._active_struct(spec)
        eo = _abi.cggm_eval_out()
        ls, ts = Lam.c_struct(), Theta.c_struct()
        self.last_active_sizes = None
        st = self.lib.cggm_newton_eval_blocked(self.h, n, p, q, _ptr(X), ld_of(X), _ptr(Y), ld_of(Y),
                                               ctypes.byref(ls), ctypes.byref(ts), int(block), ctypes.byref(ao),
                                               ctypes.byref(eo))
        self.last_active_sizes = (int(ao.m_L), int(ao.m_T))
        self._check(st)
        o = eo.obj
        ob = dict(f=o.f, g=o.g, logdet=o.logdet, tr_syy_lam=o.tr_syy_lam, tr_sxy_theta=o.tr_sxy_theta,
                  tr_sigma_m=o.tr_sigma_m, pen_L=o.pen_L, pen_T=o.pen_T, is_pd=bool(o.is_pd), fail_col=int(o.fail_col))
        return dict(logdet=eo.logdet, is_pd=bool(eo.is_pd), fail_col=int(eo.fail_col),
                    active=self._active_result(ao, spec), objective=ob)

    def cggm_newton_eval_host(self, Xh, Yh, Lam: HostCsc, Theta: HostCsc, lam_L, lam_T, penalize_diag=True,
                              tie_eps=1e-9, bufs=None, Syy=None, stream_grad_theta=False):
        """cggm_newton_eval from host buffers (column-major CPU tensors, HostCsc): uploads overlap the
        factorisation; S_yy is formed on the device into `Syy`.  Returns the cggm_newton_eval dict.
        stream_grad_theta: GradT = NULL, grad_Theta compacted chunk by chunk, never stored."""
        self._sync_stream()
        n, p = Xh.shape
        q = Yh.shape[1]
        bufs = dict(bufs) if bufs is not None else {}
        if stream_grad_theta:
            bufs["GradT"] = None
        for k, shape in (("Sigma", (q, q)), ("Psi", (q, q)), ("GradL", (q, q)), ("GradT", (p, q))):
            if k == "GradT" and stream_grad_theta:
                continue
            if bufs.get(k) is None:
                bufs[k] = colmajor_empty(*shape, device="cuda", dtype=self.tdtype)
        if Syy is None:
            Syy = colmajor_empty(q, q, device="cuda", dtype=self.tdtype)
        spec = dict(lam_L=lam_L, lam_T=lam_T, penalize_diag=int(bool(penalize_diag)), tie_eps=tie_eps,
                    L_row=bufs.get("L_row"), L_col=bufs.get("L_col"), T_row=bufs.get("T_row"), T_col=bufs.get("T_col"))
        ao = self._active_struct(spec)
        eo = _abi.cggm_eval_out()
        ls, ts = Lam.c_struct(), Theta.c_struct()
        st = self.lib.cggm_newton_eval_host(
            self.h, n, p, q, _ptr(Xh), ld_of(Xh), _ptr(Yh), ld_of(Yh), ctypes.byref(ls), ctypes.byref(ts),
            _ptr(Syy), ld_of(Syy), _ptr(bufs["Sigma"]), ld_of(bufs["Sigma"]), _ptr(bufs["Psi"]), ld_of(bufs["Psi"]),
            _ptr(bufs["GradL"]), ld_of(bufs["GradL"]), _ptr(bufs["GradT"]),
            ld_of(bufs["GradT"]) if bufs["GradT"] is not None else 1, ctypes.byref(ao), ctypes.byref(eo))
        self.last_active_sizes = (int(ao.m_L), int(ao.m_T))
        self._check(st)
        o = eo.obj
        ob = dict(f=o.f, g=o.g, logdet=o.logdet, tr_syy_lam=o.tr_syy_lam, tr_sxy_theta=o.tr_sxy_theta,
                  tr_sigma_m=o.tr_sigma_m, pen_L=o.pen_L, pen_T=o.pen_T, is_pd=bool(o.is_pd), fail_col=int(o.fail_col))
        return dict(Sigma=bufs["Sigma"], logdet=eo.logdet, is_pd=bool(eo.is_pd), fail_col=int(eo.fail_col),
                    Psi=bufs["Psi"], GradL=bufs["GradL"], GradT=bufs["GradT"], Syy=Syy,
                    active=self._active_result(ao, spec), objective=ob)


def newton_evaluation(ctx: Context, X, Y, Syy, Lam: DeviceCsc, Theta: DeviceCsc, lam_L, lam_T, penalize_diag=True,
                      bufs=None, tie_eps=1e-9, composite=True, stream_grad_theta=False):
    """One Newton-iteration evaluation (the metric's unit): invert_logdet(Lambda),
    psi_grad (+ fused active sets), objective at Lambda_trial = Lambda with its own Cholesky.
    composite=True uses the single overlapped call cggm_newton_eval; False issues the separate calls."""
    bufs = bufs if bufs is not None else {}
    if composite:
        return ctx.cggm_newton_eval(X, Y, Syy, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps, bufs,
                                    stream_grad_theta=stream_grad_theta)
    Sigma, logdet, pd, fc = ctx.cggm_invert_logdet(Lam, Sigma=bufs.get("Sigma"))
    spec = dict(lam_L=lam_L, lam_T=lam_T, penalize_diag=int(bool(penalize_diag)), tie_eps=tie_eps,
                L_row=bufs["L_row"], L_col=bufs["L_col"], T_row=bufs["T_row"], T_col=bufs["T_col"])
    r = ctx.cggm_psi_grad(X, Y, Theta, Sigma, Syy=Syy, Lam=Lam, fused=spec,
                          out=dict(Psi=bufs.get("Psi"), GradL=bufs.get("GradL"), GradT=bufs.get("GradT")))
    ob = ctx.cggm_objective(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag)
    return dict(Sigma=Sigma, logdet=logdet, is_pd=pd, fail_col=fc, **r, objective=ob)
