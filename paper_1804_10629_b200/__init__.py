"""paper_1804_10629_b200 — thin Python binding of libeks.so (include/eks.h, include/eks_kernels.h).

Argument marshalling only: every step of the s-step enlarged CG hot path runs in
the sm_100a CUDA kernels of ``csrc/``.  There is no CPU fallback — if
``libeks.so`` is missing or no CUDA device is present, the calls raise.

Arrays: numpy arrays are passed as HOST pointers (``EKS_MEM_HOST``); objects with
``data_ptr()`` (torch CUDA tensors) as DEVICE pointers (``EKS_MEM_DEVICE``).
All arrays must be C-contiguous with the dtype stated in the header.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libeks.so")

EKS_SRE_CG, EKS_SRE_CG2, EKS_MSDO_CG = 0, 1, 2
METHODS = {"sre-cg": EKS_SRE_CG, "sre-cg2": EKS_SRE_CG2, "msdo-cg": EKS_MSDO_CG,
           "ca-sre-cg": 3, "ca-sre-cg2": 4, "ca-msdo-cg": 5}
EKS_MEM_HOST, EKS_MEM_DEVICE = 0, 1
STATUS = {0: "EKS_OK", 1: "EKS_ERR_INVALID_ARG", 2: "EKS_ERR_STATE", 3: "EKS_ERR_BAD_MATRIX", 4: "EKS_ERR_OOM",
          5: "EKS_ERR_CUDA", 6: "EKS_ERR_NCCL", 7: "EKS_ERR_BREAKDOWN", 8: "EKS_ERR_MAXITER",
          9: "EKS_ERR_NONFINITE"}
EKS_OK, EKS_ERR_BREAKDOWN, EKS_ERR_MAXITER, EKS_ERR_OOM = 0, 7, 8, 4
KCLASSES = ["split", "spmm", "coef", "update", "reduce", "chol", "apply", "comm", "other", "upcoef"]


class EksError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("device", C.c_int), ("nccl_id", C.c_ubyte * 128)]


class _Report(C.Structure):
    _fields_ = [("outer_iters", C.c_int), ("converged", C.c_int), ("breakdown_block", C.c_int),
                ("max_outer_fit", C.c_int), ("rho0", C.c_double), ("rho", C.c_double),
                ("true_relres", C.c_double), ("solve_seconds", C.c_double), ("model_bytes", C.c_double),
                ("model_flops", C.c_double), ("gpu_launches", C.c_int), ("rho_history", C.POINTER(C.c_double))]


class _Options(C.Structure):
    _fields_ = [("max_outer", C.c_int), ("use_graph", C.c_int), ("profile", C.c_int), ("arnoldi", C.c_int),
                ("ortho", C.c_int), ("restructured", C.c_int), ("precond", C.c_int), ("aq_cache", C.c_int),
                ("onesynch", C.c_int), ("reserved", C.c_int * 2)]


class _Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 10), ("launches", C.c_longlong * 10), ("bytes", C.c_double * 10),
                ("flops", C.c_double * 10)]


_lib = None


def lib():
    """Load libeks.so (fails loudly: the product has no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (nvcc sm_100a)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
        sigs = {
            "eks_get_unique_id": [vp],
            "eks_create": [C.POINTER(vp), C.POINTER(_Dist)],
            "eks_set_stream": [vp, vp],
            "eks_setup_csr": [vp, i64, i64, i64, vp, vp, vp, i32],
            "eks_setup_precond": [vp, i32, i32, vp, vp, vp, i32],
            "eks_solve": [vp, i32, i32, i32, d, vp, vp, i32, i32, C.POINTER(_Report)],
            "eks_solve_ex": [vp, i32, i32, i32, d, vp, vp, i32, C.POINTER(_Options), C.POINTER(_Report)],
            "eks_basis_sweep": [vp, i32, i32, vp, vp, i32, C.POINTER(_Options), C.POINTER(_Report)],
            "eks_get_profile": [vp, C.POINTER(_Profile)],
            "eks_destroy": [vp],
            "eks_k_split": [vp, i32, vp, vp],
            "eks_k_spmm": [vp, i32, vp, vp, vp, vp, vp],
            "eks_k_cgs2": [vp, i32, i32, vp, vp, vp, vp, vp],
            "eks_k_acholqr": [vp, i32, vp, vp, vp, vp, vp],
            "eks_k_chol": [vp, i32, vp, vp],
            "eks_k_time_spmm": [vp, i32, vp, vp, vp, i32, i32, C.POINTER(d)],
            "eks_plan_halo": [i32, i32, vp, vp, vp, vp, vp, vp],
            "eks_k_last_basis": [vp, i32, vp, vp],
            "eks_plan_grid": [i64, i64, vp, vp, vp, i64, i64, vp, vp],
            "eks_k_last_residual": [vp, vp],
            "eks_plan_mpk": [i32, i32, i32, i32, vp],
            "eks_k_matrix_powers": [vp, i32, i32, i32, i32, vp, vp],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.eks_error_string.argtypes = [vp]
        L.eks_error_string.restype = C.c_char_p
        _lib = L
    return _lib


EXPORTED = ["eks_get_unique_id", "eks_create", "eks_set_stream", "eks_setup_csr", "eks_setup_precond", "eks_solve", "eks_solve_ex",
            "eks_basis_sweep", "eks_get_profile", "eks_destroy", "eks_error_string", "eks_k_split", "eks_k_spmm",
            "eks_k_cgs2", "eks_k_acholqr", "eks_k_chol", "eks_k_time_spmm", "eks_plan_halo", "eks_k_last_basis",
            "eks_k_last_residual", "eks_plan_grid", "eks_plan_mpk", "eks_k_matrix_powers"]


def eks_plan_halo(rank: int, nranks: int, ranges, row_ptr, col):
    """Host-only halo plan (see include/eks.h).  Returns (ext_col, need[nranks,2], geom dict)."""
    ranges = np.ascontiguousarray(ranges, np.int64)
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(col, np.int32)
    ext = np.empty_like(cl)
    need = np.zeros(2 * nranks, np.int64)
    geom = np.zeros(4, np.int64)
    st = lib().eks_plan_halo(int(rank), int(nranks), _ptr(ranges, np.int64), _ptr(rp, np.int64), _ptr(cl, np.int32),
                             _ptr(ext, np.int32), _ptr(need, np.int64), _ptr(geom, np.int64))
    _check(None, st)
    return ext, need.reshape(nranks, 2), dict(halo_before=int(geom[0]), halo_after=int(geom[1]),
                                              interior_lo=int(geom[2]), interior_hi=int(geom[3]))


def eks_plan_grid(row_begin: int, row_end: int, row_ptr, col, val, halo_before: int, halo_after: int):
    """Host-only stencil plan of a slab (no device): (geom dict, sv (rows × VS) or None)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(col, np.int32)
    vl = np.ascontiguousarray(val, np.float64)
    geom = np.zeros(6, np.int64)
    _check(None, lib().eks_plan_grid(int(row_begin), int(row_end), rp.ctypes.data, cl.ctypes.data, vl.ctypes.data,
                                     int(halo_before), int(halo_after), geom.ctypes.data, None))
    g = dict(zip(["nx", "ny", "nz", "w", "gb", "ga"], [int(v) for v in geom]))
    if g["w"] == 0:
        return g, None
    sv = np.zeros((row_end - row_begin, (g["w"] + 1) & ~1))
    _check(None, lib().eks_plan_grid(int(row_begin), int(row_end), rp.ctypes.data, cl.ctypes.data, vl.ctypes.data,
                                     int(halo_before), int(halo_after), geom.ctypes.data, sv.ctypes.data))
    return g, sv


def _order_after_torch():
    """The library runs on its own (non-blocking) stream or the one set by eks_set_stream: before
    it reads torch tensors, the work torch queued on its current stream must be complete (the C
    ABI's contract: the producing stream is synchronized before the call)."""
    import torch
    torch.cuda.current_stream().synchronize()


def _where(*arrays):
    dev = [hasattr(a, "data_ptr") for a in arrays if a is not None]
    if dev and all(dev):
        return EKS_MEM_DEVICE
    if any(dev):
        raise TypeError("mix of host (numpy) and device (torch) arrays in one call")
    return EKS_MEM_HOST


def _ptr(a, dtype):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if a.is_cuda:
            _order_after_torch()
        if not a.is_contiguous():
            raise ValueError("device tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags["C_CONTIGUOUS"]):
        raise TypeError(f"expected a C-contiguous numpy {np.dtype(dtype)} array")
    return a.ctypes.data_as(C.c_void_p)


def _check(ctx, st):
    if st != EKS_OK:
        msg = lib().eks_error_string(ctx).decode() if ctx else ""
        raise EksError(st, msg)


# ------------------------------------------------------------------ C-ABI mirrors
def eks_get_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(None, lib().eks_get_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def eks_create(rank: int = 0, nranks: int = 1, device: int = 0, nccl_id: bytes | None = None):
    h = C.c_void_p()
    if nranks == 1 and nccl_id is None:
        _check(None, lib().eks_create(C.byref(h), None))
    else:
        d = _Dist(rank, nranks, device)
        C.memmove(d.nccl_id, nccl_id, 128)
        _check(None, lib().eks_create(C.byref(h), C.byref(d)))
    return h


def eks_set_stream(ctx, stream_handle: int | None):
    _check(ctx, lib().eks_set_stream(ctx, C.c_void_p(stream_handle or 0)))


def eks_setup_csr(ctx, n_global, row_begin, row_end, row_ptr, col, val):
    where = _where(row_ptr, col, val)
    _check(ctx, lib().eks_setup_csr(ctx, int(n_global), int(row_begin), int(row_end), _ptr(row_ptr, np.int64),
                                    _ptr(col, np.int32), _ptr(val, np.float64), where))


PRECOND = {"ic0": 0, "chol": 1}


def eks_setup_precond(ctx, ndomains, row_ptr, col, val, kind="ic0"):
    """Block-Jacobi preconditioner of ndomains contiguous domains (same slab as eks_setup_csr):
    kind "ic0" (Table 5) or "chol" (complete Cholesky per block, Table 6)."""
    where = _where(row_ptr, col, val)
    _check(ctx, lib().eks_setup_precond(ctx, PRECOND[kind], int(ndomains), _ptr(row_ptr, np.int64),
                                        _ptr(col, np.int32), _ptr(val, np.float64), where))


def _report(rep: _Report):
    k = rep.outer_iters
    hist = np.ctypeslib.as_array(rep.rho_history, shape=(k + 1,)).copy() if rep.rho_history else None
    return dict(outer_iters=k, converged=bool(rep.converged), breakdown_block=rep.breakdown_block,
                max_outer_fit=rep.max_outer_fit, rho0=rep.rho0, rho=rep.rho, true_relres=rep.true_relres,
                solve_seconds=rep.solve_seconds, model_bytes=rep.model_bytes, model_flops=rep.model_flops,
                gpu_launches=rep.gpu_launches, hist=hist)


ORTHO = {"acholqr": 0, "pre-cholqr": 1}


AQ_CACHE = {"auto": 0, "on": 1, "off": 2}


def eks_solve_ex(ctx, method, s, t, tol, b, x, max_outer=0, profile=False, raise_on=(5, 6, 1, 2, 3), arnoldi=0,
                 ortho="acholqr", restructured=False, precond=False, use_graph=False, aq_cache="auto",
                 onesynch=False):
    """Returns (status, report dict).  x holds x0 on entry and the solution on exit.
    arnoldi (CA methods only): 7 = modified CA-Arnoldi (default), 5 = CA-Arnoldi.
    ortho: "acholqr" (default) or "pre-cholqr"; restructured: Alg 2 / Alg 1 (SRE-CG / SRE-CG2).
    onesynch: one-synch CGS2 (2s+1 collectives per outer iteration, DESIGN reading R36)."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    where = _where(b, x)
    opt = _Options(int(max_outer), int(use_graph), int(bool(profile)), int(arnoldi), ORTHO[ortho],
                   int(bool(restructured)), int(bool(precond)), AQ_CACHE[aq_cache], int(bool(onesynch)))
    rep = _Report()
    st = lib().eks_solve_ex(ctx, m, int(s), int(t), float(tol), _ptr(b, np.float64), _ptr(x, np.float64), where,
                            C.byref(opt), C.byref(rep))
    if st in raise_on:
        _check(ctx, st)
    return st, _report(rep)


def eks_solve(ctx, method, s, t, tol, b, x, max_outer=0):
    return eks_solve_ex(ctx, method, s, t, tol, b, x, max_outer=max_outer)


def eks_basis_sweep(ctx, t, nblocks, X0, W_last, profile=False, onesynch=False):
    where = _where(X0, W_last)
    opt = _Options(0, 0, int(bool(profile)))
    opt.onesynch = int(bool(onesynch))
    rep = _Report()
    st = lib().eks_basis_sweep(ctx, int(t), int(nblocks), _ptr(X0, np.float64), _ptr(W_last, np.float64), where,
                               C.byref(opt), C.byref(rep))
    _check(ctx, st)
    return _report(rep)


def eks_get_profile(ctx):
    p = _Profile()
    _check(ctx, lib().eks_get_profile(ctx, C.byref(p)))
    return dict(ms={k: p.ms[i] for i, k in enumerate(KCLASSES)},
                launches={k: int(p.launches[i]) for i, k in enumerate(KCLASSES)},
                bytes={k: p.bytes[i] for i, k in enumerate(KCLASSES)},
                flops={k: p.flops[i] for i, k in enumerate(KCLASSES)})


def eks_destroy(ctx):
    if ctx:
        lib().eks_destroy(ctx)


def eks_error_string(ctx) -> str:
    return lib().eks_error_string(ctx).decode()


# ------------------------------------------------------------------ kernel-level (device pointers)
def eks_k_split(ctx, t, r, Z):
    _check(ctx, lib().eks_k_split(ctx, int(t), _ptr(r, None), _ptr(Z, None)))


def eks_k_spmm(ctx, t, X, Y, G=None, v=None, g=None):
    _check(ctx, lib().eks_k_spmm(ctx, int(t), _ptr(X, None), _ptr(Y, None), _ptr(G, None), _ptr(v, None),
                                 _ptr(g, None)))


def eks_plan_mpk(nz: int, d: int, db: int, da: int):
    """Host-only matrix-powers plan (include/eks.h): d rows of (zlo, zhi, gb, ga)."""
    steps = np.zeros(4 * d, np.int32)
    _check(None, lib().eks_plan_mpk(int(nz), int(d), int(db), int(da), _ptr(steps, np.int32)))
    return steps.reshape(d, 4)


def eks_k_matrix_powers(ctx, t, s, z0, z1, X, V):
    _check(ctx, lib().eks_k_matrix_powers(ctx, int(t), int(s), int(z0), int(z1), _ptr(X, None), _ptr(V, None)))


def eks_k_cgs2(ctx, t, Q, AQ, Z, C1=None, C2=None):
    nq = len(Q)
    qa = (C.c_void_p * nq)(*[q.data_ptr() for q in Q])
    aqa = (C.c_void_p * nq)(*[q.data_ptr() for q in AQ])
    _check(ctx, lib().eks_k_cgs2(ctx, int(t), nq, C.cast(qa, C.c_void_p), C.cast(aqa, C.c_void_p), _ptr(Z, None),
                                 _ptr(C1, None), _ptr(C2, None)))


def eks_k_acholqr(ctx, t, Z, W, AW, R=None, B=None):
    st = lib().eks_k_acholqr(ctx, int(t), _ptr(Z, None), _ptr(W, None), _ptr(AW, None), _ptr(R, None),
                             _ptr(B, None))
    if st not in (EKS_OK, EKS_ERR_BREAKDOWN):
        _check(ctx, st)
    return st


def eks_k_chol(ctx, t, B, R):
    st = lib().eks_k_chol(ctx, int(t), _ptr(B, None), _ptr(R, None))
    if st not in (EKS_OK, EKS_ERR_BREAKDOWN):
        _check(ctx, st)
    return st


def eks_k_time_spmm(ctx, t, X, Y, v=None, variant=0, reps=10) -> float:
    """Average device time (ms) of one SpMM-block launch (see include/eks_kernels.h)."""
    ms = C.c_double(0.0)
    _check(ctx, lib().eks_k_time_spmm(ctx, int(t), _ptr(X, None), _ptr(Y, None), _ptr(v, None), int(variant),
                                      int(reps), C.byref(ms)))
    return ms.value


def eks_k_last_basis(ctx, j, W, AW=None):
    """Block j of the last solve's basis (and A·W) into device tensors W, AW."""
    _check(ctx, lib().eks_k_last_basis(ctx, int(j), _ptr(W, None), _ptr(AW, None)))


def eks_k_last_residual(ctx, r):
    _check(ctx, lib().eks_k_last_residual(ctx, _ptr(r, None)))


# ------------------------------------------------------------------ convenience
class Solver:
    """One context + one matrix slab.  ``Solver(A)`` for a single GPU where ``A`` has
    ``n, row_ptr, col, val`` (numpy, global columns)."""

    def __init__(self, A=None, *, rank=0, nranks=1, device=0, nccl_id=None, row_begin=0, row_end=None,
                 n_global=None):
        self.ctx = eks_create(rank, nranks, device, nccl_id)
        if A is not None:
            n_global = A.n if n_global is None else n_global
            row_end = A.n if row_end is None else row_end
            self.setup(n_global, row_begin, row_end, A.row_ptr, A.col, A.val)

    def setup(self, n_global, row_begin, row_end, row_ptr, col, val):
        rp = np.ascontiguousarray(row_ptr, np.int64) if isinstance(row_ptr, np.ndarray) else row_ptr
        cl = np.ascontiguousarray(col, np.int32) if isinstance(col, np.ndarray) else col
        vl = np.ascontiguousarray(val, np.float64) if isinstance(val, np.ndarray) else val
        eks_setup_csr(self.ctx, n_global, row_begin, row_end, rp, cl, vl)
        self._csr = (rp, cl, vl)

    def setup_precond(self, ndomains=64, kind="ic0"):
        """Block-Jacobi preconditioner (reading R32) for solve(..., precond=True): "ic0" or "chol"."""
        eks_setup_precond(self.ctx, ndomains, *self._csr, kind=kind)

    def solve(self, b, method="sre-cg", s=1, t=1, tol=1e-8, x0=None, max_outer=0, profile=False, arnoldi=0,
              ortho="acholqr", restructured=False, precond=False, use_graph=False, aq_cache="auto",
              onesynch=False):
        if isinstance(b, np.ndarray):
            b = np.ascontiguousarray(b, np.float64)
            x = np.zeros_like(b) if x0 is None else np.ascontiguousarray(x0, np.float64).copy()
        else:
            x = b.new_zeros(b.shape) if x0 is None else x0.clone()
        st, rep = eks_solve_ex(self.ctx, method, s, t, tol, b, x, max_outer=max_outer, profile=profile,
                               arnoldi=arnoldi, ortho=ortho, restructured=restructured, precond=precond,
                               use_graph=use_graph, aq_cache=aq_cache, onesynch=onesynch)
        rep["status"] = st
        rep["x"] = x
        return rep

    def profile(self):
        return eks_get_profile(self.ctx)

    def close(self):
        if self.ctx:
            eks_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
