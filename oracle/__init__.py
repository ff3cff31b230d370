"""ctypes wrapper around the C oracle (oracle/eks_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs — never by the product
package ``paper_1804_10629_b200``.  Every function here is argument marshalling
around the plain C routines, which cite PAPER.md line by line.
"""
from __future__ import annotations

import ctypes as C
import types
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eks_oracle.c")
_HDR = os.path.join(_HERE, "eks_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

SRE_CG, SRE_CG2, MSDO_CG = 0, 1, 2
METHODS = {"sre-cg": SRE_CG, "sre-cg2": SRE_CG2, "msdo-cg": MSDO_CG}
OK, BADARG, BREAKDOWN, MAXITER = 0, 1, 7, 8
MODE_DEFINITION, MODE_MIRROR, MODE_ONESYNCH = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -ffp-contract=off, reading R20)."""
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        cmd = ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-Wall", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p)]


class _Report(C.Structure):
    _fields_ = [("outer_iters", C.c_int), ("converged", C.c_int), ("status", C.c_int),
                ("breakdown_block", C.c_int), ("rho0", C.c_double), ("rho", C.c_double),
                ("true_relres", C.c_double), ("rho_history", C.c_void_p)]


ITER_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double)

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32, vp = C.c_double, C.c_int64, C.c_int, C.c_void_p
        _lib.or_split.argtypes = [i64, i32, vp, vp]
        _lib.or_spmm.argtypes = [C.POINTER(_Csr), i32, vp, vp]
        _lib.or_xty.argtypes = [i64, i32, vp, i32, vp, vp]
        _lib.or_chol.argtypes = [i32, vp, vp]
        _lib.or_chol.restype = i32
        _lib.or_cgs2.argtypes = [C.POINTER(_Csr), i32, i32, vp, vp, vp, vp]
        _lib.or_acholqr.argtypes = [C.POINTER(_Csr), i32, vp, vp, vp, vp]
        _lib.or_acholqr.restype = i32
        _lib.or_solve.argtypes = [C.POINTER(_Csr), vp, vp, i32, i32, i32, d, i32, i32,
                                  C.POINTER(_Report), ITER_CB, vp]
        _lib.or_solve.restype = i32
        _lib.or_basis_sweep.argtypes = [C.POINTER(_Csr), i32, vp, i32, vp]
        _lib.or_basis_sweep.restype = i32
        _lib.or_solve_ca.argtypes = [C.POINTER(_Csr), vp, vp, i32, i32, i32, i32, d, i32,
                                     C.POINTER(_Report), ITER_CB, vp]
        _lib.or_solve_ca.restype = i32
        _lib.or_precholqr.argtypes = [C.POINTER(_Csr), i32, vp, vp, vp]
        _lib.or_precholqr.restype = i32
        _lib.or_solve_ex.argtypes = [C.POINTER(_Csr), vp, vp, i32, i32, i32, d, i32, i32, i32, i32,
                                     C.POINTER(_Report), ITER_CB, vp]
        _lib.or_solve_ex.restype = i32
        _lib.or_ic0_nnz.argtypes = [C.POINTER(_Csr), i32]
        _lib.or_ic0_nnz.restype = i64
        _lib.or_ic0.argtypes = [C.POINTER(_Csr), i32, vp, vp, vp]
        _lib.or_ic0.restype = i32
        _lib.or_lsolve.argtypes = [C.POINTER(_Csr), i32, vp, vp]
        _lib.or_ltsolve.argtypes = [C.POINTER(_Csr), i32, vp, vp]
        _lib.or_solve_pc.argtypes = [C.POINTER(_Csr), vp, vp, i32, i32, i32, d, i32, i32, i32, i32,
                                     C.POINTER(_Csr), C.POINTER(_Report), ITER_CB, vp]
        _lib.or_solve_pc.restype = i32
        _lib.or_solve_ca_pc.argtypes = [C.POINTER(_Csr), vp, vp, i32, i32, i32, i32, d, i32, C.POINTER(_Csr),
                                        C.POINTER(_Report), ITER_CB, vp]
        _lib.or_solve_ca_pc.restype = i32
        _lib.or_cholblk_nnz.argtypes = [C.POINTER(_Csr), i32]
        _lib.or_cholblk_nnz.restype = i64
        _lib.or_cholblk.argtypes = [C.POINTER(_Csr), i32, vp, vp, vp]
        _lib.or_cholblk.restype = i32
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class _CsrRef:
    """Keeps the numpy arrays alive while the C struct points at them."""

    def __init__(self, A):
        self.rp = np.ascontiguousarray(A.row_ptr, np.int64)
        self.col = np.ascontiguousarray(A.col, np.int32)
        self.val = np.ascontiguousarray(A.val, np.float64)
        self.s = _Csr(int(A.n), _p(self.rp), _p(self.col), _p(self.val))


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


def split(r: np.ndarray, t: int) -> np.ndarray:
    r = _f64(r)
    Z = np.empty((r.size, t))
    lib().or_split(r.size, t, _p(r), _p(Z))
    return Z


def spmm(A, X: np.ndarray) -> np.ndarray:
    X = _f64(X)
    t = 1 if X.ndim == 1 else X.shape[1]
    Y = np.empty_like(X)
    ref = _CsrRef(A)
    lib().or_spmm(C.byref(ref.s), t, _p(X), _p(Y))
    return Y


def xty(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    X, Y = _f64(X), _f64(Y)
    X2 = X.reshape(X.shape[0], -1)
    Y2 = Y.reshape(Y.shape[0], -1)
    Cm = np.empty((X2.shape[1], Y2.shape[1]))
    lib().or_xty(X2.shape[0], X2.shape[1], _p(X2), Y2.shape[1], _p(Y2), _p(Cm))
    return Cm


def chol(B: np.ndarray):
    B = _f64(B)
    t = B.shape[0]
    R = np.empty((t, t))
    st = lib().or_chol(t, _p(B), _p(R))
    return st, R


def cgs2(A, Z: np.ndarray, Qblocks):
    """Returns (Z2, C1, C2); Qblocks is a list of n×t arrays."""
    Z = _f64(Z).copy()
    t = Z.shape[1]
    qs = [_f64(q) for q in Qblocks]
    arr = (C.c_void_p * max(1, len(qs)))(*[q.ctypes.data for q in qs])
    C1 = np.empty((len(qs) * t, t))
    C2 = np.empty((len(qs) * t, t))
    ref = _CsrRef(A)
    lib().or_cgs2(C.byref(ref.s), t, len(qs), C.cast(arr, C.c_void_p), _p(Z), _p(C1), _p(C2))
    return Z, C1, C2


def acholqr(A, Z: np.ndarray):
    """Returns (status, W, R, B)."""
    Z = _f64(Z)
    t = Z.shape[1]
    W = np.empty_like(Z)
    R = np.empty((t, t))
    B = np.empty((t, t))
    ref = _CsrRef(A)
    st = lib().or_acholqr(C.byref(ref.s), t, _p(Z), _p(W), _p(R), _p(B))
    return st, W, R, B


def precholqr(A, Z: np.ndarray):
    """Pre-CholQR (reading R30).  Returns (status, W, R) with Z = W·R."""
    Z = _f64(Z)
    t = Z.shape[1]
    W = np.empty_like(Z)
    R = np.empty((t, t))
    ref = _CsrRef(A)
    st = lib().or_precholqr(C.byref(ref.s), t, _p(Z), _p(W), _p(R))
    return st, W, R


ORTHO = {"acholqr": 0, "pre-cholqr": 1}


def ic0(A, nd=64, kind="ic0"):
    """Block-Jacobi factor L (reading R32) of nd contiguous domains: IC(0) (Table 5) or the complete
    Cholesky of each diagonal block (kind="chol", Table 6); returns (status, L as Csr)."""
    ref = _CsrRef(A)
    nnzf, fac = (lib().or_ic0_nnz, lib().or_ic0) if kind == "ic0" else (lib().or_cholblk_nnz, lib().or_cholblk)
    nnz = int(nnzf(C.byref(ref.s), nd))
    rp = np.zeros(A.n + 1, np.int64)
    col = np.zeros(nnz, np.int32)
    val = np.zeros(nnz, np.float64)
    st = fac(C.byref(ref.s), nd, _p(rp), _p(col), _p(val))
    return st, types.SimpleNamespace(n=A.n, row_ptr=rp, col=col, val=val, nnz=nnz)


def lsolve(L, Z):
    """L⁻¹Z (n×t or n)."""
    Z = _f64(Z)
    Y = np.empty_like(Z)
    ref = _CsrRef(L)
    lib().or_lsolve(C.byref(ref.s), 1 if Z.ndim == 1 else Z.shape[1], _p(Z), _p(Y))
    return Y


def ltsolve(L, Z):
    """L⁻ᵗZ (n×t or n)."""
    Z = _f64(Z)
    Y = np.empty_like(Z)
    ref = _CsrRef(L)
    lib().or_ltsolve(C.byref(ref.s), 1 if Z.ndim == 1 else Z.shape[1], _p(Z), _p(Y))
    return Y


def solve(A, b, method="sre-cg", s=1, t=1, tol=1e-8, kmax=5000, x0=None, mode=MODE_DEFINITION,
          callback=None, ortho="acholqr", restructured=False, L=None):
    """Run or_solve_ex; returns dict(x, outer_iters, converged, status, rho0, rho, true_relres, hist).
    ortho: "acholqr" (default) or "pre-cholqr"; restructured: Alg 1/2 (SRE-CG2 / SRE-CG only)."""
    b = _f64(b)
    x = np.zeros(A.n) if x0 is None else _f64(x0).copy()
    hist = np.zeros(kmax + 1)
    rep = _Report(0, 0, 0, -1, 0.0, 0.0, 0.0, hist.ctypes.data)
    ref = _CsrRef(A)
    if callback is None:
        cb = ITER_CB()
    else:
        def _cb(user, k, n, st, V, alpha, xx, rr, rho):
            callback(k,
                     np.ctypeslib.as_array(V, shape=(n, st)).copy(),
                     np.ctypeslib.as_array(alpha, shape=(st,)).copy(),
                     np.ctypeslib.as_array(xx, shape=(n,)).copy(),
                     np.ctypeslib.as_array(rr, shape=(n,)).copy(), rho)
        cb = ITER_CB(_cb)
    m = METHODS[method] if isinstance(method, str) else int(method)
    Lref = _CsrRef(L) if L is not None else None
    st = lib().or_solve_pc(C.byref(ref.s), _p(b), _p(x), m, s, t, tol, kmax, mode, ORTHO[ortho],
                           int(bool(restructured)), C.byref(Lref.s) if Lref else None, C.byref(rep), cb, None)
    k = rep.outer_iters
    return dict(x=x, outer_iters=k, converged=bool(rep.converged), status=st, rho0=rep.rho0,
                rho=rep.rho, true_relres=rep.true_relres, hist=hist[: k + 1].copy(),
                breakdown_block=rep.breakdown_block)


def solve_ca(A, b, method="sre-cg", arnoldi=7, s=1, t=1, tol=1e-8, kmax=5000, x0=None, callback=None, L=None):
    """Run or_solve_ca_pc (CA SRE-CG / CA SRE-CG2 / CA MSDO-CG with Alg 5 or Alg 7, optionally split-
    preconditioned by M = L·Lᵗ); same dict as solve()."""
    b = _f64(b)
    x = np.zeros(A.n) if x0 is None else _f64(x0).copy()
    hist = np.zeros(kmax + 1)
    rep = _Report(0, 0, 0, -1, 0.0, 0.0, 0.0, hist.ctypes.data)
    ref = _CsrRef(A)
    if callback is None:
        cb = ITER_CB()
    else:
        def _cb(user, k, n, st, V, alpha, xx, rr, rho):
            callback(k,
                     np.ctypeslib.as_array(V, shape=(n, st)).copy(),
                     np.ctypeslib.as_array(alpha, shape=(st,)).copy(),
                     np.ctypeslib.as_array(xx, shape=(n,)).copy(),
                     np.ctypeslib.as_array(rr, shape=(n,)).copy(), rho)
        cb = ITER_CB(_cb)
    m = METHODS[method] if isinstance(method, str) else int(method)
    Lref = _CsrRef(L) if L is not None else None
    st = lib().or_solve_ca_pc(C.byref(ref.s), _p(b), _p(x), m, int(arnoldi), s, t, tol, kmax,
                              C.byref(Lref.s) if Lref else None, C.byref(rep), cb, None)
    k = rep.outer_iters
    return dict(x=x, outer_iters=k, converged=bool(rep.converged), status=st, rho0=rep.rho0,
                rho=rep.rho, true_relres=rep.true_relres, hist=hist[: k + 1].copy(),
                breakdown_block=rep.breakdown_block)


def basis_sweep(A, X0: np.ndarray, nblocks: int):
    X0 = _f64(X0)
    W = np.empty_like(X0)
    ref = _CsrRef(A)
    st = lib().or_basis_sweep(C.byref(ref.s), X0.shape[1], _p(X0), nblocks, _p(W))
    return st, W
