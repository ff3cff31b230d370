"""Pins for the oracle's block-Jacobi IC(0) preconditioner and the split-preconditioned s-step
methods (Alg 8 / 9 / 10) against what the paper and
the mathematics fix:

* IC(0) on matrices whose Cholesky factor has no fill (tridiagonal blocks) IS the Cholesky factor
  of each diagonal block (numpy);
* the defining IC(0) identity (L·Lᵗ)_ij = A_ij on the pattern of the block-diagonal lower triangle;
* the triangular solves against numpy's dense solves;
* the seed identity L⁻ᵗ[T(L⁻¹r)] = M⁻¹[T(r)] for t | nd — bitwise;
* t = s = 1 is preconditioned CG (Alg 11), written here independently in numpy;
* M = A (block-diagonal tridiagonal A, IC(0) exact) converges in one outer iteration;
* per-outer-iteration invariants (A-orthonormal V, Galerkin, φ decrease) and mirror = definition.
"""
import math

import numpy as np
import pytest

import eks_inputs as ei


def domain_of(n, nd, i):
    """D_d = [floor(d n/nd), floor((d+1) n/nd)) (reading R1/R32)."""
    return next(d for d in range(nd) if d * n // nd <= i < (d + 1) * n // nd)


def csr_of(L):
    return ei.Csr(L.n, L.row_ptr, L.col, L.val)


def tridiag_blocks(n, nd, seed=1):
    """Block-diagonal SPD matrix of nd tridiagonal blocks aligned with the nd contiguous domains."""
    rng = np.random.default_rng(seed)
    D = np.zeros((n, n))
    for d in range(nd):
        lo, hi = d * n // nd, (d + 1) * n // nd
        for i in range(lo, hi):
            D[i, i] = 4.0 + rng.random()
            if i + 1 < hi:
                D[i, i + 1] = D[i + 1, i] = -1.0 - rng.random()
    return D


def test_ic0_is_cholesky_without_fill(oracle_lib):
    n, nd = 96, 8
    D = tridiag_blocks(n, nd)
    A = ei.csr_from_dense(D)
    st, L = oracle_lib.ic0(A, nd)
    assert st == 0
    Ld = csr_of(L).to_dense()
    assert np.abs(Ld - np.linalg.cholesky(D)).max() <= 1e-14 * np.abs(Ld).max()


def test_ic0_identity_on_pattern(oracle_lib):
    A = ei.poisson2d(30)
    nd = 16
    st, L = oracle_lib.ic0(A, nd)
    assert st == 0
    D = A.to_dense()
    Ld = csr_of(L).to_dense()
    dom = np.array([domain_of(A.n, nd, i) for i in range(A.n)])
    same = dom[:, None] == dom[None, :]
    pat = (D != 0) & same
    assert np.all((Ld != 0) <= np.tril(pat))             # pattern ⊆ lower(block diag of A)
    M = Ld @ Ld.T
    assert np.abs((M - D)[np.tril(pat)]).max() <= 1e-13 * np.abs(D).max()
    assert np.abs(M[~same]).max() == 0.0                 # block diagonal: no coupling across domains
    assert np.all(np.diag(Ld) > 0)


def test_triangular_solves(oracle_lib):
    A = ei.poisson2d(20)
    st, L = oracle_lib.ic0(A, 8)
    Ld = csr_of(L).to_dense()
    Z = ei.uniform_pm1(3, A.n * 4).reshape(A.n, 4)
    assert np.abs(oracle_lib.lsolve(L, Z) - np.linalg.solve(Ld, Z)).max() <= 1e-12
    assert np.abs(oracle_lib.ltsolve(L, Z) - np.linalg.solve(Ld.T, Z)).max() <= 1e-12


@pytest.mark.parametrize("t", [2, 4, 8, 16])
def test_seed_identity_block_diagonal(oracle_lib, t):
    # with a block diagonal preconditioner aligned with the t domains,
    # [T(L⁻¹ r)] = L⁻¹[T(r)], hence L⁻ᵗ[T(L⁻¹ r)] = M⁻¹[T(r)]
    A = ei.poisson2d(24)
    st, L = oracle_lib.ic0(A, 16)
    r = ei.uniform_pm1(5, A.n)
    lhs = oracle_lib.ltsolve(L, oracle_lib.split(oracle_lib.lsolve(L, r), t))
    rhs = oracle_lib.ltsolve(L, oracle_lib.lsolve(L, oracle_lib.split(r, t)))
    assert np.array_equal(lhs, rhs)


def textbook_pcg(D, Ld, b, tol, kmax=10000, record=False):
    """Alg 11 with M = Ld Ldᵗ, numpy dense, independent of the oracle's solves."""
    minv = lambda v: np.linalg.solve(Ld.T, np.linalg.solve(Ld, v))
    x = np.zeros_like(b)
    r = b.copy()
    rho0 = r @ r
    rh = minv(r)
    rhor = r @ rh
    p = rh.copy()
    k = 0
    xs = [x.copy()]
    while math.sqrt(r @ r) > tol * math.sqrt(rho0) and k < kmax:
        w = D @ p
        alpha = rhor / (p @ w)
        x = x + alpha * p
        r = r - alpha * w
        rh = minv(r)
        rhor_new = r @ rh
        p = rh + (rhor_new / rhor) * p
        rhor = rhor_new
        k += 1
        xs.append(x.copy())
    return (k, x, xs) if record else (k, x)


def test_t1_s1_is_preconditioned_cg(oracle_lib):
    A = ei.poisson2d(24)
    D = A.to_dense()
    st, L = oracle_lib.ic0(A, 8)
    Ld = csr_of(L).to_dense()
    b = ei.uniform_pm1(21, A.n)
    kp, xp, xs = textbook_pcg(D, Ld, b, 1e-8, record=True)
    for method in ("sre-cg", "sre-cg2", "msdo-cg"):
        r = oracle_lib.solve(A, b, method, s=1, t=1, tol=1e-8, L=L)
        assert r["converged"] and abs(r["outer_iters"] - kp) <= 2, (method, r["outer_iters"], kp)
        for k in (1, 2, 5):
            rk = oracle_lib.solve(A, b, method, s=1, t=1, tol=0.0, kmax=k + 1, L=L)
            assert np.linalg.norm(rk["x"] - xs[k]) <= 1e-10 * np.linalg.norm(xs[k])
    # and the preconditioner helps: fewer iterations than CG on the same system
    plain = oracle_lib.solve(A, b, "sre-cg", s=1, t=1, tol=1e-8)
    assert kp < plain["outer_iters"]


@pytest.mark.parametrize("method", ["sre-cg", "sre-cg2", "msdo-cg"])
def test_exact_preconditioner_one_iteration(oracle_lib, method):
    n, nd = 128, 16
    D = tridiag_blocks(n, nd, seed=4)
    A = ei.csr_from_dense(D)
    st, L = oracle_lib.ic0(A, nd)
    b = ei.uniform_pm1(6, n)
    r = oracle_lib.solve(A, b, method, s=2, t=4, tol=1e-12, L=L)
    assert r["converged"] and r["outer_iters"] == 1
    assert np.linalg.norm(r["x"] - np.linalg.solve(D, b)) <= 1e-12 * np.linalg.norm(r["x"])


@pytest.mark.parametrize("method,s,t", [("sre-cg", 3, 4), ("sre-cg2", 2, 8), ("msdo-cg", 2, 4)])
def test_preconditioned_invariants(oracle_lib, method, s, t):
    N = 20
    A = ei.stencil_csr(N, N, ndim=2, kappa=ei.bands_kappa(N, band=4, hi=10.0))
    D = A.to_dense()
    st, L = oracle_lib.ic0(A, 16)
    xstar = ei.uniform01(3, A.n)
    b = D @ xstar
    E0 = xstar @ D @ xstar
    state = dict(eprev=E0, count=0)

    def cb(k, V, alpha, x, r, rho):
        state["count"] += 1
        assert np.abs(V.T @ D @ V - np.eye(V.shape[1])).max() <= 1e-10
        e = xstar - x
        Ek = e @ D @ e
        assert abs((state["eprev"] - Ek) - alpha @ alpha) <= 1e-10 * E0
        state["eprev"] = Ek
        assert np.linalg.norm(V.T @ r) <= 1e-10 * max(np.linalg.norm(alpha), 1e-300)

    out = oracle_lib.solve(A, b, method, s=s, t=t, tol=1e-8, callback=cb, L=L)
    assert out["converged"] and state["count"] == out["outer_iters"] >= 3
    plain = oracle_lib.solve(A, b, method, s=s, t=t, tol=1e-8)
    assert out["outer_iters"] < plain["outer_iters"]


def test_preconditioned_mirror_agrees(oracle_lib):
    A = ei.stencil_csr(32, 32, ndim=2, kappa=ei.bands_kappa(32, band=8, hi=100.0))
    st, L = oracle_lib.ic0(A, 64)
    b = ei.uniform_pm1(14, A.n)
    d = oracle_lib.solve(A, b, "sre-cg", s=3, t=4, tol=1e-8, L=L)
    m = oracle_lib.solve(A, b, "sre-cg", s=3, t=4, tol=1e-8, L=L, mode=oracle_lib.MODE_MIRROR)
    assert d["converged"] and m["converged"] and abs(d["outer_iters"] - m["outer_iters"]) <= 1
    assert np.linalg.norm(d["x"] - m["x"]) <= 1e-6 * np.linalg.norm(d["x"])


def test_ic0_breakdown_and_badarg(oracle_lib):
    D = np.array([[1.0, 2.0], [2.0, 1.0]])  # indefinite: the second pivot is 1 − 4 < 0
    st, _ = oracle_lib.ic0(ei.csr_from_dense(D), 1)
    assert st == oracle_lib.BREAKDOWN
    A = ei.poisson2d(8)
    st, L = oracle_lib.ic0(A, 4)
    b = ei.uniform_pm1(1, A.n)
    assert oracle_lib.solve(A, b, "sre-cg", s=2, t=2, L=L, restructured=True)["status"] == oracle_lib.BADARG


@pytest.mark.parametrize("method,arnoldi", [("sre-cg", 7), ("sre-cg2", 5), ("msdo-cg", 7)])
def test_preconditioned_ca(oracle_lib, method, arnoldi):
    """CA with M⁻¹A powers and the L⁻ᵗ[T(L⁻¹r)] seed.  s = 1 (Alg 5) is the preconditioned
    s-step method exactly; Poisson2D counts equal the preconditioned s-step counts (Table 5: the CA
    versions with Alg 7 converge like s-step); per-iteration A-orthonormality and Galerkin hold."""
    A = ei.poisson2d(40)
    st, L = oracle_lib.ic0(A, 16)
    b = ei.paper_poisson_rhs(A)
    if arnoldi == 5:
        c1 = oracle_lib.solve_ca(A, b, method, arnoldi=5, s=1, t=4, tol=1e-8, L=L)
        s1 = oracle_lib.solve(A, b, method, s=1, t=4, tol=1e-8, L=L)
        assert c1["outer_iters"] == s1["outer_iters"]
        assert np.array_equal(c1["x"], s1["x"])
    D = A.to_dense()

    def cb(k, V, alpha, x, r, rho):
        assert np.abs(V.T @ D @ V - np.eye(V.shape[1])).max() <= 1e-8
        assert np.linalg.norm(V.T @ r) <= 1e-8 * max(np.linalg.norm(alpha), 1e-300)

    ca = oracle_lib.solve_ca(A, b, method, arnoldi=arnoldi, s=3, t=4, tol=1e-8, L=L, callback=cb)
    ss = oracle_lib.solve(A, b, method, s=3, t=4, tol=1e-8, L=L)
    plain = oracle_lib.solve_ca(A, b, method, arnoldi=arnoldi, s=3, t=4, tol=1e-8)
    assert ca["converged"] and ss["converged"]
    assert abs(ca["outer_iters"] - ss["outer_iters"]) <= 1, (ca["outer_iters"], ss["outer_iters"])
    assert ca["outer_iters"] < plain["outer_iters"]


def test_complete_cholesky_blocks(oracle_lib):
    """Table 6's preconditioner: L·Lᵗ equals the block diagonal of A (numpy's Cholesky of each block);
    with it the preconditioned methods need no more iterations than with IC(0) (Table 6 vs 5)."""
    A = ei.poisson2d(24)
    nd = 8
    st, L = oracle_lib.ic0(A, nd, kind="chol")
    assert st == 0
    D = A.to_dense()
    Ld = csr_of(L).to_dense()
    dom = np.array([domain_of(A.n, nd, i) for i in range(A.n)])
    Dbd = np.where(dom[:, None] == dom[None, :], D, 0.0)
    assert np.abs(Ld - np.linalg.cholesky(Dbd)).max() <= 1e-13
    b = ei.uniform_pm1(8, A.n)
    st0, L0 = oracle_lib.ic0(A, nd)
    for method in ("sre-cg", "msdo-cg"):
        c = oracle_lib.solve(A, b, method, s=2, t=4, tol=1e-8, L=L)
        i = oracle_lib.solve(A, b, method, s=2, t=4, tol=1e-8, L=L0)
        assert c["converged"] and i["converged"] and c["outer_iters"] <= i["outer_iters"]
    # one domain: M = A, one outer iteration
    st1, L1 = oracle_lib.ic0(A, 1, kind="chol")
    r = oracle_lib.solve(A, b, "sre-cg", s=1, t=1, tol=1e-10, L=L1)
    assert r["outer_iters"] == 1 and np.linalg.norm(r["x"] - np.linalg.solve(D, b)) <= 1e-10 * np.linalg.norm(r["x"])
