"""Pins for the oracle's communication-avoiding variants: CA SRE-CG,
CA SRE-CG2 and CA MSDO-CG with the CA-Arnoldi A-orthonormalization
(Alg 5) or its modified form (Alg 7).

What fixes them without a second implementation:
* s = 1 reduces Alg 5 to the s-step orthonormalization operation for operation (bitwise);
* in exact arithmetic CA SRE-CG / CA SRE-CG2 span the same enlarged Krylov space as the s-step
  versions, so on the well-conditioned Poisson2D they take the same number of
  outer iterations ("converges in the same number of iterations");
* every basis is block A-orthonormal, the φ-decrease identity and the local Galerkin condition
  hold per outer iteration, and the method terminates exactly on tiny dense SPD
  systems after n/(st) outer iterations;
* the monomial basis loses rank for large s: a breakdown is reported, never a
  wrong answer.
"""
import math

import numpy as np
import pytest

import eks_inputs as ei


@pytest.mark.parametrize("method", ["sre-cg", "sre-cg2", "msdo-cg"])
def test_alg5_s1_is_sstep_bitwise(oracle_lib, method):
    A = ei.stencil_csr(20, 20, ndim=2, kappa=ei.bands_kappa(20, band=4, hi=10.0))
    b = ei.uniform_pm1(21, A.n)
    r = oracle_lib.solve(A, b, method, s=1, t=4, tol=1e-8)
    c = oracle_lib.solve_ca(A, b, method, arnoldi=5, s=1, t=4, tol=1e-8)
    assert r["outer_iters"] == c["outer_iters"]
    assert np.array_equal(r["x"], c["x"])


@pytest.mark.parametrize("method,t", [("sre-cg", 2), ("sre-cg2", 4), ("sre-cg", 4)])
@pytest.mark.parametrize("arnoldi", [5, 7])
def test_poisson2d_same_counts_as_sstep(oracle_lib, method, t, arnoldi):
    A = ei.poisson2d(64)
    b = ei.paper_poisson_rhs(A)
    for s in (2, 3, 5):
        r = oracle_lib.solve(A, b, method, s=s, t=t, tol=1e-6)
        c = oracle_lib.solve_ca(A, b, method, arnoldi=arnoldi, s=s, t=t, tol=1e-6)
        assert c["converged"] and r["converged"]
        assert c["outer_iters"] == r["outer_iters"], (s, c["outer_iters"], r["outer_iters"])
        assert c["true_relres"] <= 1.5e-6


@pytest.mark.parametrize("method,arnoldi,s,t", [("sre-cg", 7, 3, 4), ("sre-cg2", 7, 2, 8), ("msdo-cg", 7, 3, 4),
                                                 ("msdo-cg", 5, 2, 4)])
def test_ca_invariants_per_outer_iteration(oracle_lib, method, arnoldi, s, t):
    N = 24
    A = ei.stencil_csr(N, N, ndim=2, kappa=ei.bands_kappa(N, band=4, hi=10.0))
    D = A.to_dense()
    xstar = ei.uniform01(3, A.n)
    b = D @ xstar
    st = dict(E=xstar @ D @ xstar, count=0)

    def cb(k, V, alpha, x, r, rho):
        st["count"] += 1
        assert np.abs(V.T @ D @ V - np.eye(V.shape[1])).max() <= 1e-10  # one st×st CholQR
        e = xstar - x
        Ek = e @ D @ e
        assert abs((st["E"] - Ek) - alpha @ alpha) <= 1e-10 * (xstar @ D @ xstar)
        assert np.linalg.norm(V.T @ r) <= 1e-9 * max(1.0, np.linalg.norm(alpha))
        st["E"] = Ek

    res = oracle_lib.solve_ca(A, b, method, arnoldi=arnoldi, s=s, t=t, tol=1e-8, callback=cb)
    assert res["converged"] and st["count"] == res["outer_iters"] > 2


@pytest.mark.parametrize("method,n,s,t", [("sre-cg2", 24, 2, 4), ("msdo-cg", 24, 3, 2), ("sre-cg", 16, 2, 2)])
def test_ca_tiny_dense_exact_termination(oracle_lib, method, n, s, t):
    D = ei.spd_dense(n, seed=n + 7 * s + t, hi=10.0)
    A = ei.csr_from_dense(D)
    b = ei.uniform_pm1(n + 1, n)
    kk = n // (s * t)
    r = oracle_lib.solve_ca(A, b, method, arnoldi=7, s=s, t=t, tol=0.0, kmax=kk + 1)
    assert r["outer_iters"] == kk
    xd = np.linalg.solve(D, b)
    assert np.linalg.norm(r["x"] - xd) <= 1e-9 * np.linalg.norm(xd)


def test_monomial_basis_breakdown_is_reported(oracle_lib):
    # s = 10 monomial powers of T(r0) are numerically dependent in fp64: the st×st CholQR
    # pivot test (reading R6) fires and the solve stops with x = x0, no wrong answer.
    A = ei.poisson2d(64)
    b = ei.paper_poisson_rhs(A)
    c = oracle_lib.solve_ca(A, b, "sre-cg", arnoldi=7, s=10, t=2, tol=1e-6)
    assert c["status"] == oracle_lib.BREAKDOWN and c["outer_iters"] == 0
    assert np.abs(c["x"]).max() == 0.0
