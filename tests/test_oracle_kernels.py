"""Pins for the oracle's kernel-level routines against things the paper and the
mathematics fix (never against a retyped copy of the oracle's own formula):

* T(r): Theorem 1's identity r = T(r)·1_t and SPEC's worked example.
* SpMM: exact integer A·1 face counts, Dirichlet-Laplacian eigenpairs (closed form).
* Xᵀ Y: exact integer arithmetic.
* Cholesky / A-CholQR: SPEC's hand 2×2 case, LAPACK (numpy) on random SPD,
  eigenvector blocks (R = diag(√λ)), breakdown on duplicate columns.
* CGS2: eigenvector blocks (projection = exact complement), idempotence.
"""
import json
import math
import os

import numpy as np
import pytest

import eks_inputs as ei

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))


# ---------------------------------------------------------------- T(r)
def test_split_spec_example(oracle_lib):
    g = SPEC["split_T"]
    Z = oracle_lib.split(np.array(g["r"], float), g["t"])
    assert np.array_equal(Z, np.array(g["Z"], float))


@pytest.mark.parametrize("n,t", [(10, 3), (4096, 4), (1001, 64), (7, 7), (5, 1)])
def test_split_theorem1_identity(oracle_lib, n, t):
    r = ei.uniform_pm1(11, n)
    Z = oracle_lib.split(r, t)
    # r = T(r)·1_t exactly, each column supported on its own domain
    assert np.array_equal(Z.sum(axis=1), r)
    assert np.array_equal(np.count_nonzero(Z, axis=1), np.ones(n))
    for d in range(t):
        lo, hi = d * n // t, (d + 1) * n // t
        assert np.array_equal(np.nonzero(Z[:, d])[0], np.arange(lo, hi))


# ---------------------------------------------------------------- SpMM
def test_spmm_spec_examples(oracle_lib):
    A = ei.poisson2d(2)
    y = oracle_lib.spmm(A, np.ones((4, 1)))
    assert np.array_equal(y[:, 0], np.array(SPEC["spmm_poisson2_ones"]["y"]))
    D = ei.csr_from_dense(np.array(SPEC["spmm_diag"]["A"], float))
    Y = oracle_lib.spmm(D, np.array(SPEC["spmm_diag"]["X"], float))
    assert np.array_equal(Y, np.array(SPEC["spmm_diag"]["Y"], float))
    I = ei.csr_from_dense(np.eye(5))
    X = ei.uniform_pm1(3, 15).reshape(5, 3)
    assert np.array_equal(oracle_lib.spmm(I, X), X)


@pytest.mark.parametrize("ndim,N", [(2, 9), (3, 6)])
def test_spmm_ones_counts_boundary_faces(oracle_lib, ndim, N):
    A = ei.stencil_csr(N, N, N, ndim=ndim) if ndim == 3 else ei.poisson2d(N)
    y = oracle_lib.spmm(A, np.ones((A.n, 2)))
    idx = np.arange(A.n)
    coords = [idx % N, (idx // N) % N, idx // (N * N)][:ndim]
    faces = sum((c == 0).astype(int) + (c == N - 1) for c in coords)
    assert np.array_equal(y[:, 0], faces.astype(float))
    assert np.array_equal(y[:, 1], faces.astype(float))


def _laplace_eig(N, ndim, modes):
    idx = np.arange(N ** ndim)
    coords = [idx % N, (idx // N) % N, idx // (N * N)][:ndim]
    V, lam = [], []
    for m in modes:
        v = np.ones(N ** ndim)
        l = 0.0
        for c, p in zip(coords, m):
            v = v * np.sin(p * np.pi * (c + 1) / (N + 1))
            l += 2.0 - 2.0 * np.cos(p * np.pi / (N + 1))
        V.append(v / np.linalg.norm(v))
        lam.append(l)
    return np.stack(V, 1), np.array(lam)


@pytest.mark.parametrize("ndim,N", [(2, 31), (3, 10)])
def test_spmm_laplacian_eigenvectors(oracle_lib, ndim, N):
    modes = [(1, 1, 1), (2, 3, 1), (5, 1, 2), (N, N, N), (3, 3, 3), (7, 2, 4)]
    X, lam = _laplace_eig(N, ndim, modes)
    A = ei.stencil_csr(N, N, N, ndim=ndim) if ndim == 3 else ei.poisson2d(N)
    Y = oracle_lib.spmm(A, X)
    err = np.abs(Y - X * lam).max() / np.abs(X * lam).max()
    assert err <= 1e-14


def test_spmm_symmetry_identity(oracle_lib):
    A = ei.stencil_csr(10, 10, 10, ndim=3, kappa=ei.subcubes_kappa(10, cell=2))
    U = ei.uniform_pm1(5, A.n * 2).reshape(A.n, 2)
    AU = oracle_lib.spmm(A, U)
    a, b = U[:, 0] @ AU[:, 1], U[:, 1] @ AU[:, 0]
    assert abs(a - b) <= 1e-13 * abs(a)


# ---------------------------------------------------------------- XᵀY
def test_xty_exact_integers(oracle_lib):
    rng = np.random.default_rng(0)
    X = rng.integers(-1000, 1000, size=(5000, 3)).astype(float)
    Y = rng.integers(-1000, 1000, size=(5000, 4)).astype(float)
    Cm = oracle_lib.xty(X, Y)
    exact = [[sum(int(X[i, a]) * int(Y[i, b]) for i in range(5000)) for b in range(4)] for a in range(3)]
    assert np.array_equal(Cm, np.array(exact, float))


# ---------------------------------------------------------------- Cholesky / A-CholQR
def test_acholqr_spec_hand_case(oracle_lib):
    g = SPEC["a_cholqr_2x2"]
    A = ei.csr_from_dense(np.array(g["A"], float))
    st, W, R, B = oracle_lib.acholqr(A, np.array(g["W"], float))
    assert st == 0
    assert np.allclose(R, np.array(g["R"]), atol=1e-13, rtol=0)
    assert R[0, 0] == 2.0 and R[0, 1] == 0.5 and abs(R[1, 1] - math.sqrt(2.75)) <= 1e-15
    D = np.array(g["A"], float)
    assert np.abs(W.T @ D @ W - np.eye(2)).max() <= 1e-15


@pytest.mark.parametrize("t", [1, 2, 4, 8, 16, 32, 64])
def test_chol_matches_lapack(oracle_lib, t):
    G = ei.uniform_pm1(100 + t, t * t).reshape(t, t)
    B = G @ G.T + t * np.eye(t)
    st, R = oracle_lib.chol(np.triu(B))
    assert st == 0
    L = np.linalg.cholesky(B)  # LAPACK dpotrf
    assert np.abs(R - L.T).max() <= 1e-13 * np.abs(L).max()
    assert np.array_equal(R, np.triu(R))


def test_chol_breakdown_on_singular(oracle_lib):
    v = ei.uniform_pm1(1, 4)
    B = np.outer(v, v)
    st, _ = oracle_lib.chol(B)
    assert st == oracle_lib.BREAKDOWN
    B2 = np.diag([1.0, -1.0, 1.0])
    assert oracle_lib.chol(B2)[0] == oracle_lib.BREAKDOWN
    assert oracle_lib.chol(np.diag([1.0, np.nan]))[0] == oracle_lib.BREAKDOWN


def test_acholqr_eigenvector_block_closed_form(oracle_lib):
    N = 24
    X, lam = _laplace_eig(N, 2, [(1, 1), (2, 1), (1, 2), (3, 5)])
    A = ei.poisson2d(N)
    st, W, R, _ = oracle_lib.acholqr(A, X)
    assert st == 0
    # XᵀAX = diag(λ) ⇒ R = diag(√λ), W = X diag(λ^{-1/2})
    assert np.abs(R - np.diag(np.sqrt(lam))).max() <= 1e-14 * np.sqrt(lam.max())
    assert np.abs(W - X / np.sqrt(lam)).max() <= 1e-13


def test_acholqr_duplicate_columns_breakdown_and_single_column(oracle_lib):
    A = ei.poisson2d(8)
    v = ei.uniform_pm1(4, A.n)
    st, *_ = oracle_lib.acholqr(A, np.stack([v, v], 1))
    assert st == oracle_lib.BREAKDOWN
    st, W, R, _ = oracle_lib.acholqr(A, v[:, None])
    D = A.to_dense()
    assert st == 0 and np.allclose(W[:, 0], v / math.sqrt(v @ D @ v), rtol=1e-14, atol=0)


def test_acholqr_a_orthonormal_random(oracle_lib):
    A = ei.stencil_csr(16, 16, ndim=2, kappa=ei.bands_kappa(16, band=4))
    Z = ei.uniform_pm1(9, A.n * 8).reshape(A.n, 8)
    st, W, R, B = oracle_lib.acholqr(A, Z)
    D = A.to_dense()
    assert st == 0
    assert np.abs(W.T @ D @ W - np.eye(8)).max() <= 1e-12
    assert np.abs(np.triu(Z.T @ D @ Z) - B).max() <= 1e-12 * np.abs(B).max()


# ---------------------------------------------------------------- CGS2
def test_cgs2_eigenvector_projection_exact_complement(oracle_lib):
    N = 20
    A = ei.poisson2d(N)
    X, lam = _laplace_eig(N, 2, [(1, 1), (2, 1), (1, 2), (2, 2), (3, 1), (1, 3)])
    Q = [X[:, :2] / np.sqrt(lam[:2]), X[:, 2:4] / np.sqrt(lam[2:4])]   # A-orthonormal blocks
    coef = np.array([[1.0, -2.0], [0.5, 3.0], [2.0, 1.0], [-1.0, 0.25], [4.0, -1.0], [0.0, 2.0]])
    Z = X @ coef
    Z2, C1, C2 = oracle_lib.cgs2(A, Z, Q)
    # exact: Z2 = component in span{x_5, x_6}
    assert np.abs(Z2 - X[:, 4:] @ coef[4:]).max() <= 1e-13
    # first-pass coefficients: (Q_q)ᵀ A Z = sqrt(λ) * coef rows of the block
    want = np.vstack([np.sqrt(lam[:4])[:, None] * coef[:4]])
    assert np.abs(C1 - want).max() <= 1e-13
    assert np.abs(C2).max() <= 1e-13   # second pass removes only rounding


def test_cgs2_projection_idempotent_and_member(oracle_lib):
    A = ei.stencil_csr(12, 12, ndim=2, kappa=ei.bands_kappa(12, band=3))
    D = A.to_dense()
    n, t = A.n, 4
    st, W1, _, _ = oracle_lib.acholqr(A, ei.uniform_pm1(1, n * t).reshape(n, t))
    Z = ei.uniform_pm1(2, n * t).reshape(n, t)
    Z, _, _ = oracle_lib.cgs2(A, Z, [W1])
    st, W2, _, _ = oracle_lib.acholqr(A, Z)
    Zn = ei.uniform_pm1(3, n * t).reshape(n, t)
    Z2, _, _ = oracle_lib.cgs2(A, Zn, [W1, W2])
    Qm = np.hstack([W1, W2])
    anorm = math.sqrt(np.trace(Z2.T @ D @ Z2))
    assert np.abs(Qm.T @ D @ Z2).max() <= 1e-12 * anorm
    Z3, _, _ = oracle_lib.cgs2(A, Z2, [W1, W2])   # a third pass changes nothing
    assert np.abs(Z3 - Z2).max() <= 1e-14 * np.abs(Z2).max()
    Zm, _, _ = oracle_lib.cgs2(A, W1[:, :1].repeat(t, 1), [W1])  # member of Q → 0
    assert np.abs(Zm).max() <= 1e-14
