"""Pins for the oracle's solver (Alg 3 / Alg 4 / Alg 6) against what the paper
and the mathematics fix:

* textbook CG (Hestenes–Stiefel) — written here independently in numpy —
  equals SRE-CG at t=1, s=1, and the s-step iterate x_k equals CG's x_{ks};
* exact termination on tiny dense SPD systems vs a dense direct solve;
* block A-orthonormality, the exact φ-decrease identity, local Galerkin,
  monotone A-norm error, full-Q Petrov–Galerkin;
* paper table cells on the regenerable Poisson2D (Tables 2–4, t=2 rows) and the
  ceil(k/s) relation;
* cross-method identities at k=1 (reading R14).
"""
import json
import math
import os

import numpy as np
import pytest

import eks_inputs as ei

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLD, "paper_poisson2d.json")))


def textbook_cg(A_dense_or_csr, b, tol, kmax=100000, record=False):
    """Hestenes–Stiefel CG (Alg 11 with M = I), numpy, independent of the oracle."""
    mv = (lambda v: ei.csr_matvec(A_dense_or_csr, v)) if isinstance(A_dense_or_csr, ei.Csr) \
        else (lambda v: A_dense_or_csr @ v)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = r @ r
    rho0 = math.sqrt(rr)
    xs = [x.copy()]
    k = 0
    while math.sqrt(rr) > tol * rho0 and k < kmax:
        w = mv(p)
        alpha = rr / (p @ w)
        x = x + alpha * p
        r = r - alpha * w
        rr_new = r @ r
        p = r + (rr_new / rr) * p
        rr = rr_new
        k += 1
        if record:
            xs.append(x.copy())
    return (k, x, xs) if record else (k, x)


# ---------------------------------------------------------------- CG equivalences
def test_t1_s1_equals_textbook_cg(oracle_lib):
    A = ei.poisson2d(40)
    b = ei.uniform_pm1(7, A.n)
    kcg, xcg, xs = textbook_cg(A, b, 1e-8, record=True)
    for method in ("sre-cg", "sre-cg2", "msdo-cg"):
        r = oracle_lib.solve(A, b, method, s=1, t=1, tol=1e-8)
        assert r["converged"]
        assert abs(r["outer_iters"] - kcg) <= 2, (method, r["outer_iters"], kcg)
        # iterates coincide early on (before rounding accumulates)
        for k in (1, 2, 5, 10):
            rk = oracle_lib.solve(A, b, method, s=1, t=1, tol=0.0, kmax=k + 1)
            assert np.linalg.norm(rk["x"] - xs[k]) <= 1e-10 * np.linalg.norm(xs[k])


@pytest.mark.parametrize("s", [2, 3, 5])
def test_t1_sstep_iterate_equals_cg_iterate_ks(oracle_lib, s):
    # exact arithmetic: x_k(s-step) = x_{ks}(CG)
    A = ei.poisson2d(30)
    b = ei.uniform_pm1(8, A.n)
    _, _, xs = textbook_cg(A, b, 0.0, kmax=4 * s, record=True)
    for k in (1, 2, 3):
        r = oracle_lib.solve(A, b, "sre-cg2", s=s, t=1, tol=0.0, kmax=k + 1)
        assert np.linalg.norm(r["x"] - xs[k * s]) <= 1e-9 * np.linalg.norm(xs[k * s])


# ---------------------------------------------------------------- exact termination
@pytest.mark.parametrize("method", ["sre-cg", "sre-cg2", "msdo-cg"])
@pytest.mark.parametrize("n,s,t", [(48, 3, 4), (64, 2, 8), (36, 1, 6), (32, 4, 2)])
def test_tiny_dense_spd_exact_termination(oracle_lib, method, n, s, t):
    # SRE-CG's 2-block window is exact only in exact arithmetic; its global
    # A-orthogonality decays like κ·ε·(#powers), so its pin uses Λ in [1,10].
    D = ei.spd_dense(n, seed=n + 10 * s + t, hi=10.0 if method == "sre-cg" else 100.0)
    A = ei.csr_from_dense(D)
    b = ei.uniform_pm1(n, n)
    kk = n // (s * t)
    r = oracle_lib.solve(A, b, method, s=s, t=t, tol=0.0, kmax=kk + 1)
    assert r["outer_iters"] == kk
    xd = np.linalg.solve(D, b)
    assert r["rho"] / r["rho0"] <= 1e-10
    assert np.linalg.norm(r["x"] - xd) <= 1e-10 * np.linalg.norm(xd)


# ---------------------------------------------------------------- per-iteration invariants
@pytest.mark.parametrize("method,s,t,mode,hi", [("sre-cg", 3, 4, 0, 10.0), ("sre-cg2", 2, 8, 0, 10.0),
                                                ("msdo-cg", 4, 4, 0, 10.0),
                                                # one-synch CGS2 (reading R36) on harder bands
                                                ("sre-cg", 3, 4, 2, 1e4), ("sre-cg2", 2, 8, 2, 1e4),
                                                ("msdo-cg", 4, 4, 2, 1e4)])
def test_invariants_per_outer_iteration(oracle_lib, method, s, t, mode, hi):
    N = 24
    A = ei.stencil_csr(N, N, ndim=2, kappa=ei.bands_kappa(N, band=4, hi=hi))
    D = A.to_dense()
    xstar = ei.uniform01(3, A.n)
    b = D @ xstar
    e0 = xstar.copy()
    E0 = e0 @ D @ e0
    state = dict(eprev=E0, Q=[], rho0=np.linalg.norm(b), count=0)

    def cb(k, V, alpha, x, r, rho):
        state["count"] += 1
        # block-wise A-orthonormality ‖VᵀAV − I‖_max ≤ 1e-10 (north_star)
        assert np.abs(V.T @ D @ V - np.eye(V.shape[1])).max() <= 1e-10
        # exact φ-decrease identity ‖e_{k-1}‖²_A − ‖e_k‖²_A = ‖α̃_k‖²
        e = xstar - x
        Ek = e @ D @ e
        assert abs((state["eprev"] - Ek) - alpha @ alpha) <= 1e-10 * E0
        assert Ek <= state["eprev"] * (1 + 1e-13)       # monotone A-norm error
        state["eprev"] = Ek
        # local Galerkin Vᵀ r_k = 0
        assert np.linalg.norm(V.T @ r) <= 1e-10 * max(np.linalg.norm(alpha), 1e-300)
        state["Q"].append(V)
        if method != "sre-cg":  # full-Q Petrov–Galerkin
            Qm = np.hstack(state["Q"])
            assert np.abs(Qm.T @ r).max() <= 1e-8 * state["rho0"]

    out = oracle_lib.solve(A, b, method, s=s, t=t, tol=1e-8, callback=cb, mode=mode)
    assert out["converged"] and state["count"] == out["outer_iters"] > 3
    assert out["true_relres"] <= 1e-7


# ---------------------------------------------------------------- paper cells
@pytest.fixture(scope="module")
def poisson_paper():
    A = ei.poisson2d(100)
    assert (A.n, A.nnz) == (PAPER["n"], PAPER["nnz"])
    return A, ei.paper_poisson_rhs(A)


def test_paper_cg_195(poisson_paper):
    A, b = poisson_paper
    k, _ = textbook_cg(A, b, PAPER["tol"])
    assert abs(k - PAPER["cg_iterations"]) <= PAPER["tolerance_cg"] * PAPER["cg_iterations"]


@pytest.mark.parametrize("key,method", [("sre_cg_t2", "sre-cg"), ("sre_cg2_t2", "sre-cg2"),
                                        ("msdo_cg_t2", "msdo-cg"), ("sre_cg_t4", "sre-cg")])
def test_paper_table_rows(oracle_lib, poisson_paper, key, method):
    A, b = poisson_paper
    row = PAPER[key]
    t = 4 if key.endswith("t4") else 2
    got = {}
    for s, want in zip(row["s"], row["k"]):
        r = oracle_lib.solve(A, b, method, s=s, t=t, tol=PAPER["tol"])
        assert r["converged"]
        got[s] = r["outer_iters"]
        assert abs(got[s] - want) <= PAPER["tolerance_enlarged"] * want, (key, s, got[s], want)
    if method != "msdo-cg":
        # Poisson2D: the s-step count equals ceil(k(s=1)/s) exactly
        for s in row["s"]:
            assert got[s] == math.ceil(got[1] / s), (key, s, got)


# ---------------------------------------------------------------- cross-method identities
def test_first_outer_iteration_cross_method_bitwise(oracle_lib):
    A = ei.stencil_csr(20, 20, ndim=2, kappa=ei.bands_kappa(20, band=5))
    b = ei.uniform_pm1(21, A.n)
    for s in (1, 2, 3, 4):
        r2 = oracle_lib.solve(A, b, "sre-cg2", s=s, t=4, tol=0.0, kmax=2)
        rm = oracle_lib.solve(A, b, "msdo-cg", s=s, t=4, tol=0.0, kmax=2)
        assert np.array_equal(r2["x"], rm["x"])            # reading R14
        if s <= 3:
            r1 = oracle_lib.solve(A, b, "sre-cg", s=s, t=4, tol=0.0, kmax=2)
            assert np.array_equal(r1["x"], r2["x"])         # window covers all blocks


def test_mirror_mode_agrees_with_definition(oracle_lib):
    p = ei.cfg1()
    d = oracle_lib.solve(p.A, p.b, p.method, p.s, p.t, p.tol, mode=oracle_lib.MODE_DEFINITION)
    m = oracle_lib.solve(p.A, p.b, p.method, p.s, p.t, p.tol, mode=oracle_lib.MODE_MIRROR)
    assert d["converged"] and m["converged"]
    assert abs(d["outer_iters"] - m["outer_iters"]) <= 1
    assert np.linalg.norm(d["x"] - m["x"]) <= 1e-7 * np.linalg.norm(d["x"])


@pytest.mark.parametrize("method,s,t,N,hi", [("sre-cg", 3, 16, 48, 1e3), ("sre-cg2", 2, 8, 32, 1e3),
                                            ("msdo-cg", 4, 4, 32, 1e3), ("sre-cg", 1, 1, 32, 1.0)])
def test_onesynch_agrees_with_definition(oracle_lib, method, s, t, N, hi):
    """One-synch CGS2 (reading R36: SpMM of Z1, Z2ᵀAZ2 = Z1ᵀAZ1 − C2ᵀC2, A·Z2 = A·Z1 − (AQ)C2) against
    the definition mode (two explicit CGS passes Qᵀ(A·Z), R3): the first two outer iterations'
    x within 1e-10, converged x within 1e-7, outer-iteration counts within 1."""
    A = ei.stencil_csr(N, N, ndim=2, kappa=ei.bands_kappa(N, band=4, hi=hi))
    b = ei.uniform_pm1(1806, A.n)
    pre = [oracle_lib.solve(A, b, method, s, t, 0.0, kmax=3, mode=m) for m in (0, 2)]
    assert pre[0]["outer_iters"] == pre[1]["outer_iters"] == 2
    assert np.linalg.norm(pre[1]["x"] - pre[0]["x"]) <= 1e-10 * np.linalg.norm(pre[0]["x"])
    d, o = (oracle_lib.solve(A, b, method, s, t, 1e-8, mode=m) for m in (0, 2))
    assert d["converged"] and o["converged"]
    assert abs(d["outer_iters"] - o["outer_iters"]) <= 1
    assert np.linalg.norm(o["x"] - d["x"]) <= 1e-7 * np.linalg.norm(d["x"])
    assert o["true_relres"] <= 2e-8


def test_onesynch_rejects_pre_cholqr_and_restructured(oracle_lib):
    p = ei.cfg1()
    for kw in (dict(ortho="pre-cholqr"), dict(restructured=True)):
        assert oracle_lib.solve(p.A, p.b, "sre-cg", 2, 4, 1e-8, mode=2, **kw)["status"] == oracle_lib.BADARG


# ---------------------------------------------------------------- degenerate cases
def test_zero_rhs_returns_immediately(oracle_lib):
    A = ei.poisson2d(8)
    r = oracle_lib.solve(A, np.zeros(A.n), "sre-cg", s=2, t=4, tol=1e-8)
    assert r["outer_iters"] == 0 and r["converged"] and np.all(r["x"] == 0)


def test_msdo_zero_domain_residual_is_breakdown(oracle_lib):
    A = ei.poisson2d(8)
    b = ei.uniform_pm1(2, A.n)
    b[: A.n // 4] = 0.0  # T_1(r0) = 0 → singular Gram (reading R13)
    r = oracle_lib.solve(A, b, "msdo-cg", s=2, t=4, tol=1e-8)
    assert r["status"] == oracle_lib.BREAKDOWN and r["outer_iters"] == 0
    assert r["breakdown_block"] == 0 and np.all(r["x"] == 0)


def test_kmax_cap_reports_not_converged(oracle_lib):
    p = ei.cfg1()
    r = oracle_lib.solve(p.A, p.b, p.method, p.s, p.t, p.tol, kmax=5)
    assert r["outer_iters"] == 4 and not r["converged"] and r["status"] == oracle_lib.MAXITER


def test_basis_sweep_matches_first_iteration_basis(oracle_lib):
    A = ei.poisson2d(16)
    b = ei.uniform_pm1(5, A.n)
    s, t = 4, 4
    V = {}
    oracle_lib.solve(A, b, "sre-cg", s=s, t=t, tol=0.0, kmax=2, callback=lambda k, VV, *a: V.setdefault(k, VV))
    st, W = oracle_lib.basis_sweep(A, oracle_lib.split(b, t), s)
    assert st == 0 and np.array_equal(W, V[1][:, (s - 1) * t:])


def test_cfg1_oracle_full_solve(oracle_lib):
    p = ei.cfg1()
    r = oracle_lib.solve(p.A, p.b, p.method, p.s, p.t, p.tol)
    assert r["converged"] and r["true_relres"] <= 1e-8 * 1.5
    # s=1 vs s=2 on a Poisson matrix: ceil relation
    r1 = oracle_lib.solve(p.A, p.b, p.method, 1, p.t, p.tol)
    assert r["outer_iters"] == math.ceil(r1["outer_iters"] / 2)


def _dense(A):
    D = np.zeros((A.n, A.n))
    for i in range(A.n):
        D[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
    return D


@pytest.mark.parametrize("t", [4, 8])
def test_basis_sweep_pinned_by_krylov_structure(oracle_lib, t):
    """or_basis_sweep (cfg5, reading R27) against what Alg 4 fixes, independently of the oracle's solve:
    block 1 is the A-CholQR of X0 (numpy Cholesky of X0ᵀAX0, P:380 R4); every block is A-orthonormal and
    A-orthogonal to the two before it; A·W_{j−1} lies in span{W_{j−2}, W_{j−1}, W_j} (the
    three-block recurrence of the SRE-CG basis) — so a dropped CGS term, a wrong window or
    a transposed coefficient fails one of these."""
    A = ei.stencil_csr(7, 6, 5, ndim=3)
    X0 = ei.cfg5_start_block(A.n, t)
    D = _dense(A)
    W = [oracle_lib.basis_sweep(A, X0, j)[1] for j in range(1, 7)]
    # block 1 = X0 R⁻¹ with RᵀR = X0ᵀAX0
    R = np.linalg.cholesky(X0.T @ D @ X0).T
    assert np.abs(W[0] - np.linalg.solve(R.T, X0.T).T).max() <= 1e-12 * np.abs(W[0]).max()
    for j, Wj in enumerate(W):
        assert np.abs(Wj.T @ D @ Wj - np.eye(t)).max() <= 1e-10
        for k in (j - 1, j - 2):
            if k >= 0:
                assert np.abs(W[k].T @ D @ Wj).max() <= 1e-10, (j, k)
        if j >= 1:
            Z = D @ W[j - 1]
            Pz = sum(W[k] @ (W[k].T @ D @ Z) for k in range(max(0, j - 2), j + 1))
            assert np.linalg.norm(Z - Pz) <= 1e-9 * np.linalg.norm(Z), j


@pytest.mark.parametrize("method,s,t,kw", [("sre-cg", 3, 8, {}), ("sre-cg2", 2, 4, {}), ("msdo-cg", 3, 4, {}),
                                         ("sre-cg", 2, 4, dict(ortho="pre-cholqr")),
                                         ("sre-cg2", 2, 4, dict(restructured=True)),
                                         ("sre-cg", 2, 8, dict(precond=16)), ("msdo-cg", 2, 4, dict(precond=16))])
def test_mirror_mode_prefix_pinned(oracle_lib, method, s, t, kw):
    """The oracle's MIRROR mode (the GPU's algebra: cached A·Q, C = (AQ)ᵀZ, r −= Σ(AW)α̃; reading R24/R9)
    against the DEFINITION mode step by step, not only at convergence: after each of the first three outer
    iterations x, the recursive residual r and ρ agree within 1e-10 (equal in exact arithmetic), and
    every basis block of the mirror run is A-orthonormal — on κ = 1e3 bands."""
    A = ei.stencil_csr(24, 24, ndim=2, kappa=ei.bands_kappa(24, band=4, hi=1e3))
    b = ei.uniform_pm1(1806, A.n)
    L = None
    if "precond" in kw:
        st, L = oracle_lib.ic0(A, kw.pop("precond"))
        assert st == 0
    its = {0: {}, 1: {}}
    D = _dense(A)
    for mode in (0, 1):
        def cb(k, V, alpha, x, r, rho, m=mode):
            its[m][k] = (x.copy(), r.copy(), rho, V.copy())
        res = oracle_lib.solve(A, b, method, s, t, 0.0, kmax=4, mode=mode, callback=cb, L=L, **kw)
        assert res["outer_iters"] == 3
    for k in (1, 2, 3):
        xd, rd, rhod, _ = its[0][k]
        xm, rm, rhom, Vm = its[1][k]
        assert np.abs(xm - xd).max() <= 1e-10 * np.abs(xd).max(), (k, "x")
        assert np.abs(rm - rd).max() <= 1e-10 * np.abs(rd).max(), (k, "r")
        assert abs(rhom - rhod) <= 1e-10 * rhod
        for i in range(s):
            Wi = Vm[:, i * t:(i + 1) * t]
            if not kw.get("restructured"):
                assert np.abs(Wi.T @ D @ Wi - np.eye(t)).max() <= 1e-9, (k, i)
