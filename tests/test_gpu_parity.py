"""GPU parity: every step of the hot path, called through the C ABI of libeks.so,
against the oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star):
* T(r), SpMM: bitwise (same fma order, reading R20); Cholesky factor R: bitwise for equal B.
* Gram / CGS2 / CholQR outputs: normwise relative 1e-12 (CGS2 pass-2 coefficients
  normalised by ||AQ||_F ||Z||_F, reading R25).
* End to end: both reach relres <= 1e-8, outer iterations within max(5%, 1), x within 1e-6.
"""
import math
import os

import numpy as np
import pytest

import eks_inputs as ei

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

TS = [1, 2, 4, 8, 16, 32, 64]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def eks(torch_cuda):
    from paper_1804_10629_b200 import build
    build.build()
    import paper_1804_10629_b200 as m
    return m


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ------------------------------------------------------------------ operators used below
def op_2d_bands(N=37):  # ragged n (not a multiple of any tile), jump coefficients
    return ei.stencil_csr(N, N, ndim=2, kappa=ei.bands_kappa(N, band=4))


# ------------------------------------------------------------------ (a1) split
@pytest.mark.parametrize("t", TS)
@pytest.mark.parametrize("n", [1000, 4096, 12345])
def test_split_bitwise(eks, torch_cuda, oracle_lib, t, n):
    torch = torch_cuda
    A = ei.poisson2d(int(math.isqrt(n)))
    if A.n != n:
        A = ei.stencil_csr(n, 1, ndim=2)  # 1D chain of length n
    s = eks.Solver(A)
    r = ei.uniform_pm1(3, A.n)
    Z = torch.empty(A.n, t, dtype=torch.float64, device="cuda")
    eks.eks_k_split(s.ctx, t, dev(torch, r), Z)
    assert np.array_equal(host(Z), oracle_lib.split(r, t))
    s.close()


# ------------------------------------------------------------------ (a2) SpMM + Gram
@pytest.mark.parametrize("t", TS)
@pytest.mark.parametrize("opname", ["poisson64", "bands37", "aniso13"])
def test_spmm_bitwise_and_gram(eks, torch_cuda, oracle_lib, t, opname):
    torch = torch_cuda
    A = {"poisson64": lambda: ei.poisson2d(64), "bands37": op_2d_bands,
         "aniso13": lambda: ei.stencil_csr(13, 13, 13, ndim=3, scale=(1.0, 1.0, 1e-2))}[opname]()
    s = eks.Solver(A)
    X = ei.uniform_pm1(5, A.n * t).reshape(A.n, t)
    v = ei.uniform_pm1(6, A.n)
    Y = torch.empty(A.n, t, dtype=torch.float64, device="cuda")
    G = torch.empty(t, t, dtype=torch.float64, device="cuda")
    g = torch.empty(t, dtype=torch.float64, device="cuda")
    eks.eks_k_spmm(s.ctx, t, dev(torch, X), Y, G, dev(torch, v), g)
    Yo = oracle_lib.spmm(A, X)
    assert np.array_equal(host(Y), Yo)                     # bitwise (R20)
    assert rel(host(G), oracle_lib.xty(X, Yo)) <= 1e-12    # Gram XᵀAX
    assert rel(host(g), oracle_lib.xty(X, v[:, None])[:, 0]) <= 1e-12
    s.close()


# ------------------------------------------------------------------ (a4) Cholesky
@pytest.mark.parametrize("t", TS)
def test_chol_bitwise(eks, torch_cuda, oracle_lib, t):
    torch = torch_cuda
    A = ei.poisson2d(16)
    s = eks.Solver(A)
    Gm = ei.uniform_pm1(40 + t, t * t).reshape(t, t)
    B = Gm @ Gm.T + 0.1 * np.eye(t)
    R = torch.empty(t, t, dtype=torch.float64, device="cuda")
    st = eks.eks_k_chol(s.ctx, t, dev(torch, B), R)
    so, Ro = oracle_lib.chol(B)
    assert st == 0 and so == 0
    assert np.array_equal(np.triu(host(R)), Ro)
    # breakdown on a singular Gram (duplicate columns)
    if t >= 2:
        v = ei.uniform_pm1(1, t)
        Bs = np.outer(v, v)
        assert eks.eks_k_chol(s.ctx, t, dev(torch, Bs), R) == eks.EKS_ERR_BREAKDOWN
        assert oracle_lib.chol(Bs)[0] == oracle_lib.BREAKDOWN
    s.close()


# ------------------------------------------------------------------ (a3) CGS2 and (a4) A-CholQR
@pytest.mark.parametrize("t", [1, 4, 16, 32, 64])
@pytest.mark.parametrize("nq", [1, 2, 5])
def test_cgs2_and_acholqr_parity(eks, torch_cuda, oracle_lib, t, nq):
    torch = torch_cuda
    A = op_2d_bands(41)
    n = A.n
    s = eks.Solver(A)
    # build an A-orthonormal window with the oracle, so both sides see identical Q
    Qs, AQs = [], []
    for j in range(nq):
        Z0 = ei.uniform_pm1(100 + j, n * t).reshape(n, t)
        if Qs:
            Z0, _, _ = oracle_lib.cgs2(A, Z0, Qs)
        st, W, R, B = oracle_lib.acholqr(A, Z0)
        assert st == 0
        Qs.append(W)
        AQs.append(oracle_lib.spmm(A, W))
    Z = ei.uniform_pm1(7, n * t).reshape(n, t)
    Zo, C1o, C2o = oracle_lib.cgs2(A, Z, Qs)
    Zd = dev(torch, Z)
    C1 = torch.empty(nq * t, t, dtype=torch.float64, device="cuda")
    C2 = torch.empty(nq * t, t, dtype=torch.float64, device="cuda")
    eks.eks_k_cgs2(s.ctx, t, [dev(torch, q) for q in Qs], [dev(torch, q) for q in AQs], Zd, C1, C2)
    assert rel(host(Zd), Zo) <= 1e-12
    assert rel(host(C1), C1o) <= 1e-12
    scale = math.sqrt(sum(np.linalg.norm(q) ** 2 for q in AQs)) * np.linalg.norm(Z)
    assert np.linalg.norm(host(C2) - C2o) <= 1e-12 * scale       # reading R25
    # A-CholQR of the projected block
    W = torch.empty(n, t, dtype=torch.float64, device="cuda")
    AW = torch.empty_like(W)
    R = torch.empty(t, t, dtype=torch.float64, device="cuda")
    B = torch.empty(t, t, dtype=torch.float64, device="cuda")
    st = eks.eks_k_acholqr(s.ctx, t, dev(torch, Zo), W, AW, R, B)
    so, Wo, Ro, Bo = oracle_lib.acholqr(A, Zo)
    assert st == 0 and so == 0
    assert rel(np.triu(host(B)), Bo) <= 1e-12
    assert rel(np.triu(host(R)), Ro) <= 1e-12
    assert rel(host(W), Wo) <= 1e-11
    Wh = host(W)
    D = oracle_lib.xty(Wh, oracle_lib.spmm(A, Wh))
    assert np.abs(D - np.eye(t)).max() <= 1e-10                   # block A-orthonormality
    s.close()


# ------------------------------------------------------------------ end to end
def _e2e(eks, torch, oracle_lib, A, b, method, s_, t, tol, kmax=5000, mode=0):
    S = eks.Solver(A)
    rep = S.solve(dev(torch, b), method, s_, t, tol, max_outer=kmax)
    S.close()
    ref = oracle_lib.solve(A, b, method, s_, t, tol, kmax=kmax, mode=mode)
    return rep, ref


@pytest.mark.parametrize("method,s_,t", [("sre-cg", 2, 4), ("sre-cg2", 2, 4), ("msdo-cg", 2, 4),
                                         ("sre-cg", 1, 1), ("sre-cg", 3, 16), ("msdo-cg", 4, 8)])
def test_cfg1_end_to_end(eks, torch_cuda, oracle_lib, method, s_, t):
    p = ei.cfg1()
    rep, ref = _e2e(eks, torch_cuda, oracle_lib, p.A, p.b, method, s_, t, p.tol)
    assert rep["status"] == 0 and rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    assert rep["true_relres"] <= 1.5e-8 and ref["true_relres"] <= 1.5e-8
    assert rep["rho"] <= p.tol * rep["rho0"]
    assert abs(rep["rho0"] - ref["rho0"]) <= 1e-14 * ref["rho0"]


@pytest.mark.parametrize("method", ["sre-cg", "sre-cg2"])
def test_cfg2_analog_end_to_end(eks, torch_cuda, oracle_lib, method):
    # cfg2 recipe at 64² (the oracle cannot finish 512² in seconds): bands of 32, t=16, s=3
    p = ei.cfg2(N=64, method=method)
    rep, ref = _e2e(eks, torch_cuda, oracle_lib, p.A, p.b, method, p.s, p.t, p.tol)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    assert rep["true_relres"] <= 2e-8


# ------------------------------------------------------------------ §8(f) row 3: Pre-CholQR, restructured
@pytest.mark.parametrize("method,s_,t,ortho,restr", [
    ("sre-cg", 2, 4, "pre-cholqr", False), ("sre-cg2", 2, 4, "pre-cholqr", False),
    ("msdo-cg", 2, 4, "pre-cholqr", False), ("sre-cg", 3, 16, "pre-cholqr", False),
    ("sre-cg", 4, 2, "pre-cholqr", False), ("sre-cg", 3, 4, "acholqr", True), ("sre-cg2", 2, 8, "acholqr", True),
    ("sre-cg", 3, 16, "acholqr", True), ("sre-cg", 2, 32, "pre-cholqr", True)])
def test_pre_cholqr_restructured_end_to_end(eks, torch_cuda, oracle_lib, method, s_, t, ortho, restr):
    """Pre-CholQR (reading R30) and restructured Alg 2 / Alg 1 (reading R31) on cfg1: counts within
    5 %, x within 1e-6 of the oracle (mirror mode, the GPU's algebra), and after two outer
    iterations (tol = 0) x agrees to 1e-10."""
    p = ei.cfg1()
    S = eks.Solver(p.A)
    rep = S.solve(dev(torch_cuda, p.b), method, s_, t, p.tol, ortho=ortho, restructured=restr)
    pre = S.solve(dev(torch_cuda, p.b), method, s_, t, 0.0, max_outer=3, ortho=ortho, restructured=restr)
    S.close()
    ref = oracle_lib.solve(p.A, p.b, method, s_, t, p.tol, mode=oracle_lib.MODE_MIRROR, ortho=ortho,
                           restructured=restr)
    refp = oracle_lib.solve(p.A, p.b, method, s_, t, 0.0, kmax=3, mode=oracle_lib.MODE_MIRROR, ortho=ortho,
                            restructured=restr)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    assert rep["true_relres"] <= 1.5e-8
    assert pre["outer_iters"] == refp["outer_iters"] == 2
    assert rel(host(pre["x"]), refp["x"]) <= 1e-10
    # and against the oracle's DEFINITION mode (explicit SpMMs Qᵀ(A·Z), u = Vα̃, r −= A·u)
    dref = oracle_lib.solve(p.A, p.b, method, s_, t, p.tol, ortho=ortho, restructured=restr)
    assert dref["converged"]
    assert abs(rep["outer_iters"] - dref["outer_iters"]) <= max(1, round(0.05 * dref["outer_iters"]))
    assert rel(host(rep["x"]), dref["x"]) <= 1e-6


def test_pre_restructured_argument_errors(eks, torch_cuda):
    A = ei.poisson2d(16)
    S = eks.Solver(A)
    b = dev(torch_cuda, ei.uniform_pm1(3, A.n))
    for kw, method in [(dict(restructured=True), "msdo-cg"), (dict(restructured=True), "ca-sre-cg"),
                       (dict(ortho="pre-cholqr"), "ca-sre-cg")]:
        with pytest.raises(eks.EksError) as e:
            S.solve(b, method, 2, 4, 1e-8, **kw)
        assert e.value.status == 1
    S.close()


# ------------------------------------------------------------------ §8(f) row 2: split-preconditioned (Alg 8-10)
@pytest.mark.parametrize("method,s_,t,nd", [("sre-cg", 1, 1, 64), ("sre-cg", 3, 4, 64), ("sre-cg2", 2, 8, 64),
                                            ("msdo-cg", 2, 4, 64), ("sre-cg", 3, 16, 64), ("sre-cg", 2, 32, 32),
                                            ("msdo-cg", 3, 2, 16), ("sre-cg", 2, 64, 64)])
def test_preconditioned_end_to_end(eks, torch_cuda, oracle_lib, method, s_, t, nd):
    """Block-Jacobi IC(0) split-preconditioned s-step methods (reading R32) on cfg1: counts within
    5 %, x within 1e-6 of the oracle (mirror mode), a 2-iteration prefix within 1e-9, and fewer
    outer iterations than unpreconditioned."""
    p = ei.cfg1()
    st, L = oracle_lib.ic0(p.A, nd)
    assert st == 0
    S = eks.Solver(p.A)
    S.setup_precond(nd)
    rep = S.solve(dev(torch_cuda, p.b), method, s_, t, p.tol, precond=True)
    pre = S.solve(dev(torch_cuda, p.b), method, s_, t, 0.0, max_outer=3, precond=True)
    plain = S.solve(dev(torch_cuda, p.b), method, s_, t, p.tol)
    S.close()
    ref = oracle_lib.solve(p.A, p.b, method, s_, t, p.tol, mode=oracle_lib.MODE_MIRROR, L=L)
    refp = oracle_lib.solve(p.A, p.b, method, s_, t, 0.0, kmax=3, mode=oracle_lib.MODE_MIRROR, L=L)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    assert rep["true_relres"] <= 1.5e-8
    assert pre["outer_iters"] == refp["outer_iters"] == 2
    assert rel(host(pre["x"]), refp["x"]) <= 1e-9
    assert rep["outer_iters"] < plain["outer_iters"]
    # and against the oracle's DEFINITION mode (M⁻¹A·W with explicit SpMMs, Qᵀ(A·Z), r −= A·u)
    dref = oracle_lib.solve(p.A, p.b, method, s_, t, p.tol, L=L)
    assert dref["converged"]
    assert abs(rep["outer_iters"] - dref["outer_iters"]) <= max(1, round(0.05 * dref["outer_iters"]))
    assert rel(host(rep["x"]), dref["x"]) <= 1e-6


@pytest.mark.parametrize("method,arnoldi,s_,t", [("ca-sre-cg", 7, 3, 4), ("ca-sre-cg2", 5, 2, 8),
                                                 ("ca-msdo-cg", 7, 3, 4), ("ca-sre-cg", 7, 2, 16)])
def test_preconditioned_ca_end_to_end(eks, torch_cuda, oracle_lib, method, arnoldi, s_, t):
    """CA variants with the block-Jacobi IC(0) split preconditioner (seed M⁻¹[T(r)], powers
    M⁻¹A·W) on Poisson2D 48²: counts within 5 %, x within 1e-6 of the oracle."""
    A = ei.poisson2d(48)
    b = ei.uniform_pm1(1805, A.n)
    st, L = oracle_lib.ic0(A, 16)
    S = eks.Solver(A)
    S.setup_precond(16)
    rep = S.solve(dev(torch_cuda, b), method, s_, t, 1e-8, arnoldi=arnoldi, precond=True)
    S.close()
    ref = oracle_lib.solve_ca(A, b, method[3:], arnoldi=arnoldi, s=s_, t=t, tol=1e-8, L=L)
    assert rep["converged"] and ref["converged"], (rep["status"], ref["status"])
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    assert rep["true_relres"] <= 2e-8


@pytest.mark.parametrize("method,s_,t,nd", [("sre-cg", 2, 4, 8), ("msdo-cg", 2, 8, 8), ("ca-sre-cg2", 2, 4, 8)])
def test_complete_cholesky_preconditioner(eks, torch_cuda, oracle_lib, method, s_, t, nd):
    """Block Jacobi with the complete Cholesky of each block (Table 6; envelope factor built on the
    host, sweeps through the general level-scheduled kernel): parity with the oracle on cfg1."""
    p = ei.cfg1()
    st, L = oracle_lib.ic0(p.A, nd, kind="chol")
    S = eks.Solver(p.A)
    S.setup_precond(nd, kind="chol")
    kw = dict(arnoldi=7) if method.startswith("ca-") else {}
    rep = S.solve(dev(torch_cuda, p.b), method, s_, t, p.tol, precond=True, **kw)
    S.close()
    if method.startswith("ca-"):
        ref = oracle_lib.solve_ca(p.A, p.b, method[3:], arnoldi=7, s=s_, t=t, tol=p.tol, L=L)
    else:
        ref = oracle_lib.solve(p.A, p.b, method, s_, t, p.tol, mode=oracle_lib.MODE_MIRROR, L=L)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6


@pytest.mark.parametrize("s_,t,N", [(3, 16, 64), (2, 4, 64), (4, 8, 48)])
def test_graph_replay_bitwise(eks, torch_cuda, s_, t, N):
    """eks_options.use_graph: steady-state SRE-CG outer iterations replayed from CUDA graphs give
    bitwise the plain path's x, counts and residual history (period 2 for 3 | s, else 6)."""
    A = ei.poisson2d(N)
    b = dev(torch_cuda, ei.uniform_pm1(77, A.n))
    S = eks.Solver(A)
    a = S.solve(b, "sre-cg", s_, t, 1e-10)
    g = S.solve(b, "sre-cg", s_, t, 1e-10, use_graph=True)
    S.close()
    assert a["converged"] and g["converged"] and a["outer_iters"] == g["outer_iters"] > 8
    assert torch_cuda.equal(a["x"], g["x"])
    assert a["gpu_launches"] == g["gpu_launches"]


@pytest.mark.parametrize("s_,t,N", [(3, 16, 64), (2, 4, 64), (4, 8, 48), (1, 16, 48)])
def test_device_loop_bitwise(eks, torch_cuda, s_, t, N):
    """use_graph = 2 ("while ρ > ε ρ0 and k < k_max" on the device): after the
    phases are captured the rest of the solve is ONE graph launch (while node → switch over the
    phase graphs → k_loop_check).  Bitwise the plain path's x, counts and ρ history; the graph ran
    (one k_loop_check launch per device-loop iteration on top of the plain path's launches)."""
    A = ei.poisson2d(N)
    b = dev(torch_cuda, ei.uniform_pm1(77, A.n))
    S = eks.Solver(A)
    a = S.solve(b, "sre-cg", s_, t, 1e-10)
    g = S.solve(b, "sre-cg", s_, t, 1e-10, use_graph=2)
    S.close()
    assert a["converged"] and g["converged"] and a["outer_iters"] == g["outer_iters"] > 12
    assert torch_cuda.equal(a["x"], g["x"])
    assert np.array_equal(a["hist"], g["hist"])
    period = 2 if s_ % 3 == 0 else 6
    ndev = g["gpu_launches"] - a["gpu_launches"]  # k_loop_check launches = device-loop iterations
    assert 0 < ndev <= a["outer_iters"] - 2 - period


@pytest.mark.parametrize("tol,max_outer", [(0.0, 40), (1e-10, 14)])
def test_device_loop_stop_reasons(eks, torch_cuda, tol, max_outer):
    """The device loop stops where the host loop stops: k_max (MAXITER), or, driven past
    convergence with tol = 0 on a 64-row problem, the same breakdown block / non-finite ρ.
    Status, counts, breakdown block, x and ρ history identical to the plain path."""
    A = ei.poisson2d(8 if tol == 0.0 else 64)
    b = dev(torch_cuda, ei.uniform_pm1(5, A.n))
    S = eks.Solver(A)
    out = []
    for ug in (0, 2):
        x = torch_cuda.zeros_like(b)
        st, rep = eks.eks_solve_ex(S.ctx, "sre-cg", 2, 4, tol, b, x, max_outer=max_outer, raise_on=(),
                                   use_graph=ug)
        out.append((st, rep, x))
    S.close()
    (sa, ra, xa), (sg, rg, xg) = out
    assert sa == sg and sa != 0
    assert ra["outer_iters"] == rg["outer_iters"] and ra["breakdown_block"] == rg["breakdown_block"]
    assert torch_cuda.equal(xa, xg)
    assert np.array_equal(ra["hist"], rg["hist"], equal_nan=True)


@pytest.mark.parametrize("s_,t", [(1, 4), (1, 16), (2, 8)])
def test_graph_replay_fresh_solver(eks, torch_cuda, s_, t):
    """use_graph on a FRESH context (nothing preallocated by an earlier plain solve): every ring
    slot and partial buffer is allocated before the first capture, so s = 1 (ring slot 2 first used
    at k = 3) captures and replays; bitwise equal to the plain path on a second fresh context."""
    A = ei.poisson2d(48)
    b = dev(torch_cuda, ei.uniform_pm1(78, A.n))
    S1 = eks.Solver(A)
    g = S1.solve(b, "sre-cg", s_, t, 1e-10, use_graph=True)
    S1.close()
    S2 = eks.Solver(A)
    a = S2.solve(b, "sre-cg", s_, t, 1e-10)
    S2.close()
    assert g["status"] == 0 and g["converged"] and g["outer_iters"] == a["outer_iters"] > 6
    assert torch_cuda.equal(a["x"], g["x"])


def test_trsv_ring_slot_chain(eks, torch_cuda, oracle_lib):
    """a 9-row preconditioner domain whose rows 3, 7, 8 are isolated and whose edges
    (1,0),(2,1),(4,2),(5,2),(6,5) make the slot chain r, r+W, r+2W non-monotone in level for rows
    without readers.  The ring width check now covers every row, so M⁻¹ is deterministic and equal
    to the oracle's L⁻ᵗL⁻¹ (repeat solves bitwise identical, x = oracle mirror within 1e-12)."""
    n = 9
    D = 4.0 * np.eye(n)
    for i, j in [(1, 0), (2, 1), (4, 2), (5, 2), (6, 5)]:
        D[i, j] = D[j, i] = -1.0
    A = ei.csr_from_dense(D)
    b = ei.uniform_pm1(91, n)
    st, L = oracle_lib.ic0(A, 1)
    assert st == 0
    S = eks.Solver(A)
    S.setup_precond(1)
    xs = [host(S.solve(dev(torch_cuda, b), "sre-cg", 1, 1, 1e-12, precond=True)["x"]) for _ in range(5)]
    S.close()
    assert all(np.array_equal(xs[0], x) for x in xs[1:])
    ref = oracle_lib.solve(A, b, "sre-cg", 1, 1, 1e-12, mode=oracle_lib.MODE_MIRROR, L=L)
    assert rel(xs[0], ref["x"]) <= 1e-12
    assert rel(xs[0], np.linalg.solve(D, b)) <= 1e-10


def test_preconditioner_errors(eks, torch_cuda):
    A = ei.poisson2d(16)
    S = eks.Solver(A)
    b = dev(torch_cuda, ei.uniform_pm1(3, A.n))
    with pytest.raises(eks.EksError) as e:
        S.solve(b, "sre-cg", 2, 4, 1e-8, precond=True)   # no eks_setup_precond yet
    assert e.value.status == 2
    S.setup_precond(8)
    for kw in (dict(t=16), dict(restructured=True)):
        args = dict(method="sre-cg", t=4)
        args.update(kw)
        with pytest.raises(eks.EksError) as e:
            S.solve(b, args.pop("method"), 2, args.pop("t"), 1e-8, precond=True, **args)
        assert e.value.status == 1
    # an indefinite diagonal block: IC(0) breaks down at setup
    D = np.array([[1.0, 2.0], [2.0, 1.0]])
    B = ei.csr_from_dense(D)
    S2 = eks.Solver(B)
    with pytest.raises(eks.EksError) as e:
        S2.setup_precond(1)
    assert e.value.status == 7
    S2.close()
    S.close()


def test_cfg2_full_size_prefix(eks, torch_cuda, oracle_lib):
    # full 512² operator, first 2 outer iterations (tol=0, k_max=3) — x after the same count
    p = ei.cfg2()
    rep, ref = _e2e(eks, torch_cuda, oracle_lib, p.A, p.b, "sre-cg", p.s, p.t, 0.0, kmax=3)
    assert rep["outer_iters"] == ref["outer_iters"] == 2
    assert rel(host(rep["x"]), ref["x"]) <= 1e-10
    assert abs(rep["rho"] - ref["rho"]) <= 1e-8 * ref["rho"]


@pytest.mark.parametrize("method,s_,t", [("sre-cg2", 2, 4), ("msdo-cg", 3, 8), ("msdo-cg", 2, 16), ("sre-cg2", 3, 32)])
def test_store_q_only(eks, torch_cuda, oracle_lib, method, s_, t):
    """Full-basis methods with and without the A·Q cache (eks_options.aq_cache, reading R24): store-Q-only
    (the default) takes C = Qᵀ(A·Z) with explicit SpMMs — the oracle's definition algebra — and holds
    twice the outer iterations in memory.  Both agree with the oracle's definition mode (counts within
    5 %, x within 1e-6; two-iteration prefix within 1e-10) and the planner reports max_outer_fit."""
    p = ei.cfg1()
    S = eks.Solver(p.A)
    b = dev(torch_cuda, p.b)
    off = S.solve(b, method, s_, t, p.tol)                       # auto = store Q only
    on = S.solve(b, method, s_, t, p.tol, aq_cache="on")
    pre_off = S.solve(b, method, s_, t, 0.0, max_outer=3, aq_cache="off")
    S.close()
    ref = oracle_lib.solve(p.A, p.b, method, s_, t, p.tol)
    refp = oracle_lib.solve(p.A, p.b, method, s_, t, 0.0, kmax=3)
    for rep in (off, on):
        assert rep["converged"] and rep["status"] == 0
        assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
        assert rel(host(rep["x"]), ref["x"]) <= 1e-6
        assert rep["max_outer_fit"] > rep["outer_iters"]
    assert off["max_outer_fit"] > 1.5 * on["max_outer_fit"]  # A·W no longer stored per block
    assert pre_off["outer_iters"] == refp["outer_iters"] == 2
    assert rel(host(pre_off["x"]), refp["x"]) <= 1e-10


def test_cfg3_analog_msdo(eks, torch_cuda, oracle_lib):
    p = ei.cfg3(N=16)  # 16³ analog of the 128³ subcube problem, t=32 (a domain = 8 rows... 128 rows), s=4
    rep, ref = _e2e(eks, torch_cuda, oracle_lib, p.A, p.b, "msdo-cg", p.s, p.t, p.tol)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6


def test_cfg4_analog_sre_t64(eks, torch_cuda, oracle_lib):
    p = ei.cfg4(N=16)  # 16³ analog of the 256³ anisotropic problem, t=64, s=2
    rep, ref = _e2e(eks, torch_cuda, oracle_lib, p.A, p.b, "sre-cg", p.s, p.t, p.tol)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6


_ORACLE_ITS = {}


def _oracle_iterations(oracle_lib, p, kmax, key=None):
    """Per-outer-iteration V (n×st), x, r of the oracle's DEFINITION mode (callback of or_solve).
    `key`: the same oracle run serves several tests of one session (the 64³ prefixes take minutes)."""
    if key is not None and (key, kmax) in _ORACLE_ITS:
        return _ORACLE_ITS[(key, kmax)]
    its = {}

    def cb(k, V, alpha, x, r, rho):
        its[k] = dict(V=V, x=x, r=r, rho=rho)
    ref = oracle_lib.solve(p.A, p.b, p.method, p.s, p.t, 0.0, kmax=kmax, callback=cb)
    if key is not None:
        _ORACLE_ITS[(key, kmax)] = (ref, its)
    return ref, its


@pytest.mark.parametrize("cfg", ["cfg4", "cfg3"])
def test_path_size_prefix_vs_definition(eks, torch_cuda, oracle_lib, cfg):
    """64³ analogs of cfg4 (SRE-CG, t=64, s=2, anisotropic z 1e-2, b=1) and cfg3 (MSDO-CG, t=32, s=4,
    κ=1e3 subcubes): n = 262,144 rows, i.e. ≈ 28 TR-tiles per CTA of the DMMA/cp.async sweeps and
    many plane-marching units per CTA at t = 32/64 — the multi-tile paths of the full-size kernels.
    The first two outer iterations (tol = 0) against the oracle's DEFINITION mode (explicit SpMMs
    Qᵀ(A·Z), u = Vα̃, r −= A·u; reading R24/R9 give equality in exact arithmetic): every basis block
    W, x and the recursive r element-wise within 1e-10 (relative to their max-norm)."""
    torch = torch_cuda
    p = ei.cfg4(N=64) if cfg == "cfg4" else ei.cfg3(N=64)
    ref, its = _oracle_iterations(oracle_lib, p, kmax=3, key=cfg + "-64")
    assert ref["outer_iters"] == 2 and sorted(its) == [1, 2]
    n, t, s_ = p.A.n, p.t, p.s
    S = eks.Solver(p.A)
    b = dev(torch, p.b)
    W = torch.empty(n, t, dtype=torch.float64, device="cuda")
    r = torch.empty(n, dtype=torch.float64, device="cuda")

    def close(a, o, tol=1e-10):
        return np.abs(a - o).max() <= tol * np.abs(o).max()
    seen = set()
    for k in (1, 2):
        rep = S.solve(b, p.method, s_, t, 0.0, max_outer=k + 1)
        assert rep["outer_iters"] == k
        assert close(host(rep["x"]), its[k]["x"]), (cfg, k, "x")
        eks.eks_k_last_residual(S.ctx, r)
        assert close(host(r), its[k]["r"]), (cfg, k, "r")
        assert abs(rep["rho"] - its[k]["rho"]) <= 1e-10 * its[k]["rho"]
        for kk in range(1, k + 1):
            for i in range(s_):
                j = (kk - 1) * s_ + i
                try:
                    eks.eks_k_last_basis(S.ctx, j, W)
                except eks.EksError:
                    continue  # SRE-CG ring: block overwritten (it was compared at the earlier k)
                Vo = its[kk]["V"][:, i * t:(i + 1) * t]
                assert close(host(W), Vo), (cfg, k, j)
                seen.add(j)
    S.close()
    assert seen == set(range(2 * s_))


@pytest.mark.parametrize("t,nblocks", [(8, 4), (16, 8), (32, 6)])
def test_basis_sweep_parity(eks, torch_cuda, oracle_lib, t, nblocks):
    torch = torch_cuda
    A = ei.stencil_csr(12, 12, 12, ndim=3)
    X0 = ei.cfg5_start_block(A.n, t)
    S = eks.Solver(A)
    W = torch.empty(A.n, t, dtype=torch.float64, device="cuda")
    rep = eks.eks_basis_sweep(S.ctx, t, nblocks, dev(torch, X0), W)
    st, Wo = oracle_lib.basis_sweep(A, X0, nblocks)
    assert st == 0 and rep["outer_iters"] == nblocks
    assert rel(host(W), Wo) <= 1e-9
    Wh = host(W)
    assert np.abs(oracle_lib.xty(Wh, oracle_lib.spmm(A, Wh)) - np.eye(t)).max() <= 1e-10
    S.close()


# ------------------------------------------------------------------ degenerate / error cases
def test_zero_rhs_and_errors(eks, torch_cuda):
    torch = torch_cuda
    A = ei.poisson2d(10)
    S = eks.Solver(A)
    rep = S.solve(torch.zeros(A.n, dtype=torch.float64, device="cuda"), "sre-cg", 2, 4, 1e-8)
    assert rep["status"] == 0 and rep["outer_iters"] == 0 and rep["converged"]
    with pytest.raises(eks.EksError) as e:
        S.solve(torch.ones(A.n, dtype=torch.float64, device="cuda"), "sre-cg", 2, 3, 1e-8)  # t=3
    assert e.value.status == 1
    with pytest.raises(eks.EksError):
        S.solve(torch.ones(A.n, dtype=torch.float64, device="cuda"), "sre-cg", 0, 4, 1e-8)  # s=0
    S.close()


def test_bad_matrix_rejected(eks, torch_cuda):
    A = ei.poisson2d(4)
    ctx = eks.eks_create()
    col = A.col.copy()
    col[0], col[1] = col[1], col[0]  # unsorted row
    with pytest.raises(eks.EksError) as e:
        eks.eks_setup_csr(ctx, A.n, 0, A.n, A.row_ptr, col, A.val)
    assert e.value.status == 3
    val = A.val.copy()
    val[0] = -1.0  # negative diagonal
    with pytest.raises(eks.EksError) as e:
        eks.eks_setup_csr(ctx, A.n, 0, A.n, A.row_ptr, A.col, val)
    assert e.value.status == 3
    eks.eks_destroy(ctx)


def test_msdo_breakdown_keeps_x0(eks, torch_cuda, oracle_lib):
    torch = torch_cuda
    A = ei.poisson2d(8)
    b = ei.uniform_pm1(2, A.n)
    b[: A.n // 4] = 0.0
    S = eks.Solver(A)
    rep = S.solve(dev(torch, b), "msdo-cg", 2, 4, 1e-8)
    assert rep["status"] == eks.EKS_ERR_BREAKDOWN and rep["outer_iters"] == 0
    assert rep["breakdown_block"] == 0 and float(rep["x"].abs().max()) == 0.0
    ref = oracle_lib.solve(A, b, "msdo-cg", 2, 4, 1e-8)
    assert ref["status"] == oracle_lib.BREAKDOWN
    S.close()


def test_maxiter_and_determinism_and_host_pointers(eks, torch_cuda):
    torch = torch_cuda
    p = ei.cfg1()
    S = eks.Solver(p.A)
    r1 = S.solve(dev(torch, p.b), p.method, p.s, p.t, p.tol, max_outer=5)
    assert r1["status"] == eks.EKS_ERR_MAXITER and r1["outer_iters"] == 4 and not r1["converged"]
    a = S.solve(dev(torch, p.b), p.method, p.s, p.t, p.tol)
    b = S.solve(dev(torch, p.b), p.method, p.s, p.t, p.tol)
    c = S.solve(p.b.copy(), p.method, p.s, p.t, p.tol)  # host pointers (EKS_MEM_HOST)
    assert torch.equal(a["x"], b["x"])                       # bitwise run-to-run
    assert np.array_equal(host(a["x"]), c["x"])
    assert np.array_equal(a["hist"], c["hist"])
    S.close()


# ------------------------------------------------------------------ BASELINE full sizes
def _full_operator(cfg):
    return {"cfg3": lambda: ei.cfg3().A, "cfg4": lambda: ei.cfg4().A, "cfg5": lambda: ei.cfg5_operator()}[cfg]()


def _sub_csr(A, rows):
    """Rows `rows` of A with their columns renumbered into the set of columns they use."""
    starts, ends = A.row_ptr[rows], A.row_ptr[rows + 1]
    idx = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)])
    ucols, inv = np.unique(A.col[idx], return_inverse=True)
    rp = np.concatenate([[0], np.cumsum(ends - starts)]).astype(np.int64)
    return ei.Csr(len(rows), rp, inv.astype(np.int32), A.val[idx].copy()), ucols


@pytest.mark.parametrize("cfg,t", [("cfg3", 32), ("cfg4", 64), ("cfg5", 16)])
def test_full_size_spmm_gram_sampled(eks, torch_cuda, oracle_lib, cfg, t):
    """The SpMM-block kernel eks_solve launches, at the BASELINE operator sizes: sampled rows of
    Y = A·X bitwise against the oracle's row products (SpMM order, R20), the Gram XᵀY and Xᵀv
    against a cuBLAS fp64 reference within 1e-12."""
    torch = torch_cuda
    A = _full_operator(cfg)
    S = eks.Solver(A)
    X = ei.uniform_pm1_torch(77, A.n * t, "cuda").view(A.n, t)
    v = ei.uniform_pm1_torch(78, A.n, "cuda")
    Y = torch.empty_like(X)
    G = torch.empty(t, t, dtype=torch.float64, device="cuda")
    g = torch.empty(t, dtype=torch.float64, device="cuda")
    eks.eks_k_spmm(S.ctx, t, X, Y, G, v, g)
    rng = np.random.default_rng(11)
    edges = [0, 1, 15, 16, 63, 64, A.n // 2, A.n - 65, A.n - 64, A.n - 2, A.n - 1]
    rows = np.unique(np.concatenate([rng.integers(0, A.n, 3000), edges])).astype(np.int64)
    sub, ucols = _sub_csr(A, rows)
    Xs = host(X[torch.from_numpy(ucols).cuda()])
    Yo = oracle_lib.spmm(sub, Xs)[: len(rows)]
    assert np.array_equal(host(Y[torch.from_numpy(rows).cuda()]), Yo)
    if cfg == "cfg3":
        # cfg3 fits the oracle whole (2.1M × 32): every row of Y bitwise, Gram and Xᵀv vs or_xty
        Xh, vh = host(X), host(v)
        Yf = oracle_lib.spmm(A, Xh)
        assert np.array_equal(host(Y), Yf)
        assert rel(host(G), oracle_lib.xty(Xh, Yf)) <= 1e-12
        assert rel(host(g), oracle_lib.xty(Xh, vh[:, None])[:, 0]) <= 1e-12
    else:
        # cfg4 / cfg5 (8.6 / 7.2 GB blocks): too large for the single-thread oracle's Gram; a cuBLAS
        # fp64 XᵀY stands in (sampled rows above are the oracle's)
        assert rel(host(G), host(X.T @ Y)) <= 1e-12
        assert rel(host(g), host(X.T @ v)) <= 1e-12
    S.close()


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4"])
def test_full_size_solve_prefix_properties(eks, torch_cuda, cfg):
    """First outer iterations of the BASELINE solves at full size (the oracle cannot run them):
    the library's true residual matches a cuSPARSE fp64 b − A·x, the recursive residual tracks
    it, and φ(x) = ½xᵀAx − bᵀx decreases (the A-norm error is minimised over a growing space)."""
    torch = torch_cuda
    p = ei.cfg3() if cfg == "cfg3" else ei.cfg4()
    A = p.A
    At = torch.sparse_csr_tensor(torch.from_numpy(A.row_ptr), torch.from_numpy(A.col.astype(np.int64)),
                                 torch.from_numpy(A.val), size=(A.n, A.n)).cuda()
    b = dev(torch, p.b)
    S = eks.Solver(A)
    phis = [0.0]
    for k in (1, 2):
        rep = S.solve(b, p.method, p.s, p.t, 0.0, max_outer=k + 1)
        assert rep["outer_iters"] == k
        x = rep["x"]
        Ax = (At @ x.unsqueeze(1)).squeeze(1)
        r = b - Ax
        relres = float(r.norm() / b.norm())
        assert abs(relres - rep["true_relres"]) <= 1e-10 * max(1.0, relres)
        assert abs(float(r.norm()) - rep["rho"]) <= 1e-9 * float(b.norm())
        phis.append(float(0.5 * x.dot(Ax) - b.dot(x)))
    assert phis[2] < phis[1] < phis[0]
    S.close()


# ------------------------------------------------------------------ paper Table 2-4 protocol on the GPU
@pytest.mark.parametrize("key,method", [("sre_cg_t2", "sre-cg"), ("sre_cg2_t2", "sre-cg2"),
                                        ("msdo_cg_t2", "msdo-cg"), ("sre_cg_t4", "sre-cg")])
def test_paper_poisson2d_rows_gpu(eks, torch_cuda, oracle_lib, key, method):
    """Poisson2D (gallery('poisson',100)), b = A·x_rand, tol 1e-6: the GPU's outer-iteration
    counts equal the oracle's and lie within the paper's printed cells (Tables 2-4, ±15 %: the
    partition is contiguous, not Metis)."""
    import json
    import os
    paper = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_poisson2d.json")))
    A = ei.poisson2d(100)
    b = ei.paper_poisson_rhs(A)
    t = 4 if key.endswith("t4") else 2
    S = eks.Solver(A)
    for s_, want in zip(paper[key]["s"], paper[key]["k"]):
        rep = S.solve(dev(torch_cuda, b), method, s_, t, paper["tol"])
        ref = oracle_lib.solve(A, b, method, s=s_, t=t, tol=paper["tol"])
        assert rep["converged"] and ref["converged"]
        assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"])), (s_,)
        assert abs(rep["outer_iters"] - want) <= paper["tolerance_enlarged"] * want, (key, s_, rep["outer_iters"], want)
    S.close()


@pytest.mark.parametrize("method,t", [("sre-cg", 8), ("sre-cg", 16), ("sre-cg", 32), ("sre-cg2", 8),
                                      ("msdo-cg", 8)])
def test_paper_poisson2d_large_t_gpu(eks, torch_cuda, oracle_lib, method, t):
    """The Table 2-4 protocol at the partition counts the DMMA/TMA kernels serve (t ≥ 8), s = 3:
    GPU and oracle counts agree and x agrees to 1e-6; for SRE-CG k(s=3) = ⌈k(s=1)/3⌉.
    (Larger t and full-basis t ≥ 16 are left out: the single-thread oracle's cost grows with k·s·t.)"""
    A = ei.poisson2d(100)
    b = ei.paper_poisson_rhs(A)
    S = eks.Solver(A)
    rep = S.solve(dev(torch_cuda, b), method, 3, t, 1e-6)
    ref = oracle_lib.solve(A, b, method, s=3, t=t, tol=1e-6)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    if method == "sre-cg":
        r1 = S.solve(dev(torch_cuda, b), method, 1, t, 1e-6)
        assert rep["outer_iters"] == math.ceil(r1["outer_iters"] / 3)
    S.close()


# ------------------------------------------------------------------ §8(f) row 1: communication-avoiding variants
@pytest.mark.parametrize("method,arnoldi,s_,t", [("ca-sre-cg", 7, 3, 4), ("ca-sre-cg", 5, 2, 4), ("ca-sre-cg2", 7, 2, 8),
                                                 ("ca-msdo-cg", 7, 3, 4), ("ca-msdo-cg", 5, 2, 8),
                                                 ("ca-sre-cg", 7, 3, 16), ("ca-sre-cg", 7, 2, 32),
                                                 ("ca-sre-cg", 7, 3, 64)])  # st = 192: global-memory Cholesky
def test_ca_end_to_end(eks, torch_cuda, oracle_lib, method, arnoldi, s_, t):
    """CA SRE-CG / CA SRE-CG2 / CA MSDO-CG (Alg 5 or 7, one st-column A-CholQR per outer iteration)
    on the well-conditioned Poisson2D 48² (the paper's CA regime): GPU and oracle
    reach 1e-8 with counts within max(5 %, 1) and x within 1e-6."""
    A = ei.poisson2d(48)
    b = ei.uniform_pm1(1805, A.n)
    base = method[3:]
    S = eks.Solver(A)
    rep = S.solve(dev(torch_cuda, b), method, s_, t, 1e-8, arnoldi=arnoldi)
    S.close()
    ref = oracle_lib.solve_ca(A, b, base, arnoldi=arnoldi, s=s_, t=t, tol=1e-8)
    assert rep["converged"] and ref["converged"], (rep["status"], ref["status"])
    assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"]))
    assert rel(host(rep["x"]), ref["x"]) <= 1e-6
    assert rep["true_relres"] <= 2e-8


def test_poisson2d_tables_sweep_gpu(eks, torch_cuda):
    """§8(f) item 4: every Poisson2D cell of Tables 2-4 through libeks (tools/poisson_tables.py):
    all converge; t = 2 (partition-comparable, reading R1) within 15 % of the printed cells; the
    paper's Poisson2D relations hold on our counts (restructured and s-step = ceil(k/s), P:482-484;
    CA SRE-CG/SRE-CG2 with Alg 7 = s-step for s ≤ 4, Tables 2/3)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("poisson_tables", os.path.join(ROOT, "tools", "poisson_tables.py"))
    pt = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(pt)
    cells, _ = pt.sweep(eks, torch_cuda)
    assert all(c["converged"] for c in cells.values()), [k for k, c in cells.items() if not c["converged"]]
    for k, c in cells.items():
        key, t, s = k.split("|")
        if t == "2" and not key.startswith("pc-"):  # Table 5: 64 Metis preconditioner domains, context only
            want = [c["paper"]]
            if key == "msdo-cg/ca7":  # reading R28: the literal Alg 7 seed gives the s-step count
                want.append(cells[f"msdo-cg/s-step|{t}|{s}"]["paper"])
            assert min(abs(c["k"] - w) - 0.15 * w for w in want) <= 0, (k, c)
    assert pt.relations(cells) == []


def test_ca_ill_conditioned_agrees_with_oracle(eks, torch_cuda, oracle_lib):
    """On the κ = 1e3 band problem (cfg2 recipe at 64²) CA SRE-CG converges for s = 2 and its
    monomial basis breaks down for s = 3 — on both sides (the paper's instability)."""
    p = ei.cfg2(N=64)
    S = eks.Solver(p.A)
    ok = S.solve(dev(torch_cuda, p.b), "ca-sre-cg", 2, 4, 1e-8, arnoldi=5)
    bad = S.solve(dev(torch_cuda, p.b), "ca-sre-cg", 3, 4, 1e-8)
    S.close()
    ref_ok = oracle_lib.solve_ca(p.A, p.b, "sre-cg", arnoldi=5, s=2, t=4, tol=1e-8)
    ref_bad = oracle_lib.solve_ca(p.A, p.b, "sre-cg", arnoldi=7, s=3, t=4, tol=1e-8)
    assert ok["converged"] and ref_ok["converged"]
    assert abs(ok["outer_iters"] - ref_ok["outer_iters"]) <= max(1, round(0.05 * ref_ok["outer_iters"]))
    assert bad["status"] == eks.EKS_ERR_BREAKDOWN and ref_bad["status"] == oracle_lib.BREAKDOWN
    assert bad["outer_iters"] == ref_bad["outer_iters"]


def test_ca_breakdown_reported(eks, torch_cuda, oracle_lib):
    A = ei.poisson2d(64)
    b = ei.paper_poisson_rhs(A)
    S = eks.Solver(A)
    rep = S.solve(dev(torch_cuda, b), "ca-sre-cg", 10, 2, 1e-6)
    S.close()
    assert rep["status"] == eks.EKS_ERR_BREAKDOWN and rep["outer_iters"] == 0
    assert float(rep["x"].abs().max()) == 0.0


# ------------------------------------------------------------------ (a3) one-synch CGS2 (reading R36)
@pytest.mark.parametrize("method,s_,t,N,aq", [("sre-cg", 3, 16, 64, "auto"), ("sre-cg", 2, 4, 48, "auto"),
                                              ("sre-cg", 1, 1, 32, "auto"), ("sre-cg", 2, 32, 48, "auto"),
                                              ("sre-cg2", 2, 8, 48, "on"), ("msdo-cg", 4, 4, 32, "auto"),
                                              ("msdo-cg", 2, 16, 48, "on")])
def test_onesynch_end_to_end(eks, torch_cuda, oracle_lib, method, s_, t, N, aq):
    """eks_options.onesynch (SpMM of Z1, one stacked reduction of [C2 | B1 | g1], B = B1 − C2ᵀC2,
    A·Z2 = A·Z1 − (AQ)C2) against the oracle's MODE_ONESYNCH and its DEFINITION mode on κ = 1e3
    bands: counts within max(5 %, 1), x within 1e-6 after convergence; the first two outer
    iterations (tol = 0) within 1e-10 of both (equal in exact arithmetic)."""
    A = ei.stencil_csr(N, N, ndim=2, kappa=ei.bands_kappa(N, band=4, hi=1e3))
    bh = ei.uniform_pm1(1806, A.n)
    S = eks.Solver(A)
    b = dev(torch_cuda, bh)
    rep = S.solve(b, method, s_, t, 1e-8, onesynch=True, aq_cache=aq)
    pre = S.solve(b, method, s_, t, 0.0, max_outer=3, onesynch=True, aq_cache=aq)
    S.close()
    for mode in (oracle_lib.MODE_ONESYNCH, oracle_lib.MODE_DEFINITION):
        ref = oracle_lib.solve(A, bh, method, s_, t, 1e-8, mode=mode)
        refp = oracle_lib.solve(A, bh, method, s_, t, 0.0, kmax=3, mode=mode)
        assert rep["status"] == 0 and rep["converged"] and ref["converged"]
        assert abs(rep["outer_iters"] - ref["outer_iters"]) <= max(1, round(0.05 * ref["outer_iters"])), \
            (mode, rep["outer_iters"], ref["outer_iters"])
        assert rel(host(rep["x"]), ref["x"]) <= 1e-6, mode
        assert pre["outer_iters"] == refp["outer_iters"] == 2
        assert rel(host(pre["x"]), refp["x"]) <= 1e-10, mode
    assert rep["true_relres"] <= 2e-8


def test_onesynch_graph_replay_bitwise_and_errors(eks, torch_cuda):
    """One-synch under CUDA-graph replay: bitwise the plain one-synch path; the options it does not
    combine with are rejected (EKS_ERR_INVALID_ARG)."""
    A = ei.poisson2d(64)
    b = dev(torch_cuda, ei.uniform_pm1(79, A.n))
    S = eks.Solver(A)
    a = S.solve(b, "sre-cg", 3, 16, 1e-10, onesynch=True)
    g = S.solve(b, "sre-cg", 3, 16, 1e-10, onesynch=True, use_graph=True)
    assert a["converged"] and g["converged"] and a["outer_iters"] == g["outer_iters"] > 8
    assert torch_cuda.equal(a["x"], g["x"])
    for method, kw in [("ca-sre-cg", {}), ("sre-cg", dict(ortho="pre-cholqr")), ("sre-cg", dict(restructured=True)),
                       ("msdo-cg", dict(aq_cache="off"))]:
        with pytest.raises(eks.EksError) as e:
            S.solve(b, method, 2, 4, 1e-8, onesynch=True, **kw)
        assert e.value.status == 1
    S.close()


@pytest.mark.parametrize("cfg", ["cfg4", "cfg3"])
def test_onesynch_path_size_prefix(eks, torch_cuda, oracle_lib, cfg):
    """One-synch at the 64³ analogs of cfg4 (SRE-CG t=64 s=2) and cfg3 (MSDO-CG t=32 s=4, A·Q cached):
    after two outer iterations x and r agree with the oracle's DEFINITION mode within 1e-10 of their
    max-norm (multi-tile sweeps and plane-marching units at t = 32/64)."""
    torch = torch_cuda
    p = ei.cfg4(N=64) if cfg == "cfg4" else ei.cfg3(N=64)
    ref, its = _oracle_iterations(oracle_lib, p, kmax=3, key=cfg + "-64")
    S = eks.Solver(p.A)
    b = dev(torch, p.b)
    r = torch.empty(p.A.n, dtype=torch.float64, device="cuda")
    rep = S.solve(b, p.method, p.s, p.t, 0.0, max_outer=3, onesynch=True, aq_cache="on")
    assert rep["outer_iters"] == 2
    eks.eks_k_last_residual(S.ctx, r)
    S.close()
    for got, exp in ((host(rep["x"]), its[2]["x"]), (host(r), its[2]["r"])):
        assert np.abs(got - exp).max() <= 1e-10 * np.abs(exp).max()


@pytest.mark.parametrize("t", [8, 16, 32])
def test_onesynch_basis_sweep(eks, torch_cuda, oracle_lib, t):
    """cfg5's basis sweep with one-synch CGS2: W_last within 1e-9 of the oracle's sweep and
    A-orthonormal to 1e-10."""
    torch = torch_cuda
    A = ei.stencil_csr(12, 12, 12, ndim=3)
    X0 = ei.cfg5_start_block(A.n, t)
    S = eks.Solver(A)
    W = torch.empty(A.n, t, dtype=torch.float64, device="cuda")
    rep = eks.eks_basis_sweep(S.ctx, t, 8, dev(torch, X0), W, onesynch=True)
    S.close()
    st, Wo = oracle_lib.basis_sweep(A, X0, 8)
    assert st == 0 and rep["outer_iters"] == 8
    assert rel(host(W), Wo) <= 1e-9
    Wh = host(W)
    assert np.abs(oracle_lib.xty(Wh, oracle_lib.spmm(A, Wh)) - np.eye(t)).max() <= 1e-10


# ------------------------------------------------------------------ §8(f)1 at N > 1: matrix-powers kernel
@pytest.mark.parametrize("t,s,opname,z0,z1", [
    (8, 3, "aniso24", 8, 16), (16, 4, "aniso24", 0, 6), (16, 4, "aniso24", 18, 24), (32, 3, "aniso24", 1, 23),
    (64, 2, "aniso24", 12, 13), (16, 5, "aniso24", 2, 5), (16, 3, "bands96", 30, 60), (8, 6, "bands96", 3, 96)])
def test_matrix_powers_virtual_slab_bitwise(eks, torch_cuda, oracle_lib, t, s, opname, z0, z1):
    """Depth-(s−1) ghost-zone matrix powers (reading R37): planes [z0, z1) as a rank's slab —
    the slab rows of A·X, …, A^(s−1)·X from the shrinking plane-range launches equal the oracle's global
    powers bitwise (interior slabs, slabs at / near the grid boundary, a one-plane slab)."""
    torch = torch_cuda
    A = {"aniso24": lambda: ei.stencil_csr(24, 24, 24, ndim=3, scale=(1.0, 1.0, 1e-2)),
         "bands96": lambda: ei.stencil_csr(96, 96, ndim=2, kappa=ei.bands_kappa(96, band=8))}[opname]()
    plane = 24 * 24 if opname == "aniso24" else 96
    S = eks.Solver(A)
    X = ei.uniform_pm1(41, A.n * t).reshape(A.n, t)
    rows = (z1 - z0) * plane
    V = torch.full((s - 1, rows, t), float("nan"), dtype=torch.float64, device="cuda")
    eks.eks_k_matrix_powers(S.ctx, t, s, z0, z1, dev(torch, X), V)
    P = X
    for i in range(s - 1):
        P = oracle_lib.spmm(A, P)
        assert np.array_equal(host(V[i]), P[z0 * plane:z1 * plane]), (i, t, s)
    S.close()


def test_matrix_powers_full_size_sampled(eks, torch_cuda, oracle_lib):
    """The same at a size whose launches span many units per CTA (128³, t = 16, s = 4, an interior slab of
    32 planes): the slab rows of the powers equal repeated global eks_k_spmm products bitwise (those are
    bitwise the oracle's, test_spmm_bitwise_and_gram / test_full_size_spmm_gram_sampled)."""
    torch = torch_cuda
    N, t, s, z0, z1 = 128, 16, 4, 48, 80
    A = ei.stencil_csr(N, N, N, ndim=3, scale=(1.0, 1.0, 1e-2))
    S = eks.Solver(A)
    X = dev(torch, ei.uniform_pm1(43, A.n * t).reshape(A.n, t))
    rows = (z1 - z0) * N * N
    V = torch.empty(s - 1, rows, t, dtype=torch.float64, device="cuda")
    eks.eks_k_matrix_powers(S.ctx, t, s, z0, z1, X, V)
    P = X
    for i in range(s - 1):
        Y = torch.empty_like(P)
        eks.eks_k_spmm(S.ctx, t, P, Y)
        P = Y
        assert torch.equal(V[i], P[z0 * N * N:z1 * N * N]), i
    S.close()


_MPK_SCRIPT = r"""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import eks_inputs as ei
import paper_1804_10629_b200 as eks
out = []
for A in (ei.poisson2d(48), ei.stencil_csr(16, 16, 16, ndim=3)):
    b = torch.from_numpy(ei.uniform_pm1(51, A.n)).cuda()
    S = eks.Solver(A)
    for method, s, t, arn in (("ca-sre-cg", 3, 8, 7), ("ca-sre-cg2", 2, 16, 5), ("ca-msdo-cg", 3, 8, 7)):
        try:
            rep = S.solve(b, method, s, t, 1e-8, arnoldi=arn)
            out.append(f"{method} it={rep['outer_iters']} st={rep['status']} "
                       + hashlib.sha256(rep['x'].cpu().numpy().tobytes()).hexdigest())
        except Exception as e:
            out.append(f"{method} raised {getattr(e, 'status', '?')}")
    S.close()
print("|".join(out))
"""


def test_matrix_powers_path_in_ca_solve(eks, torch_cuda):
    """EKS_MPK=force: the CA outer iteration takes the matrix-powers code path (deep-ghost V blocks,
    mpk_powers → mpk_local) on one rank, where it issues the same products without neighbours: x, the
    outer-iteration count and the status of CA SRE-CG / CA SRE-CG2 / CA MSDO-CG solves are bitwise those
    of the default path (the environment switch is read once per process: two subprocesses)."""
    import subprocess
    import sys
    outs = []
    for mode in (None, "force"):
        env = dict(os.environ)
        env.pop("EKS_MPK", None)
        if mode:
            env["EKS_MPK"] = mode
        r = subprocess.run([sys.executable, "-c", _MPK_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs
    parts = outs[0].split("|")
    assert len(parts) == 6 and all(" st=0 " in part for part in parts[:3]), outs[0]  # Poisson2D: converged
