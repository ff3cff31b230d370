"""Pins for the shared input generators (eks_inputs): SplitMix64 reference outputs,
stencil nnz counts from the paper / SPEC, symmetry, closed-form diagonals."""
import json
import os

import numpy as np
import pytest

import eks_inputs as ei

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_splitmix64_reference_outputs():
    g = _gold("spec_examples.json")["splitmix64_seed0"]
    want = [int(z, 16) for z in g["z"]]
    assert [ei.splitmix64_scalar(0, i) for i in range(3)] == want
    assert [int(v) for v in ei.splitmix64(0, 3)] == want


def test_splitmix64_vectorised_matches_scalar_and_offsets():
    z = ei.splitmix64(1806, 1000)
    assert all(int(z[i]) == ei.splitmix64_scalar(1806, i) for i in (0, 1, 17, 999))
    assert np.array_equal(ei.splitmix64(1806, 10, start=5), z[5:15])
    u = ei.uniform_pm1(1806, 100000)
    assert u.min() >= -1.0 and u.max() < 1.0 and abs(u.mean()) < 0.01


@pytest.mark.parametrize("N,n,nnz", _gold("spec_examples.json")["gen_poisson2d"]["cases"])
def test_poisson2d_sizes(N, n, nnz):
    A = ei.poisson2d(N)
    assert A.n == n and A.nnz == nnz


def test_poisson2d_is_gallery_poisson():
    # gallery('poisson',N) = kron(I,T)+kron(T,I), T = tridiag(-1,2,-1)
    N = 5
    T = 2 * np.eye(N) - np.eye(N, k=1) - np.eye(N, k=-1)
    G = np.kron(np.eye(N), T) + np.kron(T, np.eye(N))
    assert np.array_equal(ei.poisson2d(N).to_dense(), G)


def _is_symmetric(A):
    D = A.to_dense()
    return np.array_equal(D, D.T)


def test_config_operators_symmetric_sorted_positive_diag():
    ops = [ei.stencil_csr(12, 12, ndim=2, kappa=ei.bands_kappa(12, band=3)),
           ei.stencil_csr(8, 8, 8, ndim=3, kappa=ei.subcubes_kappa(8, cell=2)),
           ei.stencil_csr(6, 6, 6, ndim=3, scale=(1.0, 1.0, 1e-2))]
    for A in ops:
        assert _is_symmetric(A)
        for i in range(A.n):
            cols = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
            assert np.all(np.diff(cols) > 0)
            assert i in cols
        D = A.to_dense()
        assert np.all(np.diag(D) > 0)
        # weak diagonal dominance with strict dominance on the boundary → SPD
        assert np.all(np.diag(D) >= np.abs(D).sum(1) - np.diag(D) - 1e-12)
        assert np.linalg.eigvalsh(D).min() > 0


def test_nnz_formula_and_configs():
    # nnz = n + 2·d·N^{d-1}(N-1)
    for N, d in ((64, 2), (512, 2), (20, 3)):
        A = ei.stencil_csr(N, N, N, ndim=d) if d == 3 else ei.stencil_csr(N, N, ndim=2)
        assert A.nnz == N ** d + 2 * d * N ** (d - 1) * (N - 1)
    p = ei.cfg1()
    assert (p.A.n, p.A.nnz, p.s, p.t) == (4096, 20224, 2, 4)
    assert 384 ** 3 + 6 * 384 ** 2 * 383 == 395476992
    assert 256 ** 3 + 6 * 256 ** 2 * 255 == 117047296


def test_anisotropic_diag_and_bands():
    A = ei.stencil_csr(5, 5, 5, ndim=3, scale=(1.0, 1.0, 1e-2))
    D = A.to_dense()
    assert np.allclose(np.diag(D), 4.02)
    k = ei.bands_kappa(64)
    assert k[0] == 1.0 and k[32 * 64] == 1e3 and k[64 * 64 - 1] == 1e3


def test_subcubes_fraction_exact():
    k = ei.subcubes_kappa(32)
    assert np.count_nonzero(k == 1e3) == (32 ** 3) // 4
    perm = ei.fisher_yates(1834, 4096)
    assert sorted(perm) == list(range(4096))


def test_cfg5_start_block_unit_columns():
    X = ei.cfg5_start_block(1000, 8)
    assert np.allclose(np.linalg.norm(X, axis=0), 1.0, atol=1e-14)


def test_torch_splitmix_matches_numpy():
    """The device-side generator (used for the cfg5 block in bench.py) draws the same bits."""
    import torch
    for seed, start, count in [(1855, 0, 1000), (1806, 12345, 70001), (0, 0, 17)]:
        a = ei.uniform_pm1(seed, count, start=start)
        b = ei.uniform_pm1_torch(seed, count, "cpu", start=start, chunk=4096).numpy()
        assert np.array_equal(a, b)
    X = ei.cfg5_start_block_torch(500, 8, "cpu").numpy()
    assert np.allclose(X, ei.cfg5_start_block(500, 8), rtol=1e-14, atol=0)
