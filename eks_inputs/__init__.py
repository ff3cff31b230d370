"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no split, no SpMM of a basis, no
orthonormalization, no update).  It only builds the *inputs* of a solve:

* SplitMix64 (Steele, Lea, Flood 2014) counter-based generator, SURVEY §8(d)-G0:
  ``z_i = mix(seed + (i+1)*0x9E3779B97F4A7C15)``, ``u = (z >> 11) * 2^-53``,
  ``uniform[-1,1) = 2u - 1``; draws are taken in ascending row order (row-major
  n×t order for blocks).
* Dirichlet finite-difference stencil operators in CSR (fp64 values, int32
  column indices, int64 row pointers), lexicographic ordering ``idx = x + nx*(y + ny*z)``
  (reading R2), face coefficient = harmonic mean of the two cell
  coefficients times a per-direction scale, a Dirichlet boundary face adds the
  cell's own coefficient to the diagonal (reading R17).  With κ≡1 in 2D this is
  MATLAB's ``gallery('poisson', N)`` used for Poisson2D (§4).
* The five BASELINE.json configurations and the reduced
  analogs used where the single-thread oracle cannot finish the full size.

Stand-ins: the paper's FreeFem++ matrices (Table 1) and the
Metis partitions are not available; these generators replace them
(see DESIGN.md "Input recipe").
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

# Seeds, SURVEY §8(d)-G0.
SEED_B = {1: 1805, 2: 1806, 3: 1807}
SEED_CFG3_CELLS = 1834
SEED_CFG5_BLOCK = 1855


# ----------------------------------------------------------------------------
# SplitMix64
# ----------------------------------------------------------------------------
def splitmix64(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Return draws ``start .. start+count-1`` of SplitMix64 seeded with ``seed`` (uint64)."""
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + i * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def splitmix64_scalar(seed: int, i: int) -> int:
    """Draw number ``i`` (0-based) with plain Python integers — used to pin the vectorised form."""
    z = (seed + (i + 1) * GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def uniform01(seed: int, count: int, start: int = 0) -> np.ndarray:
    z = splitmix64(seed, count, start)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(seed: int, count: int, start: int = 0) -> np.ndarray:
    return 2.0 * uniform01(seed, count, start) - 1.0


def uniform_pm1_torch(seed: int, count: int, device, start: int = 0, chunk: int = 1 << 26):
    """The same SplitMix64 U[-1,1) draws as :func:`uniform_pm1`, generated on a torch device in
    int64 arithmetic (wrapping multiply, logical shifts by masking) — bitwise equal values; used
    where a host-side block would be tens of GB (cfg5)."""
    import torch

    def s64(v):  # uint64 constant → the int64 with the same bits
        v &= MASK64
        return v - (1 << 64) if v >= (1 << 63) else v

    def lsr(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)

    out = torch.empty(count, dtype=torch.float64, device=device)
    for lo in range(0, count, chunk):
        hi = min(count, lo + chunk)
        i = torch.arange(start + lo + 1, start + hi + 1, dtype=torch.int64, device=device)
        z = i * s64(GOLDEN) + s64(seed)
        z = (z ^ lsr(z, 30)) * s64(0xBF58476D1CE4E5B9)
        z = (z ^ lsr(z, 27)) * s64(0x94D049BB133111EB)
        z = z ^ lsr(z, 31)
        out[lo:hi] = lsr(z, 11).to(torch.float64) * (2.0 ** -53) * 2.0 - 1.0
    return out


# ----------------------------------------------------------------------------
# CSR container
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Csr:
    n: int
    row_ptr: np.ndarray  # int64, n+1
    col: np.ndarray      # int32, nnz
    val: np.ndarray      # float64, nnz

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def rows(self, lo: int, hi: int) -> "Csr":
        """Row slab [lo, hi) with GLOBAL column indices and row_ptr rebased to 0."""
        a, b = int(self.row_ptr[lo]), int(self.row_ptr[hi])
        return Csr(hi - lo, (self.row_ptr[lo:hi + 1] - a).astype(np.int64), self.col[a:b], self.val[a:b])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        for i in range(self.n):
            for p in range(self.row_ptr[i], self.row_ptr[i + 1]):
                d[i, self.col[p]] += self.val[p]
        return d


def csr_from_dense(d: np.ndarray) -> Csr:
    n = d.shape[0]
    rp = [0]
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(d[i])[0]
        cols.extend(nz.tolist())
        vals.extend(d[i, nz].tolist())
        rp.append(len(cols))
    return Csr(n, np.asarray(rp, np.int64), np.asarray(cols, np.int32), np.asarray(vals, np.float64))


# ----------------------------------------------------------------------------
# Stencil operators
# ----------------------------------------------------------------------------
def _hm(a, b):
    return 2.0 * a * b / (a + b)


def stencil_csr(nx: int, ny: int, nz: int = 1, ndim: int = 2,
                kappa: Optional[np.ndarray] = None,
                scale=(1.0, 1.0, 1.0), chunk_rows: int = 1 << 22) -> Csr:
    """Dirichlet 5-point (ndim=2) / 7-point (ndim=3) operator on an nx×ny(×nz) cell grid.

    ``kappa``: per-cell coefficient (length nx*ny*nz, lexicographic) or None for κ≡1.
    ``scale``: per-direction multiplier of the face coefficient (x, y, z).
    Column order within a row is ascending: -z, -y, -x, diag, +x, +y, +z.
    """
    if ndim == 2:
        nz = 1
    n = nx * ny * nz
    plane = nx * ny
    dirs = [(-plane, 2, -1), (-nx, 1, -1), (-1, 0, -1), (0, None, 0), (1, 0, 1), (nx, 1, 1), (plane, 2, 1)]
    if ndim == 2:
        dirs = dirs[1:-1]
    # count nonzeros per row
    counts = np.empty(n, np.int64)
    for lo in range(0, n, chunk_rows):
        hi = min(n, lo + chunk_rows)
        idx = np.arange(lo, hi, dtype=np.int64)
        x = idx % nx
        y = (idx // nx) % ny
        z = idx // plane
        c = np.ones(hi - lo, np.int64)
        c += (x > 0).astype(np.int64) + (x < nx - 1) + (y > 0) + (y < ny - 1)
        if ndim == 3:
            c += (z > 0).astype(np.int64) + (z < nz - 1)
        counts[lo:hi] = c
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    for lo in range(0, n, chunk_rows):
        hi = min(n, lo + chunk_rows)
        idx = np.arange(lo, hi, dtype=np.int64)
        coord = [idx % nx, (idx // nx) % ny, idx // plane]
        extent = [nx, ny, nz]
        kp = None if kappa is None else kappa[lo:hi]
        pos = row_ptr[lo:hi].copy()
        diag = np.zeros(hi - lo)
        # first pass: diagonal = sum of all face coefficients (interior + Dirichlet boundary)
        for (off, ax, sgn) in dirs:
            if ax is None:
                continue
            has = coord[ax] > 0 if sgn < 0 else coord[ax] < extent[ax] - 1
            if kp is None:
                face = np.full(hi - lo, float(scale[ax]))
            else:
                nb = np.where(has, idx + off, idx)
                face = scale[ax] * np.where(has, _hm(kp, kappa[nb]), kp)
            diag += face  # boundary face contributes κ_p (reading R17)
        for (off, ax, sgn) in dirs:
            if ax is None:
                col[pos] = idx.astype(np.int32)
                val[pos] = diag
                pos += 1
                continue
            has = coord[ax] > 0 if sgn < 0 else coord[ax] < extent[ax] - 1
            r = np.nonzero(has)[0]
            if kp is None:
                face = np.full(r.size, float(scale[ax]))
            else:
                face = scale[ax] * _hm(kp[r], kappa[idx[r] + off])
            col[pos[r]] = (idx[r] + off).astype(np.int32)
            val[pos[r]] = -face
            pos[r] += 1
    return Csr(n, row_ptr, col, val)


def poisson2d(N: int) -> Csr:
    """MATLAB gallery('poisson', N): n=N², nnz = n + 4N(N-1)."""
    return stencil_csr(N, N, ndim=2)


def csr_matvec(A: Csr, x: np.ndarray) -> np.ndarray:
    """Plain CSR matvec used only to form b = A·x_rand for the paper-protocol right-hand side."""
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    return np.bincount(rows, weights=A.val * x[A.col], minlength=A.n)


# ----------------------------------------------------------------------------
# Coefficient fields
# ----------------------------------------------------------------------------
def bands_kappa(N: int, band: int = 32, hi: float = 1e3) -> np.ndarray:
    """cfg2: κ = 1 in even bands ⌊y/band⌋, `hi` in odd bands (reading R19)."""
    y = np.arange(N * N) // N
    return np.where((y // band) % 2 == 1, hi, 1.0)


def fisher_yates(seed: int, m: int) -> list:
    """Seeded Fisher–Yates permutation of range(m): for i=m-1..1, j = ⌊u·(i+1)⌋ with u the next draw."""
    perm = list(range(m))
    k = 0
    for i in range(m - 1, 0, -1):
        z = splitmix64_scalar(seed, k)
        k += 1
        j = ((z >> 11) * (i + 1)) >> 53
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def subcubes_kappa(N: int, cell: int = 8, frac_num: int = 1, frac_den: int = 4,
                   hi: float = 1e3, seed: int = SEED_CFG3_CELLS) -> np.ndarray:
    """cfg3: tile N³ into aligned cell³ cubes; the first ⌊count·frac⌋ of a seeded shuffle get κ=hi (R18)."""
    c = N // cell
    ncell = c ** 3
    chosen = fisher_yates(seed, ncell)[: ncell * frac_num // frac_den]
    mark = np.zeros(ncell, bool)
    mark[chosen] = True
    idx = np.arange(N ** 3, dtype=np.int64)
    x, y, z = idx % N, (idx // N) % N, idx // (N * N)
    cid = (x // cell) + c * ((y // cell) + c * (z // cell))
    return np.where(mark[cid], hi, 1.0)


# ----------------------------------------------------------------------------
# BASELINE.json configurations
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Problem:
    name: str
    A: Csr
    b: np.ndarray
    method: str        # "sre-cg" | "sre-cg2" | "msdo-cg"
    s: int
    t: int
    tol: float
    grid: tuple
    note: str = ""


def cfg1() -> Problem:
    A = poisson2d(64)
    return Problem("cfg1", A, uniform_pm1(SEED_B[1], A.n), "sre-cg", 2, 4, 1e-8, (64, 64),
                   "2D Poisson 64x64, b~U[-1,1) seed 1805")


def cfg2(N: int = 512, method: str = "sre-cg") -> Problem:
    A = stencil_csr(N, N, ndim=2, kappa=bands_kappa(N))
    return Problem("cfg2" if N == 512 else f"cfg2-analog{N}", A, uniform_pm1(SEED_B[2], A.n), method, 3, 16, 1e-8,
                   (N, N), f"2D bands {N}x{N}, kappa in {{1,1e3}} bands of 32, b~U[-1,1) seed 1806")


def cfg3(N: int = 128) -> Problem:
    A = stencil_csr(N, N, N, ndim=3, kappa=subcubes_kappa(N))
    return Problem("cfg3" if N == 128 else f"cfg3-analog{N}", A, uniform_pm1(SEED_B[3], A.n), "msdo-cg", 4, 32, 1e-8,
                   (N, N, N), f"3D subcubes {N}^3, 25% of 8^3 cells kappa=1e3 (seed 1834), b~U[-1,1) seed 1807")


def cfg4(N: int = 256) -> Problem:
    A = stencil_csr(N, N, N, ndim=3, scale=(1.0, 1.0, 1e-2))
    return Problem("cfg4" if N == 256 else f"cfg4-analog{N}", A, np.ones(A.n), "sre-cg", 2, 64, 1e-8,
                   (N, N, N), f"3D anisotropic {N}^3, z faces 1e-2, b=1")


def cfg5_operator(N: int = 384) -> Csr:
    return stencil_csr(N, N, N, ndim=3)


def cfg5_start_block(n: int, t: int, seed: int = SEED_CFG5_BLOCK) -> np.ndarray:
    """cfg5 random start: U[-1,1) drawn in row-major n×t order, columns scaled to unit 2-norm (R27)."""
    X = uniform_pm1(seed, n * t).reshape(n, t)
    X /= np.sqrt((X * X).sum(axis=0))
    return X


def cfg5_start_block_torch(n: int, t: int, device, seed: int = SEED_CFG5_BLOCK):
    """cfg5 start block generated on the device (same draws as :func:`cfg5_start_block`; the
    column norms are summed by torch, so the scaling may differ from the numpy block by rounding)."""
    X = uniform_pm1_torch(seed, n * t, device).view(n, t)
    X /= X.pow(2).sum(dim=0).sqrt()
    return X


def paper_poisson_rhs(A: Csr, seed: int = 1804) -> np.ndarray:
    """Paper protocol: x_rand ~ U(0,1), b = A·x_rand."""
    return csr_matvec(A, uniform01(seed, A.n))


def spd_dense(n: int, seed: int, lo: float = 1.0, hi: float = 100.0) -> np.ndarray:
    """Tiny dense SPD A = QΛQᵀ with seeded Q (QR of a U[-1,1) matrix) and Λ log-uniform in [lo, hi]."""
    G = uniform_pm1(seed, n * n).reshape(n, n)
    Q, _ = np.linalg.qr(G)
    lam = np.exp(np.log(lo) + (np.log(hi) - np.log(lo)) * uniform01(seed + 1, n))
    A = (Q * lam) @ Q.T
    return 0.5 * (A + A.T)
