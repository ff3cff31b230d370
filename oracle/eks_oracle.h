/* eks_oracle.h — CPU reference ("oracle") for the s-step enlarged CG hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * The product (paper_1804_10629_b200/, libeks.so) never links, imports or
 * executes it, and this tree shares no source, header, table or helper with
 * the CUDA path.
 *
 * Plain single-threaded C99, fp64, no BLAS, no OpenMP, built with
 * -O2 -ffp-contract=off (reading R20).  Every routine cites the
 * PAPER.md passage it follows ("P:<line>", section / algorithm).
 *
 * Layout: every n×t block is ROW-MAJOR (row i's t values contiguous).
 */
#ifndef EKS_ORACLE_H
#define EKS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n;
  const int64_t* row_ptr;  /* n+1, row_ptr[0] == 0 */
  const int32_t* col;      /* nnz, ascending within a row */
  const double* val;       /* nnz */
} or_csr;

enum { OR_SRE_CG = 0, OR_SRE_CG2 = 1, OR_MSDO_CG = 2 };
enum { OR_OK = 0, OR_BREAKDOWN = 7, OR_MAXITER = 8, OR_BADARG = 1 };
/* DEFINITION: the paper's algebra (explicit SpMMs Qᵀ(A·Z), u = Vα̃, r −= A·u);  MIRROR: the GPU's
 * algebra (cached A·Q, C = (AQ)ᵀZ, r −= Σ (AW)α̃);  ONESYNCH: MIRROR with the one-synch CGS2 of
 * reading R36 (SpMM of Z1, Z2ᵀAZ2 = Z1ᵀAZ1 − C2ᵀC2, A·Z2 = A·Z1 − (AQ)C2). */
enum { OR_MODE_DEFINITION = 0, OR_MODE_MIRROR = 1, OR_MODE_ONESYNCH = 2 };
enum { OR_ORTHO_ACHOLQR = 0, OR_ORTHO_PRE = 1 };

/* Per-outer-iteration hook for the invariant pins (tests only).
 * V is the n×(s·t) basis of this outer iteration, row-major; alpha = Vᵀr_{k-1};
 * x, r are x_k, r_k after the update. */
typedef void (*or_iter_cb)(void* user, int k, int64_t n, int st, const double* V,
                           const double* alpha, const double* x, const double* r, double rho);

typedef struct {
  int outer_iters;      /* loop bodies executed (= k-1 at exit, P:146 / reading R7) */
  int converged;        /* rho <= eps*rho0 */
  int status;           /* OR_OK / OR_BREAKDOWN / OR_MAXITER */
  int breakdown_block;  /* global block index of the failed Cholesky, or -1 */
  double rho0, rho, true_relres;
  double* rho_history;  /* caller-owned, capacity kmax+1, may be NULL */
} or_report;

/* T(r): Z[i][d] = r[i] if i in D_d else 0, D_d = [floor(d n/t), floor((d+1) n/t)).
 * P:41 (§2, "T(r_0) is an operator that splits r_0 into t vectors"). */
void or_split(int64_t n, int t, const double* r, double* Z);

/* Y = A·X (n×t), accumulation p ascending from 0.0 with fma (reading R20).
 * P:54 (§3.1, "W_k = AW_{k-1}"). */
void or_spmm(const or_csr* A, int t, const double* X, double* Y);

/* C = Xᵀ Y (p×q, row-major), X n×p, Y n×q, Neumaier-compensated sums over rows. */
void or_xty(int64_t n, int p, const double* X, int q, const double* Y, double* C);

/* Cholesky B = RᵀR (t×t, R upper, row-major), only B's upper triangle read.
 * Breakdown (returns OR_BREAKDOWN) when a pivot d_k <= t·2^-52·max|B_ij| (reading R6). */
int or_chol(int t, const double* B, double* R);

/* CGS2 "A-orthonormalize Z against Q" (reading R3):
 * twice { C = Qᵀ(A·Z) ; Z = Z − Q·C }.  Q is given as nq blocks of n×t.
 * C1, C2 (nq·t × t, row-major) receive the two passes' coefficients (may be NULL). */
void or_cgs2(const or_csr* A, int t, int nq, const double* const* Q, double* Z,
             double* C1, double* C2);

/* A-CholQR "A-orthonormalize W" (reading R4):
 * B = upper(Zᵀ(A·Z)), B = RᵀR, W = Z·R⁻¹ (row-wise forward substitution). */
int or_acholqr(const or_csr* A, int t, const double* Z, double* W, double* R, double* B);

/* Pre-CholQR "A-orthonormalize W" (reading R30): Euclidean CholQR of Z
 * (G = upper(ZᵀZ) = R1ᵀR1, Z1 = Z·R1⁻¹), then A-CholQR of Z1 (R2); W = Z1·R2⁻¹ and
 * R = R2·R1 (so Z = W·R).  OR_BREAKDOWN from either Cholesky. */
int or_precholqr(const or_csr* A, int t, const double* Z, double* W, double* R);

/* Solve with s-step SRE-CG (Alg 4), SRE-CG2 (Alg 3) or
 * MSDO-CG (Alg 6).  x holds x0 on entry, x_k on exit. */
int or_solve(const or_csr* A, const double* b, double* x, int method, int s, int t,
             double eps, int kmax, int mode, or_report* rep, or_iter_cb cb, void* user);

/* or_solve with the self-orthonormalization chosen (ortho = OR_ORTHO_ACHOLQR | OR_ORTHO_PRE,
 * P:198) and, for SRE-CG / SRE-CG2, the restructured Alg 2 / Alg 1 (restructured = 1,
 * P:58-120): the same s blocks, then s sequential updates alpha~_i = W_iᵀ r_{i-1},
 * x_i = x_{i-1} + W_i alpha~_i, r_i = r_{i-1} − A W_i alpha~_i; convergence tested once per s.
 * MSDO-CG has no restructured form → OR_BADARG. */
int or_solve_ex(const or_csr* A, const double* b, double* x, int method, int s, int t,
                double eps, int kmax, int mode, int ortho, int restructured, or_report* rep,
                or_iter_cb cb, void* user);

/* Block-Jacobi IC(0) preconditioner M = L·Lᵗ (Table 5; reading R32): nd contiguous
 * domains D_d = [floor(d n/nd), floor((d+1) n/nd)), each diagonal block factorized by incomplete
 * Cholesky with zero fill-in.  L is CSR (ascending columns, diagonal last) with the pattern of
 * the lower triangle of the block diagonal of A; or_ic0_nnz gives its nnz. */
int64_t or_ic0_nnz(const or_csr* A, int nd);
int or_ic0(const or_csr* A, int nd, int64_t* Lrp, int32_t* Lcol, double* Lval);
/* The same with a complete Cholesky of each diagonal block (Table 6; reading R32): L holds
 * the row envelope (columns f_i..i of the domain, f_i = first nonzero of row i of A_dd), where
 * the natural-order factor's fill lives; envelope (skyline) Cholesky. */
int64_t or_cholblk_nnz(const or_csr* A, int nd);
int or_cholblk(const or_csr* A, int nd, int64_t* Lrp, int32_t* Lcol, double* Lval);
/* Y = L⁻¹Z and Y = L⁻ᵗZ for n×t row-major blocks (Y may alias Z). */
void or_lsolve(const or_csr* L, int t, const double* Z, double* Y);
void or_ltsolve(const or_csr* L, int t, const double* Z, double* Y);

/* or_solve_ex with a split preconditioner M = L·Lᵗ (L NULL: none): the split-preconditioned
 * s-step SRE-CG / SRE-CG2 / MSDO-CG of Alg 8 / 9 / 10: seed L⁻ᵗ[T(L⁻¹r)], powers
 * M⁻¹A·W, A-orthonormalization and the x/r update unchanged.  Not with
 * restructured (OR_BADARG). */
int or_solve_pc(const or_csr* A, const double* b, double* x, int method, int s, int t,
                double eps, int kmax, int mode, int ortho, int restructured, const or_csr* L,
                or_report* rep, or_iter_cb cb, void* user);

/* Communication-avoiding s-step enlarged CG: CA SRE-CG, CA SRE-CG2
 * (method 0 / 1) and CA MSDO-CG (method 2) with the CA-Arnoldi
 * A-orthonormalization (arnoldi = 5, Alg 5) or its modified, stabilised form
 * (arnoldi = 7, Alg 7).  The st vectors of an outer iteration are formed as a
 * monomial block [W, AW, …, A^{s-1}W] and A-orthonormalized together (one st×st CholQR). */
int or_solve_ca(const or_csr* A, const double* b, double* x, int method, int arnoldi, int s, int t,
                double eps, int kmax, or_report* rep, or_iter_cb cb, void* user);

/* or_solve_ca with the split preconditioner M = L·Lᵗ (L NULL: none): the seed
 * L⁻ᵗ[T(L⁻¹r)] and the monomial powers M⁻¹A·W. */
int or_solve_ca_pc(const or_csr* A, const double* b, double* x, int method, int arnoldi, int s, int t,
                   double eps, int kmax, const or_csr* L, or_report* rep, or_iter_cb cb, void* user);

/* s-step SRE-CG basis sweep only (cfg5, reading R27): starting block X0 (n×t)
 * is A-orthonormalized, then nblocks-1 further blocks W=A-orth(A·W_prev) against
 * the last min(2,#) blocks.  Writes the last block to W_last.  Returns status. */
int or_basis_sweep(const or_csr* A, int t, const double* X0, int nblocks, double* W_last);

#ifdef __cplusplus
}
#endif
#endif
