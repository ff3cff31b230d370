/* eks_oracle.c — plain, slow, single-threaded fp64 CPU oracle for the
 * s-step enlarged CG methods of arXiv:1804.10629.
 *
 * TEST INFRASTRUCTURE ONLY (see eks_oracle.h).  Shares no code with the
 * CUDA product.  Build: gcc -O2 -ffp-contract=off -fPIC -shared.
 *
 * The routines follow the paper's algorithm boxes step by step:
 *   s-step SRE-CG2  Alg 3
 *   s-step SRE-CG   Alg 4, window of 2 blocks
 *   s-step MSDO-CG  Alg 6
 *   A-orthonormalization = CGS2 against the window + A-CholQR
 * Readings of silent/ambiguous points (R1..R27) are listed in DESIGN.md.
 *
 * Parity status: every routine here is pinned by tests/test_oracle_*.py
 * (closed forms, textbook CG, dense direct solves, paper table cells).
 */
#include "eks_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Small helpers                                                             */
/* ------------------------------------------------------------------------ */

/* Neumaier-compensated running sum. */
typedef struct { double s, c; } ksum;
static void ks_add(ksum* k, double v) {
  double t = k->s + v;
  if (fabs(k->s) >= fabs(v)) k->c += (k->s - t) + v;
  else k->c += (v - t) + k->s;
  k->s = t;
}
static double ks_val(const ksum* k) { return k->s + k->c; }

static double* dalloc(size_t count) {
  double* p = (double*)calloc(count ? count : 1, sizeof(double));
  if (!p) abort();
  return p;
}

static double norm2(int64_t n, const double* v) {
  ksum k = {0, 0};
  for (int64_t i = 0; i < n; ++i) ks_add(&k, v[i] * v[i]);
  return sqrt(ks_val(&k));
}

/* ------------------------------------------------------------------------ */
/* T(r) — P:41 (§2), P:311-312 (proof of Theorem 1: r = T(r)·1_t)            */
/* ------------------------------------------------------------------------ */
void or_split(int64_t n, int t, const double* r, double* Z) {
  /* Domains D_d = [floor(d n / t), floor((d+1) n / t)) (reading R1). */
  memset(Z, 0, sizeof(double) * (size_t)n * (size_t)t);
  for (int d = 0; d < t; ++d) {
    int64_t lo = (int64_t)d * n / t, hi = (int64_t)(d + 1) * n / t;
    for (int64_t i = lo; i < hi; ++i) Z[i * t + d] = r[i];
  }
}

/* ------------------------------------------------------------------------ */
/* Y = A X — P:54 ("W_k = AW_{k-1}"); fixed ascending fma order (R20)        */
/* ------------------------------------------------------------------------ */
void or_spmm(const or_csr* A, int t, const double* X, double* Y) {
  for (int64_t i = 0; i < A->n; ++i) {
    for (int c = 0; c < t; ++c) {
      double acc = 0.0;
      for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p)
        acc = fma(A->val[p], X[(int64_t)A->col[p] * t + c], acc);
      Y[i * t + c] = acc;
    }
  }
}

/* C = Xᵀ Y, compensated over rows. */
void or_xty(int64_t n, int p, const double* X, int q, const double* Y, double* C) {
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < q; ++b) {
      ksum k = {0, 0};
      for (int64_t i = 0; i < n; ++i) ks_add(&k, X[i * p + a] * Y[i * q + b]);
      C[a * q + b] = ks_val(&k);
    }
}

/* ------------------------------------------------------------------------ */
/* Cholesky B = RᵀR — A-CholQR's factorization ("A-CholQR"; R4, R6)   */
/* Column-by-column, left-to-right sums, no fma (compiled -ffp-contract=off). */
/* ------------------------------------------------------------------------ */
int or_chol(int t, const double* B, double* R) {
  double bmax = 0.0;
  for (int i = 0; i < t; ++i)
    for (int j = i; j < t; ++j)
      if (fabs(B[i * t + j]) > bmax) bmax = fabs(B[i * t + j]);
  double thr = (double)t * ldexp(1.0, -52) * bmax;
  memset(R, 0, sizeof(double) * (size_t)t * (size_t)t);
  for (int k = 0; k < t; ++k) {
    double d = B[k * t + k];
    for (int i = 0; i < k; ++i) d = d - R[i * t + k] * R[i * t + k];
    if (!(d > thr)) return OR_BREAKDOWN;
    double rkk = sqrt(d);
    R[k * t + k] = rkk;
    for (int j = k + 1; j < t; ++j) {
      double v = B[k * t + j];
      for (int i = 0; i < k; ++i) v = v - R[i * t + k] * R[i * t + j];
      R[k * t + j] = v / rkk;
    }
  }
  return OR_OK;
}

/* W = Z R⁻¹ row by row: w R = z  ⇒  w_j = (z_j − Σ_{i<j} w_i R_ij) / R_jj. */
static void rsolve_rows(int64_t n, int t, const double* R, const double* Z, double* W) {
  for (int64_t r = 0; r < n; ++r) {
    const double* z = Z + r * t;
    double* w = W + r * t;
    for (int j = 0; j < t; ++j) {
      double v = z[j];
      for (int i = 0; i < j; ++i) v = v - w[i] * R[i * t + j];
      w[j] = v / R[j * t + j];
    }
  }
}

/* Rᵀ a = g (forward substitution on the lower-triangular Rᵀ). */
static void rtsolve_vec(int t, const double* R, const double* g, double* a) {
  for (int j = 0; j < t; ++j) {
    double v = g[j];
    for (int i = 0; i < j; ++i) v = v - R[i * t + j] * a[i];
    a[j] = v / R[j * t + j];
  }
}

/* ------------------------------------------------------------------------ */
/* CGS2 in the A-inner product — P:198 ("A-orthonormalized against all the   */
/* previously computed vectors using CGS2"); reading R3.         */
/* ------------------------------------------------------------------------ */
static void cgs_pass_from_AZ(int64_t n, int t, int nq, const double* const* Q,
                             const double* const* AQ_or_null, const double* AZ_or_Z,
                             double* Z, double* C) {
  /* C_q = Q_qᵀ (A Z)  [definition]   or   C_q = (A Q_q)ᵀ Z  [mirror]. */
  for (int q = 0; q < nq; ++q) {
    const double* left = AQ_or_null ? AQ_or_null[q] : Q[q];
    or_xty(n, t, left, t, AZ_or_Z, C + (size_t)q * t * t);
  }
  /* Z = Z − Q C, per row: z_c −= Σ_q Σ_a Q_q[row][a] C_q[a][c]. */
  for (int64_t r = 0; r < n; ++r)
    for (int c = 0; c < t; ++c) {
      double acc = 0.0;
      for (int q = 0; q < nq; ++q)
        for (int a = 0; a < t; ++a) acc += Q[q][r * t + a] * C[((size_t)q * t + a) * t + c];
      Z[r * t + c] -= acc;
    }
}

void or_cgs2(const or_csr* A, int t, int nq, const double* const* Q, double* Z,
             double* C1, double* C2) {
  int64_t n = A->n;
  double* AZ = dalloc((size_t)n * t);
  double* Cbuf = dalloc((size_t)nq * t * t);
  for (int pass = 0; pass < 2; ++pass) {
    or_spmm(A, t, Z, AZ);
    cgs_pass_from_AZ(n, t, nq, Q, NULL, AZ, Z, Cbuf);
    double* dst = pass == 0 ? C1 : C2;
    if (dst) memcpy(dst, Cbuf, sizeof(double) * (size_t)nq * t * t);
  }
  free(AZ);
  free(Cbuf);
}

/* ------------------------------------------------------------------------ */
/* A-CholQR — P:198; reading R4                                       */
/* ------------------------------------------------------------------------ */
int or_acholqr(const or_csr* A, int t, const double* Z, double* W, double* R, double* Bout) {
  int64_t n = A->n;
  double* AZ = dalloc((size_t)n * t);
  double* B = dalloc((size_t)t * t);
  or_spmm(A, t, Z, AZ);
  or_xty(n, t, Z, t, AZ, B);
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < i; ++j) B[i * t + j] = 0.0; /* upper triangle only (R4) */
  if (Bout) memcpy(Bout, B, sizeof(double) * (size_t)t * t);
  int st = or_chol(t, B, R);
  if (st == OR_OK) rsolve_rows(n, t, R, Z, W);
  free(AZ);
  free(B);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Pre-CholQR — P:198 ("A-orthonormalized using A-CholQR or Pre-CholQR"),    */
/* P:380 ("Pre-CholQR is numerically more stable than A-CholQR"); the cited */
/* thesis's Algorithm 23 is not in the paper, so the standard definition    */
/* (reading R30): a Euclidean CholQR of Z (G = ZᵀZ = R1ᵀR1, */
/* Z1 = Z R1⁻¹), then A-CholQR of Z1 (R2); Z = W·R with R = R2·R1.           */
/* ------------------------------------------------------------------------ */
int or_precholqr(const or_csr* A, int t, const double* Z, double* W, double* R) {
  int64_t n = A->n;
  double* G = dalloc((size_t)t * t);
  double* R1 = dalloc((size_t)t * t);
  double* R2 = dalloc((size_t)t * t);
  double* Z1 = dalloc((size_t)n * t);
  or_xty(n, t, Z, t, Z, G);
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < i; ++j) G[i * t + j] = 0.0;
  int st = or_chol(t, G, R1);
  if (st == OR_OK) {
    rsolve_rows(n, t, R1, Z, Z1);
    st = or_acholqr(A, t, Z1, W, R2, NULL);
  }
  if (st == OR_OK && R) {
    for (int i = 0; i < t; ++i)
      for (int j = 0; j < t; ++j) {
        double v = 0.0;
        for (int k = i; k <= j; ++k) v += R2[i * t + k] * R1[k * t + j];
        R[i * t + j] = j >= i ? v : 0.0;
      }
  }
  free(G); free(R1); free(R2); free(Z1);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Block-Jacobi IC(0) preconditioner M = L Lᵗ — P:872-882 (§5.2): nd        */
/* contiguous domains (Metis in the paper, reading R32), each diagonal block */
/* A_dd factorized by incomplete Cholesky with zero fill-in (Table 5).       */
/* ------------------------------------------------------------------------ */
static int64_t dom_of(int64_t n, int nd, int64_t i) {
  int64_t d = i * nd / n;  /* candidate, then fix up against floor(d n / nd) */
  while (d > 0 && d * n / nd > i) --d;
  while (d + 1 < nd && (d + 1) * n / nd <= i) ++d;
  return d;
}

int64_t or_ic0_nnz(const or_csr* A, int nd) {
  int64_t cnt = 0;
  for (int64_t i = 0; i < A->n; ++i)
    for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
      int64_t j = A->col[p];
      if (j <= i && dom_of(A->n, nd, j) == dom_of(A->n, nd, i)) ++cnt;
    }
  return cnt;
}

/* L (CSR, rows ascending columns, diagonal last) with the pattern of the lower triangle of
 * the block diagonal of A.  Row-oriented IC(0): for k < i in the pattern of row i,
 * L_ik = (A_ik − Σ_{j<k} L_ij L_kj) / L_kk over j in both rows' patterns;
 * L_ii = sqrt(A_ii − Σ_{j<i} L_ij²).  OR_BREAKDOWN if a diagonal argument is ≤ 0. */
int or_ic0(const or_csr* A, int nd, int64_t* Lrp, int32_t* Lcol, double* Lval) {
  int64_t n = A->n, q = 0;
  Lrp[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t di = dom_of(n, nd, i);
    for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
      int64_t j = A->col[p];
      if (j <= i && dom_of(n, nd, j) == di) { Lcol[q] = (int32_t)j; Lval[q] = A->val[p]; ++q; }
    }
    Lrp[i + 1] = q;
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = Lrp[i], e = Lrp[i + 1];
    if (e == a || Lcol[e - 1] != i) return OR_BADARG;  /* a missing diagonal */
    for (int64_t p = a; p < e - 1; ++p) {
      int64_t k = Lcol[p];
      double v = Lval[p];
      /* Σ over j < k present in row i (positions a..p-1) and in row k */
      int64_t pk = Lrp[k], ek = Lrp[k + 1] - 1;
      for (int64_t pi = a; pi < p; ++pi) {
        while (pk < ek && Lcol[pk] < Lcol[pi]) ++pk;
        if (pk < ek && Lcol[pk] == Lcol[pi]) v = v - Lval[pi] * Lval[pk];
      }
      Lval[p] = v / Lval[Lrp[k + 1] - 1];
    }
    double d = Lval[e - 1];
    for (int64_t p = a; p < e - 1; ++p) d = d - Lval[p] * Lval[p];
    if (!(d > 0.0)) return OR_BREAKDOWN;
    Lval[e - 1] = sqrt(d);
  }
  return OR_OK;
}

/* Block-Jacobi with a COMPLETE Cholesky of each diagonal block (Table 6).  For the
 * natural ordering the factor's fill stays inside the row envelope (profile): row i of L holds
 * the columns f_i..i of its domain, f_i = the first nonzero column of row i of A_dd.  Envelope
 * (skyline) Cholesky, row by row: L_ij = (A_ij − Σ_{k=max(f_i,f_j)}^{j-1} L_ik L_jk) / L_jj,
 * L_ii = sqrt(A_ii − Σ_{k=f_i}^{i-1} L_ik²).  or_cholblk_nnz gives the envelope size. */
static int64_t env_first(const or_csr* A, int nd, int64_t i) {
  int64_t di = dom_of(A->n, nd, i), f = i;
  for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
    int64_t j = A->col[p];
    if (j < f && dom_of(A->n, nd, j) == di) f = j;
  }
  return f;
}

int64_t or_cholblk_nnz(const or_csr* A, int nd) {
  int64_t cnt = 0;
  for (int64_t i = 0; i < A->n; ++i) cnt += i - env_first(A, nd, i) + 1;
  return cnt;
}

int or_cholblk(const or_csr* A, int nd, int64_t* Lrp, int32_t* Lcol, double* Lval) {
  int64_t n = A->n, q = 0;
  Lrp[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t f = env_first(A, nd, i);
    for (int64_t j = f; j <= i; ++j) { Lcol[q] = (int32_t)j; Lval[q] = 0.0; ++q; }
    Lrp[i + 1] = q;
    /* A's entries of the envelope */
    for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
      int64_t j = A->col[p];
      if (j >= f && j <= i) Lval[Lrp[i] + (j - f)] = A->val[p];
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t fi = Lcol[Lrp[i]];
    double* Li = Lval + Lrp[i];  /* Li[j - fi] = L_ij */
    for (int64_t j = fi; j < i; ++j) {
      int64_t fj = Lcol[Lrp[j]];
      const double* Lj = Lval + Lrp[j];
      double v = Li[j - fi];
      for (int64_t k = fi > fj ? fi : fj; k < j; ++k) v = v - Li[k - fi] * Lj[k - fj];
      Li[j - fi] = v / Lj[j - fj];
    }
    double d = Li[i - fi];
    for (int64_t k = fi; k < i; ++k) d = d - Li[k - fi] * Li[k - fi];
    if (!(d > 0.0)) return OR_BREAKDOWN;
    Li[i - fi] = sqrt(d);
  }
  return OR_OK;
}

/* Y = L⁻¹ Z (n×t, row-major; Y may alias Z): forward substitution per column. */
void or_lsolve(const or_csr* L, int t, const double* Z, double* Y) {
  for (int64_t i = 0; i < L->n; ++i) {
    int64_t a = L->row_ptr[i], e = L->row_ptr[i + 1];
    for (int c = 0; c < t; ++c) {
      double v = Z[i * t + c];
      for (int64_t p = a; p < e - 1; ++p) v = v - L->val[p] * Y[(int64_t)L->col[p] * t + c];
      Y[i * t + c] = v / L->val[e - 1];
    }
  }
}

/* Y = L⁻ᵗ Z (Y may alias Z): backward substitution, column-oriented over L's rows. */
void or_ltsolve(const or_csr* L, int t, const double* Z, double* Y) {
  if (Y != Z) memcpy(Y, Z, sizeof(double) * (size_t)L->n * (size_t)t);
  for (int64_t i = L->n - 1; i >= 0; --i) {
    int64_t a = L->row_ptr[i], e = L->row_ptr[i + 1];
    for (int c = 0; c < t; ++c) {
      double yi = Y[i * t + c] / L->val[e - 1];
      Y[i * t + c] = yi;
      for (int64_t p = a; p < e - 1; ++p) Y[(int64_t)L->col[p] * t + c] -= L->val[p] * yi;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Block list (the Q of Alg 3/6 or the 2-block window of Alg 4)              */
/* ------------------------------------------------------------------------ */
typedef struct {
  int count, cap;
  double** W;   /* A-orthonormal blocks */
  double** AW;  /* mirror mode: cached A·W */
} blist;

static void bl_push(blist* L, double* W, double* AW) {
  if (L->count == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 8;
    L->W = (double**)realloc(L->W, sizeof(double*) * (size_t)L->cap);
    L->AW = (double**)realloc(L->AW, sizeof(double*) * (size_t)L->cap);
  }
  L->W[L->count] = W;
  L->AW[L->count] = AW;
  L->count++;
}

static void bl_free(blist* L) {
  for (int i = 0; i < L->count; ++i) { free(L->W[i]); free(L->AW[i]); }
  free(L->W);
  free(L->AW);
}

/* Window for the next block: SRE-CG → the last min(2, #) blocks (Alg 4,
 * P:182/"against W_{j-2} and W_{j-1}"; R11); SRE-CG2 and MSDO-CG →
 * all of Q (Alg 3; Alg 6). */
static int window_start(const blist* L, int method) {
  if (method == OR_SRE_CG) return L->count > 2 ? L->count - 2 : 0;
  return 0;
}

/* SRE-CG keeps only the last 2 blocks: drop older ones to bound memory. */
static void bl_trim(blist* L, int method) {
  if (method != OR_SRE_CG) return;
  while (L->count > 2) {
    free(L->W[0]);
    free(L->AW[0]);
    memmove(L->W, L->W + 1, sizeof(double*) * (size_t)(L->count - 1));
    memmove(L->AW, L->AW + 1, sizeof(double*) * (size_t)(L->count - 1));
    L->count--;
  }
}

/* ------------------------------------------------------------------------ */
/* Solver — Alg 3 / Alg 4 / Alg 6                                            */
/* ------------------------------------------------------------------------ */
int or_solve(const or_csr* A, const double* b, double* x, int method, int s, int t,
             double eps, int kmax, int mode, or_report* rep, or_iter_cb cb, void* user) {
  return or_solve_ex(A, b, x, method, s, t, eps, kmax, mode, OR_ORTHO_ACHOLQR, 0, rep, cb, user);
}

int or_solve_ex(const or_csr* A, const double* b, double* x, int method, int s, int t,
                double eps, int kmax, int mode, int ortho, int restructured, or_report* rep,
                or_iter_cb cb, void* user) {
  return or_solve_pc(A, b, x, method, s, t, eps, kmax, mode, ortho, restructured, NULL, rep, cb, user);
}

int or_solve_pc(const or_csr* A, const double* b, double* x, int method, int s, int t,
                double eps, int kmax, int mode, int ortho, int restructured, const or_csr* L,
                or_report* rep, or_iter_cb cb, void* user) {
  int64_t n = A->n;
  if (L && (L->n != n || restructured)) return OR_BADARG;
  if (s < 1 || t < 1 || t > n || !(eps >= 0.0) || method < 0 || method > 2) return OR_BADARG;
  if (ortho != OR_ORTHO_ACHOLQR && ortho != OR_ORTHO_PRE) return OR_BADARG;
  /* restructured Alg 1/2 exist for SRE-CG2 / SRE-CG only (no restructured MSDO-CG) */
  if (restructured && method == OR_MSDO_CG) return OR_BADARG;
  if (mode < OR_MODE_DEFINITION || mode > OR_MODE_ONESYNCH) return OR_BADARG;
  /* one-synch CGS2 (reading R36): A-CholQR only, not with the restructured update */
  if (mode == OR_MODE_ONESYNCH && (ortho != OR_ORTHO_ACHOLQR || restructured)) return OR_BADARG;
  size_t blk = (size_t)n * (size_t)t;

  double* r = dalloc((size_t)n);
  double* tmp = dalloc((size_t)n);
  double* u = dalloc((size_t)n);
  /* r_0 = b − A x_0 ; rho_0 = ||r_0||_2  (line 1 of every algorithm box) */
  or_spmm(A, 1, x, tmp);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
  double rho0 = norm2(n, r), rho = rho0;
  if (rep) {
    rep->rho0 = rho0;
    rep->breakdown_block = -1;
    if (rep->rho_history) rep->rho_history[0] = rho0;
  }

  blist Q = {0, 0, NULL, NULL};
  double** V = (double**)calloc((size_t)s, sizeof(double*));
  double** AV = (double**)calloc((size_t)s, sizeof(double*));
  double* alpha = dalloc((size_t)s * t);
  double* R = dalloc((size_t)t * t);
  double* B = dalloc((size_t)t * t);
  double* g = dalloc((size_t)t);
  double* Cb = NULL;
  int status = OR_OK, k = 1, gblock = 0;
  double* rnew = dalloc((size_t)n);

  /* while (rho > eps*rho0 and k < kmax)   — P:146 / P:177 / P:329 (R7) */
  while (rho > eps * rho0 && k < kmax) {
    memcpy(rnew, r, sizeof(double) * (size_t)n);
    int ok = 1;
    for (int i = 0; i < s; ++i) {
      double* Z = dalloc(blk);
      /* Seed block: T(r_{k-1}) for MSDO-CG every k (Alg 6) and for
       * SRE-CG/SRE-CG2 at k=1 (Alg 3, Alg 4); otherwise the next
       * power A·W_{j-1}. */
      if (i == 0 && (method == OR_MSDO_CG || k == 1)) {
        if (L) {
          /* Alg 8/9 line 5, Alg 10 line 3: W = L⁻ᵗ[T(L⁻¹ r_{k-1})] */
          or_lsolve(L, 1, r, tmp);
          or_split(n, t, tmp, Z);
          or_ltsolve(L, t, Z, Z);
        } else {
          or_split(n, t, r, Z);
        }
      } else {
        const double* Wprev = Q.W[Q.count - 1];
        if (mode != OR_MODE_DEFINITION) memcpy(Z, Q.AW[Q.count - 1], sizeof(double) * blk);
        else or_spmm(A, t, Wprev, Z);
        if (L) { /* Alg 8-10: W_{j} = M⁻¹ A W_{j-1} = L⁻ᵗ L⁻¹ (A W_{j-1}) */
          or_lsolve(L, t, Z, Z);
          or_ltsolve(L, t, Z, Z);
        }
      }
      int w0 = window_start(&Q, method), nq = Q.count - w0;
      double* W = dalloc(blk);
      double* AW = NULL;
      if (mode == OR_MODE_DEFINITION) {
        /* "A-orthonormalize W against Q" (CGS2), then "A-orthonormalize W" (A-CholQR). */
        if (nq > 0) or_cgs2(A, t, nq, (const double* const*)(Q.W + w0), Z, NULL, NULL);
        int st = ortho == OR_ORTHO_PRE ? or_precholqr(A, t, Z, W, R) : or_acholqr(A, t, Z, W, R, NULL);
        if (st != OR_OK) { status = OR_BREAKDOWN; free(Z); free(W); ok = 0; break; }
        AW = dalloc(1);
      } else {
        /* Mirror of the GPU algebra: C = (AQ)ᵀZ with cached AQ, one SpMM of Z2,
         * AW = (A Z2) R⁻¹, alpha_b = R⁻ᵀ (Z2ᵀ r_{k-1}). Equal to the definition in
         * exact arithmetic (A symmetric, reading R24). */
        double* AZ = dalloc(blk);
        int synched = 0; /* one-synch: B, g, Z2 and A·Z2 already formed below */
        if (nq > 0) {
          Cb = (double*)realloc(Cb, sizeof(double) * (size_t)nq * t * t);
          for (int pass = 0; pass < (mode == OR_MODE_ONESYNCH ? 1 : 2); ++pass)
            cgs_pass_from_AZ(n, t, nq, (const double* const*)(Q.W + w0),
                             (const double* const*)(Q.AW + w0), Z, Z, Cb);
        }
        if (nq > 0 && mode == OR_MODE_ONESYNCH) {
          /* One-synch CGS2 (DESIGN reading R36): the SpMM runs on Z1 and
           * C2 = (AQ)ᵀZ1, B1 = Z1ᵀ(A Z1), g1 = Z1ᵀr_{k-1} are reduced together; then, since
           * QᵀAQ = I and QᵀAZ1 = C2 (A-orthonormal window):
           *   Z2ᵀAZ2 = B1 − C2ᵀC2,   Z2ᵀr = g1 − C2ᵀ(Qᵀr_{k-1}),
           *   Z2 = Z1 − Q C2,        A Z2 = A Z1 − (AQ) C2,
           * where Qᵀr_{k-1} stacks alpha~ = W_qᵀr_{k-1} of the window blocks built in this outer
           * iteration and 0 for older blocks (r_{k-1} ⊥ the earlier search space). */
          or_spmm(A, t, Z, AZ);
          for (int q = 0; q < nq; ++q)
            or_xty(n, t, Q.AW[w0 + q], t, Z, Cb + (size_t)q * t * t);
          or_xty(n, t, Z, t, AZ, B);
          or_xty(n, t, Z, 1, r, g);
          for (int a = 0; a < t; ++a)
            for (int c = a; c < t; ++c) {
              double v = B[a * t + c];
              for (int qa = 0; qa < nq * t; ++qa) v = v - Cb[(size_t)qa * t + a] * Cb[(size_t)qa * t + c];
              B[a * t + c] = v;
            }
          for (int a = 0; a < t; ++a)
            for (int c = 0; c < a; ++c) B[a * t + c] = 0.0;
          for (int q = 0; q < nq; ++q) {
            int cur = (w0 + q) - (Q.count - i); /* position in this outer iteration, < 0: older */
            if (cur < 0) continue;
            const double* aq = alpha + (size_t)cur * t;
            for (int c = 0; c < t; ++c) {
              double v = g[c];
              for (int a = 0; a < t; ++a) v = v - Cb[((size_t)q * t + a) * t + c] * aq[a];
              g[c] = v;
            }
          }
          for (int64_t row = 0; row < n; ++row)
            for (int c = 0; c < t; ++c) {
              double dz = 0.0, daz = 0.0;
              for (int q = 0; q < nq; ++q)
                for (int a = 0; a < t; ++a) {
                  double cc = Cb[((size_t)q * t + a) * t + c];
                  dz += Q.W[w0 + q][row * t + a] * cc;
                  daz += Q.AW[w0 + q][row * t + a] * cc;
                }
              Z[row * t + c] -= dz;
              AZ[row * t + c] -= daz;
            }
          synched = 1;
        }
        if (ortho == OR_ORTHO_PRE) {
          /* Pre-CholQR's Euclidean stage on the explicit block: Z ← Z R1⁻¹ (reading R30) */
          or_xty(n, t, Z, t, Z, B);
          for (int a = 0; a < t; ++a)
            for (int c = 0; c < a; ++c) B[a * t + c] = 0.0;
          if (or_chol(t, B, R) != OR_OK) { status = OR_BREAKDOWN; free(Z); free(W); free(AZ); ok = 0; break; }
          rsolve_rows(n, t, R, Z, W);
          memcpy(Z, W, sizeof(double) * blk);
        }
        if (!synched) {
          or_spmm(A, t, Z, AZ);
          or_xty(n, t, Z, t, AZ, B);
          for (int a = 0; a < t; ++a)
            for (int c = 0; c < a; ++c) B[a * t + c] = 0.0;
          or_xty(n, t, Z, 1, r, g);
        }
        if (or_chol(t, B, R) != OR_OK) { status = OR_BREAKDOWN; free(Z); free(W); free(AZ); ok = 0; break; }
        AW = dalloc(blk);
        rsolve_rows(n, t, R, Z, W);
        rsolve_rows(n, t, R, AZ, AW);
        rtsolve_vec(t, R, g, alpha + (size_t)i * t);
        free(AZ);
      }
      free(Z);
      V[i] = W;
      AV[i] = AW;
      bl_push(&Q, W, AW);
      gblock++;
    }
    if (!ok) {
      if (rep) rep->breakdown_block = gblock;
      /* blocks already pushed belong to Q; nothing else to release here */
      break;
    }
    if (restructured) {
      /* Alg 1 / Alg 2 lines 14-17: for i = k..k+s-1,
       * alpha~ = W_iᵀ r_{i-1}, x_i = x_{i-1} + W_i alpha~, r_i = r_{i-1} − A W_i alpha~
       * (definition: A·(W_i alpha~) as one SpMV, reading R9; mirror: cached A W_i). */
      for (int i = 0; i < s; ++i) {
        double* a = alpha + (size_t)i * t;
        or_xty(n, t, V[i], 1, r, a);
        for (int64_t row = 0; row < n; ++row) {
          double acc = 0.0;
          for (int c = 0; c < t; ++c) acc += V[i][row * t + c] * a[c];
          u[row] = acc;
        }
        if (mode == OR_MODE_DEFINITION) {
          or_spmm(A, 1, u, tmp);
        } else {
          for (int64_t row = 0; row < n; ++row) {
            double acc = 0.0;
            for (int c = 0; c < t; ++c) acc += AV[i][row * t + c] * a[c];
            tmp[row] = acc;
          }
        }
        for (int64_t row = 0; row < n; ++row) { x[row] += u[row]; r[row] -= tmp[row]; }
      }
    } else if (mode == OR_MODE_DEFINITION) {
      /* alpha~ = Vᵀ r_{k-1};  x_k = x_{k-1} + V alpha~;  r_k = r_{k-1} − A V alpha~
       * (Alg 3, Alg 4, Alg 6).  Reading R9:
       * u = V alpha~ first, then r −= A·u. */
      for (int i = 0; i < s; ++i) or_xty(n, t, V[i], 1, r, alpha + (size_t)i * t);
      for (int64_t row = 0; row < n; ++row) {
        double acc = 0.0;
        for (int i = 0; i < s; ++i)
          for (int c = 0; c < t; ++c) acc += V[i][row * t + c] * alpha[(size_t)i * t + c];
        u[row] = acc;
      }
      or_spmm(A, 1, u, tmp);
      for (int64_t row = 0; row < n; ++row) { x[row] += u[row]; r[row] -= tmp[row]; }
    } else {
      for (int i = 0; i < s; ++i)
        for (int64_t row = 0; row < n; ++row) {
          double dx = 0.0, dr = 0.0;
          for (int c = 0; c < t; ++c) {
            dx += V[i][row * t + c] * alpha[(size_t)i * t + c];
            dr += AV[i][row * t + c] * alpha[(size_t)i * t + c];
          }
          x[row] += dx;
          rnew[row] -= dr;
        }
      memcpy(r, rnew, sizeof(double) * (size_t)n);
    }
    rho = norm2(n, r);  /* rho = ||r_k||_2, the recursive residual (R8) */
    if (cb) {
      int st = s * t;
      double* Vc = dalloc((size_t)n * st);
      for (int i = 0; i < s; ++i)
        for (int64_t row = 0; row < n; ++row)
          for (int c = 0; c < t; ++c) Vc[row * st + i * t + c] = V[i][row * t + c];
      cb(user, k, n, st, Vc, alpha, x, r, rho);
      free(Vc);
    }
    if (rep && rep->rho_history) rep->rho_history[k] = rho;
    k = k + 1;
    bl_trim(&Q, method);
  }

  if (rep) {
    rep->outer_iters = k - 1;
    rep->rho = rho;
    rep->converged = rho <= eps * rho0;
    or_spmm(A, 1, x, tmp);
    for (int64_t i = 0; i < n; ++i) tmp[i] = b[i] - tmp[i];
    double nb = norm2(n, b);
    rep->true_relres = nb > 0 ? norm2(n, tmp) / nb : 0.0;
  }
  if (status == OR_OK && !(rho <= eps * rho0)) status = OR_MAXITER;
  if (rep) rep->status = status;
  bl_free(&Q);
  free(V); free(AV); free(alpha); free(R); free(B); free(g); free(Cb);
  free(r); free(tmp); free(u); free(rnew);
  return status;
}

/* ------------------------------------------------------------------------ */
/* cfg5 basis sweep (reading R27): Alg 4 lines 178-188 with T(r0) replaced  */
/* by a given start block; no update, no convergence test.                   */
/* ------------------------------------------------------------------------ */
int or_basis_sweep(const or_csr* A, int t, const double* X0, int nblocks, double* W_last) {
  int64_t n = A->n;
  size_t blk = (size_t)n * t;
  double* R = dalloc((size_t)t * t);
  blist Q = {0, 0, NULL, NULL};
  int status = OR_OK;
  for (int j = 0; j < nblocks; ++j) {
    double* Z = dalloc(blk);
    if (j == 0) memcpy(Z, X0, sizeof(double) * blk);
    else or_spmm(A, t, Q.W[Q.count - 1], Z);
    int w0 = window_start(&Q, OR_SRE_CG), nq = Q.count - w0;
    if (nq > 0) or_cgs2(A, t, nq, (const double* const*)(Q.W + w0), Z, NULL, NULL);
    double* W = dalloc(blk);
    int st = or_acholqr(A, t, Z, W, R, NULL);
    free(Z);
    if (st != OR_OK) { free(W); status = st; break; }
    bl_push(&Q, W, dalloc(1));
    bl_trim(&Q, OR_SRE_CG);
  }
  if (status == OR_OK) memcpy(W_last, Q.W[Q.count - 1], sizeof(double) * blk);
  bl_free(&Q);
  free(R);
  return status;
}

/* ------------------------------------------------------------------------ */
/* Communication-avoiding variants                      */
/* ------------------------------------------------------------------------ */
/* CGS2 of the wide block V (n × zc) against nq blocks Q_j (n × t) — "A-orthonormalize V
 * against Q" of Alg 5 line 8 / Alg 7 line 9: twice
 * { AV = A·V ; C_j = Q_jᵀ AV (t × zc) ; V = V − Σ_j Q_j C_j }, the arithmetic of or_cgs2
 * column by column (for zc = t it is or_cgs2 itself). */
static void cgs2_wide(const or_csr* A, int t, int zc, int nq, const double* const* Q, double* V) {
  int64_t n = A->n;
  double* AV = dalloc((size_t)n * zc);
  double* C = dalloc((size_t)nq * t * zc);
  for (int pass = 0; pass < 2; ++pass) {
    or_spmm(A, zc, V, AV);
    for (int j = 0; j < nq; ++j) or_xty(n, t, Q[j], zc, AV, C + (size_t)j * t * zc);
    for (int64_t row = 0; row < n; ++row)
      for (int c = 0; c < zc; ++c) {
        double acc = 0.0;
        for (int j = 0; j < nq; ++j)
          for (int a = 0; a < t; ++a) acc += Q[j][row * t + a] * C[((size_t)j * t + a) * zc + c];
        V[row * zc + c] -= acc;
      }
  }
  free(AV);
  free(C);
}

/* Alg 5 / Alg 7 basis of one outer iteration into V (n × st), then the update of
 * Alg 3/4/6 lines "α̃ = Vᵀr_{k-1}; x_k = x_{k-1} + Vα̃; r_k = r_{k-1} − AVα̃".
 *   Alg 5: W_j = T(r_{k-1}) or A·W_{j-1};  V = [W_j, A W_j, …, A^{s-1} W_j];
 *                      A-orthonormalize V against Q (k > 1), then V itself.
 *   Alg 7: as Alg 5 but W_j is first A-orthonormalized against Q and itself.
 * Window Q: CA SRE-CG the last (s+1)t vectors (Alg 5 input m = (s+1)t); CA SRE-CG2 and
 * CA MSDO-CG all previous vectors (m = kst).  CA MSDO-CG seeds every iteration with
 * T(r_{k-1}) ("W_j = W_{j-1}"). */
int or_solve_ca(const or_csr* A, const double* b, double* x, int method, int arnoldi, int s, int t,
                double eps, int kmax, or_report* rep, or_iter_cb cb, void* user) {
  return or_solve_ca_pc(A, b, x, method, arnoldi, s, t, eps, kmax, NULL, rep, cb, user);
}

int or_solve_ca_pc(const or_csr* A, const double* b, double* x, int method, int arnoldi, int s, int t,
                   double eps, int kmax, const or_csr* L, or_report* rep, or_iter_cb cb, void* user) {
  int64_t n = A->n;
  if (L && L->n != n) return OR_BADARG;
  if (s < 1 || t < 1 || (int64_t)s * t > n || !(eps >= 0.0) || method < 0 || method > 2 ||
      (arnoldi != 5 && arnoldi != 7))
    return OR_BADARG;
  const int st = s * t;
  const size_t blk = (size_t)n * t, big = (size_t)n * st;
  double* r = dalloc((size_t)n);
  double* tmp = dalloc((size_t)n);
  double* u = dalloc((size_t)n);
  or_spmm(A, 1, x, tmp);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
  double rho0 = norm2(n, r), rho = rho0;
  if (rep) {
    rep->rho0 = rho0;
    rep->breakdown_block = -1;
    if (rep->rho_history) rep->rho_history[0] = rho0;
  }
  blist Q = {0, 0, NULL, NULL};
  double* W = dalloc(blk);
  double* W1 = dalloc(blk);
  double* V = dalloc(big);
  double* Vo = dalloc(big);
  double* Rt = dalloc((size_t)t * t);
  double* Rs = dalloc((size_t)st * st);
  double* alpha = dalloc((size_t)st);
  double* pw = dalloc(blk);
  double* nw = dalloc(blk);
  int status = OR_OK, k = 1;
  while (rho > eps * rho0 && k < kmax) {
    /* window: the last (s+1) blocks (CA SRE-CG) or all blocks */
    int w0 = (method == OR_SRE_CG && Q.count > s + 1) ? Q.count - (s + 1) : 0, nq = Q.count - w0;
    if (method == OR_MSDO_CG || k == 1) {
      if (L) {  /* W_{j-1} = L⁻ᵗ[T(L⁻¹ r_{k-1})] */
        or_lsolve(L, 1, r, tmp);
        or_split(n, t, tmp, W);
        or_ltsolve(L, t, W, W);
      } else {
        or_split(n, t, r, W);
      }
    } else {
      or_spmm(A, t, Q.W[Q.count - 1], W);
      if (L) { or_lsolve(L, t, W, W); or_ltsolve(L, t, W, W); }  /* M⁻¹A W_{j-1} */
    }
    if (arnoldi == 7) {  /* Alg 7 lines 1-4 */
      if (nq > 0) or_cgs2(A, t, nq, (const double* const*)(Q.W + w0), W, NULL, NULL);
      if (or_acholqr(A, t, W, W1, Rt, NULL) != OR_OK) { status = OR_BREAKDOWN; break; }
      memcpy(W, W1, sizeof(double) * blk);
    }
    /* V = [W, A W, …, A^{s-1} W] (Alg 5 lines 1-7 / Alg 7 lines 5-8) */
    memcpy(pw, W, sizeof(double) * blk);
    for (int i = 0; i < s; ++i) {
      if (i > 0) {
        or_spmm(A, t, pw, nw);
        if (L) { or_lsolve(L, t, nw, nw); or_ltsolve(L, t, nw, nw); }  /* M⁻¹A powers */
        memcpy(pw, nw, sizeof(double) * blk);
      }
      for (int64_t row = 0; row < n; ++row)
        for (int c = 0; c < t; ++c) V[row * st + i * t + c] = pw[row * t + c];
    }
    if (nq > 0) cgs2_wide(A, t, st, nq, (const double* const*)(Q.W + w0), V);
    if (or_acholqr(A, st, V, Vo, Rs, NULL) != OR_OK) { status = OR_BREAKDOWN; break; }
    /* α̃ = Vᵀ r_{k-1}; u = V α̃; x += u; r −= A u  (reading R9) */
    or_xty(n, st, Vo, 1, r, alpha);
    for (int64_t row = 0; row < n; ++row) {
      double acc = 0.0;
      for (int c = 0; c < st; ++c) acc += Vo[row * st + c] * alpha[c];
      u[row] = acc;
    }
    or_spmm(A, 1, u, tmp);
    for (int64_t row = 0; row < n; ++row) { x[row] += u[row]; r[row] -= tmp[row]; }
    rho = norm2(n, r);
    for (int i = 0; i < s; ++i) {  /* the s new blocks join Q */
      double* Wb = dalloc(blk);
      for (int64_t row = 0; row < n; ++row)
        for (int c = 0; c < t; ++c) Wb[row * t + c] = Vo[row * st + i * t + c];
      bl_push(&Q, Wb, dalloc(1));
    }
    if (method == OR_SRE_CG)
      while (Q.count > s + 1) {
        free(Q.W[0]);
        free(Q.AW[0]);
        memmove(Q.W, Q.W + 1, sizeof(double*) * (size_t)(Q.count - 1));
        memmove(Q.AW, Q.AW + 1, sizeof(double*) * (size_t)(Q.count - 1));
        Q.count--;
      }
    if (cb) cb(user, k, n, st, Vo, alpha, x, r, rho);
    if (rep && rep->rho_history) rep->rho_history[k] = rho;
    k = k + 1;
  }
  if (rep) {
    if (status == OR_BREAKDOWN) rep->breakdown_block = (k - 1) * s;
    rep->outer_iters = k - 1;
    rep->rho = rho;
    rep->converged = rho <= eps * rho0;
    or_spmm(A, 1, x, tmp);
    for (int64_t i = 0; i < n; ++i) tmp[i] = b[i] - tmp[i];
    double nb = norm2(n, b);
    rep->true_relres = nb > 0 ? norm2(n, tmp) / nb : 0.0;
  }
  if (status == OR_OK && !(rho <= eps * rho0)) status = OR_MAXITER;
  if (rep) rep->status = status;
  bl_free(&Q);
  free(W); free(W1); free(V); free(Vo); free(Rt); free(Rs); free(alpha); free(pw); free(nw);
  free(r); free(tmp); free(u);
  return status;
}

