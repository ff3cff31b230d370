/* eks.h — C ABI of libeks.so, the B200-native hot path of the s-step enlarged
 * Conjugate Gradient methods (s-step SRE-CG, SRE-CG2, MSDO-CG) of
 * arXiv:1804.10629.  Citations "P:<line>" refer to the paper's LaTeX
 * (PAPER.md), "S:<line>" to SPEC.md; readings R1..R27 are in DESIGN.md.
 *
 * Problem statement (Alg 3/4/6 inputs): solve A x = b for a
 * sparse symmetric positive definite A, given b, x0, tolerance eps, s, k_max.
 *
 * Conventions for every entry point
 *  - Return value: eks_status.  No C++ exception, abort() or exit() crosses the
 *    ABI; on failure eks_error_string() gives a one-line reason.
 *  - Pointers are plain host or device pointers as stated by the eks_mem flag of
 *    the call; sizes are element counts.  Blocks of t vectors are ROW-MAJOR
 *    (row i's t doubles contiguous).
 *  - Ownership: eks_setup_csr copies the matrix (the caller may free its arrays
 *    on return); b and x are borrowed for the duration of the call only.
 *  - All calls are synchronous with respect to the host (they return after the
 *    device work they issued has completed), and run on the context's stream
 *    (eks_set_stream; default: a stream the context creates).  The caller must
 *    synchronize its producing stream before passing device pointers.
 *  - Thread safety: one context per host thread and per rank; no global state
 *    besides the CUDA runtime and NCCL.
 */
#ifndef EKS_H
#define EKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct eks_ctx eks_ctx;

/* The three s-step methods: Alg 4, Alg 3, Alg 6. */
/* 0-2: s-step methods (Alg 4 / Alg 3 / Alg 6).  3-5: their communication-avoiding versions
 * (CA SRE-CG, CA SRE-CG2 P:245-281; CA MSDO-CG P:351): each outer iteration forms the monomial
 * block [W, AW, …, A^{s-1}W], A-orthonormalizes it against the window with CGS2 and then with ONE
 * A-CholQR of its s·t columns (s·t ≤ 640, s ≤ 12); the CA-Arnoldi variant is eks_options.arnoldi. */
typedef enum {
  EKS_SRE_CG = 0, EKS_SRE_CG2 = 1, EKS_MSDO_CG = 2,
  EKS_CA_SRE_CG = 3, EKS_CA_SRE_CG2 = 4, EKS_CA_MSDO_CG = 5
} eks_method;

typedef enum { EKS_MEM_HOST = 0, EKS_MEM_DEVICE = 1 } eks_mem;

typedef enum {
  EKS_OK = 0,
  EKS_ERR_INVALID_ARG = 1, /* s<1, t not in {1,2,4,...,64}, t>n, tol<0/NaN, NULL pointer,
                              t % nranks != 0, slab not a union of domains, nnz >= 2^31 */
  EKS_ERR_STATE = 2,       /* solve before setup, use after destroy */
  EKS_ERR_BAD_MATRIX = 3,  /* col out of range, unsorted/duplicate cols in a row, missing or <=0 diagonal */
  EKS_ERR_OOM = 4,         /* device memory exhausted; for SRE-CG2/MSDO-CG report.max_outer_fit says
                              how many outer iterations the full basis Q can hold */
  EKS_ERR_CUDA = 5,
  EKS_ERR_NCCL = 6,
  EKS_ERR_BREAKDOWN = 7,   /* A-CholQR pivot <= t*2^-52*max|B| (reading R6): x = last completed iterate */
  EKS_ERR_MAXITER = 8,     /* k_max reached with rho > tol*rho0: x = last iterate */
  EKS_ERR_NONFINITE = 9    /* the recursive residual norm rho became NaN/Inf (overflow or a corrupted
                              basis): x = the iterate of that outer iteration, the loop stops at once */
} eks_status;

/* Multi-GPU description: one process per GPU; rank r owns the contiguous row
 * slab it passes to eks_setup_csr.  nccl_id comes from eks_get_unique_id() on
 * rank 0 and is broadcast by the caller (e.g. torch.distributed). */
typedef struct {
  int rank, nranks, device;
  unsigned char nccl_id[128];
} eks_dist;

typedef struct {
  int outer_iters;        /* k_s: loop bodies executed (= k-1 at exit, reading R7) */
  int converged;          /* rho <= tol*rho0 */
  int breakdown_block;    /* -1, or global block index whose Cholesky failed */
  int max_outer_fit;      /* memory planner cap for full-Q methods (SRE-CG2/MSDO-CG), else -1 */
  double rho0, rho;       /* ||r0||_2 and final recursive ||r_k||_2 (reading R8) */
  double true_relres;     /* ||b - A x||_2 / ||b||_2, computed once at exit */
  double solve_seconds;   /* device time of the solve (CUDA events on the ctx stream) */
  double model_bytes;     /* algorithmic bytes of the whole solve (DESIGN.md byte model) */
  double model_flops;     /* algorithmic flops of the whole solve */
  int gpu_launches;       /* kernels launched by the solve */
  const double* rho_history; /* outer_iters+1 entries, owned by ctx, valid until next solve/destroy */
} eks_report;

/* Extended options; zero-initialise and set fields.  Defaults reproduce the
 * oracle's defaults (A-CholQR, k_max 5000). */
typedef struct {
  int max_outer;          /* <=0: 5000 (reading R7) */
  int use_graph;          /* 1: s-step SRE-CG on one rank (no ortho/restructured/precond/profile):
                             steady-state outer iterations (k ≥ 3) are captured once per phase of
                             their slot/pointer period as CUDA graphs and replayed (launch-bound
                             small problems); results are bitwise those of the plain path.
                             2: in addition, once every phase is captured the rest of the solve
                             is ONE graph launch: a while node (the loop test of P:146/P:177,
                             evaluated on the device by k_loop_check after each outer iteration)
                             around a switch node over the phase graphs — no host synchronisation
                             per outer iteration; falls back to 1 if the driver
                             rejects the conditional graph.  Ignored where it does not apply. */
  int profile;            /* 1: record per-kernel-class CUDA events (see eks_profile) */
  int arnoldi;            /* CA methods: 7 = modified CA-Arnoldi (Alg 7, default when 0),
                             5 = CA-Arnoldi (Alg 5) */
  int ortho;              /* self-orthonormalization of each block: 0 = A-CholQR
                             (default), 1 = Pre-CholQR (Euclidean CholQR, then A-CholQR; DESIGN
                             R30).  s-step methods only (CA methods: EKS_ERR_INVALID_ARG) */
  int restructured;       /* 1: restructured SRE-CG / SRE-CG2 (Alg 2 / Alg 1; DESIGN R31):
                             the same s blocks, then s sequential updates with α̃_i = W_iᵀ r_{i-1};
                             MSDO-CG and CA methods: EKS_ERR_INVALID_ARG */
  int precond;            /* 1: split-preconditioned s-step method (Alg 8/9/10) with the block-Jacobi
                             IC(0) M of eks_setup_precond: seed M⁻¹[T(r)], powers M⁻¹A·W.
                             With a CA method: seed M⁻¹[T(r)] and monomial powers M⁻¹A·W.
                             Restructured: EKS_ERR_INVALID_ARG */
  int aq_cache;           /* SRE-CG2 / MSDO-CG (full basis Q): 0 = auto (= off), 1 = keep A·Q
                             for every block (C = (AQ)ᵀZ, fused CGS sweeps; 2× the memory per outer
                             iteration), 2 = off: store Q only, C = Qᵀ(A·Z) with two more SpMMs per block
                             (reading R24).  report.max_outer_fit = outer iterations the device holds */
  int onesynch;           /* 1: one-synch CGS2 (DESIGN reading R36) for the s-step methods with
                             A-CholQR: the SpMM of each block runs on Z1 (after CGS pass 1) and [C2 | B1 | g1]
                             is reduced in ONE collective; B = B1 − C2ᵀC2, g = g1 − C2ᵀ(Qᵀr),
                             Z2 = Z1 − QC2, A·Z2 = A·Z1 − (AQ)C2 (QᵀAQ = I).  2 reductions per block
                             (C1, [C2|B1|g1]) + ρ²: 2s+1 collectives per outer iteration instead of 3s+1.
                             Needs A·Q (SRE-CG2/MSDO-CG: aq_cache 0 or 1); CA methods, Pre-CholQR and
                             restructured: EKS_ERR_INVALID_ARG */
  int reserved[2];
} eks_options;

/* Per-kernel-class device time accumulated while options.profile == 1. */
typedef enum {
  EKS_K_SPLIT = 0, EKS_K_SPMM = 1, EKS_K_COEF = 2, EKS_K_UPDATE = 3, EKS_K_REDUCE = 4,
  EKS_K_CHOL = 5, EKS_K_APPLY = 6, EKS_K_COMM = 7, EKS_K_OTHER = 8,
  EKS_K_UPCOEF = 9,  /* the fused CGS sweep Z1 = Z − Q·C1 with C2 = (AQ)ᵀZ1 (EKS_K_UPDATE: Z2 = Z1 − Q·C2) */
  EKS_K_NCLASSES = 10
} eks_kclass;
typedef struct {
  double ms[EKS_K_NCLASSES];      /* summed event time per class */
  long long launches[EKS_K_NCLASSES];
  double bytes[EKS_K_NCLASSES];   /* algorithmic bytes per class (DESIGN.md byte model); SpMM: 12nnz+4(n+1)+16nt */
  double flops[EKS_K_NCLASSES];   /* algorithmic flops per class */
} eks_profile;

/* rank 0 only: a fresh NCCL unique id (128 bytes) for eks_create on all ranks. */
eks_status eks_get_unique_id(unsigned char id[128]);

/* dist == NULL: single GPU (current device), no NCCL.  Creates a stream. */
eks_status eks_create(eks_ctx** out, const eks_dist* dist);

/* Use the caller's cudaStream_t (passed as void*) for all later work; NULL = own stream. */
eks_status eks_set_stream(eks_ctx* ctx, void* stream);

/* Rows [row_begin,row_end) of an n_global×n_global SPD matrix in CSR with GLOBAL
 * int32 column indices (ascending, unique within a row, diagonal present and >0).
 * row_ptr has row_end-row_begin+1 entries with row_ptr[0]==0.  Validated on the
 * host side of the copy (EKS_ERR_BAD_MATRIX).  Symmetry is assumed, not checked. */
eks_status eks_setup_csr(eks_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                         const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                         eks_mem where);

/* Block-Jacobi IC(0) preconditioner M = L·Lᵗ for the split-preconditioned s-step methods
 * (Alg 8/9/10; §5.2; DESIGN reading R32): ndomains contiguous domains
 * D_d = [floor(d n/ndomains), floor((d+1) n/ndomains)) (Metis in the paper), each diagonal block
 * factorized (kind: IC(0) or complete Cholesky) on the host at setup (a one-time cost),
 * L and Lᵗ uploaded with per-domain level schedules.  Pass the SAME local slab (global columns)
 * as eks_setup_csr; the slab must be a union of preconditioner domains.  Entries coupling two
 * domains are dropped (block Jacobi).  Errors: EKS_ERR_STATE (no eks_setup_csr), EKS_ERR_INVALID_ARG
 * (ndomains < 1, slab not a union of domains, unknown kind), EKS_ERR_BREAKDOWN (a pivot ≤ 0),
 * EKS_ERR_OOM (the Cholesky envelope exceeds 2^31 entries).
 * A solve uses it when eks_options.precond = 1; then ndomains must be a multiple of t (each of
 * the t domains is the union of ndomains/t preconditioner domains). */
typedef enum {
  EKS_PREC_IC0 = 0,  /* incomplete Cholesky with zero fill-in per block (Table 5) */
  EKS_PREC_CHOL = 1  /* complete Cholesky per block (Table 6), the fill kept in each row's envelope */
} eks_precond;
eks_status eks_setup_precond(eks_ctx* ctx, eks_precond kind, int ndomains, const int64_t* row_ptr,
                             const int32_t* col_idx, const double* vals, eks_mem where);

/* Solve A x = b with the chosen s-step method (Alg 3/4/6), t domains
 * D_d = [floor(d n/t), floor((d+1) n/t)) (reading R1), tolerance tol on the
 * recursive residual.  b, x: this rank's rows; x holds x0 on entry.
 * max_outer <= 0 means 5000.  rep may be NULL. */
eks_status eks_solve(eks_ctx* ctx, eks_method method, int s, int t, double tol,
                     const double* b, double* x, eks_mem where, int max_outer, eks_report* rep);

eks_status eks_solve_ex(eks_ctx* ctx, eks_method method, int s, int t, double tol,
                        const double* b, double* x, eks_mem where, const eks_options* opt,
                        eks_report* rep);

/* cfg5 basis-generation sweep (reading R27): A-orthonormalize the start block X0
 * (this rank's rows, n_local×t), then build nblocks-1 further blocks
 * W = A-orth(A·W_prev) against the last two blocks (Alg 4), no
 * update.  W_last (n_local×t) receives the final block.  rep->outer_iters = nblocks. */
eks_status eks_basis_sweep(eks_ctx* ctx, int t, int nblocks, const double* X0, double* W_last,
                           eks_mem where, const eks_options* opt, eks_report* rep);

/* Host-only halo plan that eks_setup_csr uses on every rank (no device, no NCCL;
 * exported so the multi-rank logic can be tested on CPUs).  Rank r owns rows
 * [ranges[2r], ranges[2r+1]) (the ranges must tile [0,n) in rank order
 * "processor i owns D_i"); row_ptr/col are its slab with GLOBAL columns.
 * Outputs: ext_col[nnz] — columns remapped to the extended layout
 * [ghost rows of lower ranks | local rows | ghost rows of higher ranks];
 * need[2*nranks] — the ghost range [lo,hi) received from each rank (0,0: none;
 * rank q therefore sends rows need_p[2q..2q+1] of its slab to rank p);
 * geom[4] — halo_before, halo_after, interior_lo, interior_hi (local rows whose
 * columns are all local, multiplied while the halo is in flight). */
eks_status eks_plan_halo(int rank, int nranks, const int64_t* ranges, const int64_t* row_ptr,
                         const int32_t* col, int32_t* ext_col, int64_t* need, int64_t* geom);

/* Host-only stencil plan that eks_setup_csr builds on every rank for the plane-marching SpMM
 * (exported so the multi-rank ghost-plane logic can be tested on CPUs).  Rows [row_begin, row_end)
 * of a 5-point (2D) / 7-point (3D) lexicographic-grid operator in CSR with GLOBAL columns; halo_before
 * and halo_after = the ghost rows eks_plan_halo gives this slab.  geom[6] = {nx, ny, nz_local, w,
 * gb, ga} (gb/ga: ghost plane before/after the local planes), all 0 when the matrix is not
 * stencil-structured or the slab is not whole planes with one-plane ghosts.  sv (may be NULL):
 * (row_end-row_begin) × ((w+1)&~1) stencil values per row in ascending column order (slots -plane,
 * -nx, -1, 0, +1, +nx, +plane; 0 where a neighbour is absent). */
eks_status eks_plan_grid(int64_t row_begin, int64_t row_end, const int64_t* row_ptr, const int32_t* col,
                         const double* vals, int64_t halo_before, int64_t halo_after, int64_t* geom, double* sv);

/* Host-only plan of the matrix-powers kernel the CA variants run on several ranks (P:1092-1097,
 * reading R37): a slab of nz planes with db / da ghost planes below / above (d = s − 1 next to a
 * neighbour rank, 0 at the grid boundary).  steps[4·(i−1) .. 4·(i−1)+3] = {zlo, zhi, gb, ga} for
 * power i = 1..d: A^i·V is computed on planes [zlo, zhi) (slab-relative, zlo = −min(db, d−i),
 * zhi = nz + min(da, d−i)) and reads one further plane below / above iff gb / ga = 1. */
eks_status eks_plan_mpk(int nz, int d, int db, int da, int* steps);

/* Kernel-class timings of the last solve/sweep run with opt.profile = 1. */
eks_status eks_get_profile(const eks_ctx* ctx, eks_profile* out);

eks_status eks_destroy(eks_ctx* ctx);             /* NULL-safe */
const char* eks_error_string(const eks_ctx* ctx); /* last error detail, owned by ctx */

#ifdef __cplusplus
}
#endif
#endif /* EKS_H */
