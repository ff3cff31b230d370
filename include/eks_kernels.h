/* eks_kernels.h — kernel-level C ABI of libeks.so, used by the parity tests and
 * by bench.py's roofline measurement.  Each call runs ONE step of the hot path
 * on the context's matrix (set by eks_setup_csr) and stream, on DEVICE
 * pointers (e.g. torch tensors' data_ptr()), single-rank contexts only
 * (EKS_ERR_INVALID_ARG when nranks > 1).  Blocks are row-major n×t fp64,
 * t ∈ {1,2,4,8,16,32,64}; n = the context's local row count.  All calls are
 * synchronous (they return after the device work completed).
 */
#ifndef EKS_KERNELS_H
#define EKS_KERNELS_H

#include "eks.h"

#ifdef __cplusplus
extern "C" {
#endif

/* (a1) Z = T(r): Z[i][d] = r[i] if row i is in domain D_d = [floor(d n/t), floor((d+1) n/t)),
 * else 0 (reading R1). */
eks_status eks_k_split(eks_ctx* ctx, int t, const double* r, double* Z);

/* (a2) Y = A·X, p-ascending fma from 0 (bitwise equal to the oracle, R20).
 * If G != NULL: G = XᵀY (t×t, full, fixed-order sums).  If v and g != NULL: g = Xᵀv (t). */
eks_status eks_k_spmm(eks_ctx* ctx, int t, const double* X, double* Y, double* G, const double* v, double* g);

/* §8(f)1 at N > 1, the matrix-powers kernel with depth-(s−1) ghost zones (reading
 * R37) on ONE GPU: planes [z0, z1) of the context's stencil operator play a rank's slab; its
 * d = s − 1 ghost planes on each side (fewer next to the grid boundary) are copied from X (n×t device,
 * the whole block) as the one exchange would deliver them, and power i = 1..d is computed on the slab
 * plus (d − i) ghost planes by the same launches the multi-rank CA outer iteration issues.
 * V (device, d × (z1−z0)·nx·ny × t) receives the slab rows of A·X, …, A^d·X — bitwise the rows of the
 * global powers.  Rows a power must not read are NaN in the scratch.  Needs the plane-marching
 * SpMM (stencil operator, t ∈ {8,16,32,64}); EKS_ERR_INVALID_ARG otherwise. */
eks_status eks_k_matrix_powers(eks_ctx* ctx, int t, int s, int z0, int z1, const double* X, double* V);

/* (a3) CGS2: twice { C = (AQ)ᵀZ ; Z = Z − Q·C } against nq window blocks (
 * readings R3, R24).  Q and AQ are HOST arrays of nq DEVICE pointers (each an n×t block,
 * AQ[j] = A·Q[j]).  Z is updated in place; C1, C2 ((nq·t)×t device, may be NULL) receive the
 * two passes' coefficients. */
eks_status eks_k_cgs2(eks_ctx* ctx, int t, int nq, const double* const* Q, const double* const* AQ,
                      double* Z, double* C1, double* C2);

/* (a4) A-CholQR of Z (reading R4): AZ = A·Z, B = Zᵀ(AZ), B = RᵀR, W = Z R⁻¹,
 * AW = (AZ) R⁻¹.  Outputs W, AW (n×t), R, B (t×t; device, B/R may be NULL).
 * Returns EKS_ERR_BREAKDOWN when a pivot <= t·2^-52·max|B| (reading R6). */
eks_status eks_k_acholqr(eks_ctx* ctx, int t, const double* Z, double* W, double* AW, double* R, double* B);

/* Cholesky alone: B (t×t device, upper triangle read) = RᵀR, R upper (device). */
eks_status eks_k_chol(eks_ctx* ctx, int t, const double* B, double* R);

/* Timing of the SpMM-block kernel on the device (bench.py's SpMM roofline and the
 * kernel micro-benchmarks): `reps` back-to-back launches of Y = A·X between two CUDA
 * events on the context stream after one warm-up launch; *ms = average per launch.
 * variant 0: plain CSR SpMM (k_spmm); 1: the fused SpMM + Gram [XᵀY | Xᵀv] kernel eks_solve
 * selects for this t, per-CTA partials only; 2: + the tail reduction of the partials (what
 * eks_solve launches); 3: + the block's Cholesky; 4: the ELL gather kernel forced; 5: the CSR
 * gather kernel forced, 6: the plane-marching stencil kernel forced (4-6 with the tail; 6 needs a
 * stencil-structured matrix), 7: exactly the step eks_solve runs (the fused kernel, or at t = 64 the
 * Gram-free plane-marching SpMM followed by the Gram sweep).  v may be NULL.  Variants 1-7 need t in
 * {8,16,32,64}. */
eks_status eks_k_time_spmm(eks_ctx* ctx, int t, const double* X, double* Y, const double* v, int variant, int reps,
                           double* ms);

/* Read back the A-orthonormal basis of the LAST eks_solve_ex / eks_basis_sweep on this context
 * (parity tests of whole outer iterations against the oracle's per-iteration V, Alg 3/4/6 lines
 * 5-11): block j (global block index, 0-based, block i of outer iteration k is j = (k-1)·s + i)
 * into W (n×t device) and, when AW != NULL, A·W into AW.  Full-basis methods keep every block;
 * SRE-CG keeps a ring of the last 3 blocks (restructured: max(3, s+1); CA SRE-CG 2s+1):
 * EKS_ERR_INVALID_ARG when block j is no longer resident or was never built. */
eks_status eks_k_last_basis(eks_ctx* ctx, int j, double* W, double* AW);

/* The recursive residual r_k (n, device) at the end of the last eks_solve_ex. */
eks_status eks_k_last_residual(eks_ctx* ctx, double* r);

#ifdef __cplusplus
}
#endif
#endif
