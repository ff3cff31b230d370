// eks_kernels.cuh — launch wrappers for the sm_100a kernels of the s-step
// enlarged CG hot path (kernels in eks_kernels.cu).  All blocks are row-major
// n×T fp64; T ∈ {1,2,4,8,16,32,64}.  Every wrapper returns the cudaError_t of
// its launch.  Citations: PAPER.md line numbers "P:<line>".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace eks {

constexpr int kThreads = 256;

// Number of CTAs of the persistent row-sweep kernels (fixed per device so that
// every fixed-order reduction is deterministic run to run).
int sweep_ctas(int sms);

// ---- (a1) T(r) — P:41: Z[i][d(i)] = r[i], zeros elsewhere, with
// d(i) = floor(((i_global+1) t - 1) / n_global) (reading R1).
cudaError_t launch_split(cudaStream_t st, int t, int64_t n_local, int64_t row0, int64_t n_global,
                         const double* r, double* Z);

// ---- (a2) SpMM Y = A·X ("W_k = AW_{k-1}") over local rows [r0, r1):
// CSR int32 row_ptr/col (col indexes the extended X with halo rows), fp64 val;
// ascending-p fma accumulation from 0.0 (bitwise equal to the oracle, R20).
cudaError_t launch_spmm(cudaStream_t st, int t, int r0, int r1, const int* rp, const int* col,
                        const double* val, const double* Xext, double* Y, int sms);

// ---- partials of Lᵀ R (nl left blocks, each n×t) and optionally L_0ᵀ v:
// part[b][j][a][c] for CTA b (nblk CTAs, contiguous row chunks).  Used for the
// CGS2 coefficients (AQ)ᵀZ (reading R24) and the Gram Z2ᵀ(AZ2)
// (A-CholQR) with Z2ᵀ r (α̃).
cudaError_t launch_tn_partials(cudaStream_t st, int t, int64_t n, int nl, const double* const* Ldev,
                               const double* R, const double* v, double* part, int nblk);
size_t tn_partials_stride(int t, int nl, bool has_v);  // doubles per CTA

// ---- fixed-order reduction out[e] = Σ_b part[b*stride + e], e < count.
cudaError_t launch_reduce(cudaStream_t st, const double* part, int nblk, size_t stride, size_t count,
                          double* out);

// ---- CGS update Zout = Zin − Σ_j Q_j C_j  (Z − Q·C; reading R3).
// C is (nq·t)×t row-major (block j = rows j·t..j·t+t-1).  Zout may alias Zin.
cudaError_t launch_ts_update(cudaStream_t st, int t, int64_t n, int nq, const double* const* Qdev,
                             const double* C, const double* Zin, double* Zout, int nblk);

// ---- small Cholesky + inverse (A-CholQR; reading R4/R6), one CTA:
// B (t×t, upper read) = RᵀR; Rinv = R⁻¹; alpha = R⁻ᵀ g (if g != nullptr);
// breakdown: atomicMin(flag, gblock) when a pivot <= t·2^-52·max|B|.
cudaError_t launch_chol(cudaStream_t st, int t, const double* B, const double* g, double* R,
                        double* Rinv, double* alpha, int* flag, int gblock);
// The solve path's Cholesky (same contract): one warp, reciprocal-square-root pivots
// (chol_warp_fast) — R agrees with launch_chol to a few ulps; t = 64 falls back to launch_chol.
cudaError_t launch_chol_fast(cudaStream_t st, int t, const double* B, const double* g, double* R,
                             double* Rinv, double* alpha, int* flag, int gblock);

// ---- apply R⁻¹ and the update (fused per block):
// W = Z2·Rinv, AW = AZ2·Rinv in place; u = W·alpha, q = AW·alpha;
// mode bit0 (first block): dx = u, rnew = r − q; else dx += u, rnew −= q;
// mode bit1 (last block): x += dx (+u) and partial ‖rnew‖² per CTA into rho_part —
// skipped when *flag != INT_MAX (breakdown in this outer iteration).
// mode bit2 (basis only): no update at all.
cudaError_t launch_apply(cudaStream_t st, int t, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                         const double* alpha, double* x, double* dx, const double* r, double* rnew,
                         double* rho_part, const int* flag, int mode, int nblk);

// ---- communication-avoiding variants (CA SRE-CG / CA SRE-CG2 / CA MSDO-CG): one CholQR of the
// s·t columns of an outer iteration (s·t ≤ kCaMax, s ≤ kCaMaxBlocks).
// st ≤ kCaMax columns per CA outer iteration (t = 64, s = 10); the st×st Cholesky runs in shared
// memory up to kCaSmem columns, in global memory (one CTA) above
constexpr int kCaMax = 640, kCaMaxBlocks = 12, kCaSmem = 118;
struct CaPtrs {
  const double* in[kCaMaxBlocks];  // combine: V_i (or AV_i);  update: W_j
  double* out[kCaMaxBlocks];       // combine: W_j (or AW_j);  update: AW_j (read)
  const int* flag;                 // breakdown flag (INT_MAX = none)
};
// Cholesky of the m×m Gram B (upper read) = RᵀR, R⁻¹, α̃ = R⁻ᵀ g (g may be NULL); breakdown as launch_chol.
// global workspace (chol_dyn_work(m) doubles) needed when m > kCaSmem
size_t chol_dyn_work(int m);
cudaError_t launch_chol_dyn(cudaStream_t st, int m, const double* B, const double* g, double* R, double* Rinv,
                            double* alpha, int* flag, int gblock,
                            double* work);
// out_j = Σ_{i ≤ j} in_i Rinv[i·t.., j·t..] for j < s (n×t blocks, row-major); optionally skipped on breakdown.
cudaError_t launch_ca_combine(cudaStream_t st, int64_t n, int t, int s, const CaPtrs& P, const double* Rinv,
                              int sms, bool skip_on_breakdown);
// x += Σ_j in_j α_j, rnew = r − Σ_j out_j α_j (in = W, out = AW), partial ‖rnew‖² per CTA into part[nblk].
// level-scheduled block-diagonal triangular solve (one CTA per domain), Y may alias Z
cudaError_t launch_trsv_lev(cudaStream_t st, int ndom, int t, const int* rp, const int* col, const double* val,
                            const double* diag, const int* dom_lev, const int* lev_ptr, const int* rows,
                            const double* Z, double* Y);
// the same with a warp per (row, column) for long rows (complete-Cholesky envelopes)
cudaError_t launch_trsv_lev_long(cudaStream_t st, int ndom, int t, const int* rp, const int* col, const double* val,
                                 const double* diag, const int* dom_lev, const int* lev_ptr, const int* rows,
                                 const double* Z, double* Y);
// the same with a shared-memory ring of wrows (power of two) solved rows and a flattened level-order
// schedule (position → row, output index, #entries ≤ E ∈ {1,2,3,4,8}, 1/diagonal, entries at pos·E + e);
// the input Zp is in schedule order (launch_perm_gather), the output goes to Y[out index]
constexpr int kTrsvMaxE = 8;
size_t trsv_ring_smem(int wrows, int t, int maxlev);
cudaError_t launch_trsv_ring(cudaStream_t st, int ndom, int t, int wrows, int maxlev, int maxrows,
                             const int* pos_row, const int* pos_out, const int* pos_ne, const double* pos_rdiag,
                             const int* pos_col, const double* pos_val, int E, const int* dom_lev, const int* lev_ptr,
                             const double* Zp, double* Y);
cudaError_t launch_perm_gather(cudaStream_t st, int64_t npos, int t, const int* pos_row, const double* Z,
                               double* Zp, int sms);
cudaError_t launch_wtv(cudaStream_t st, int64_t n, int t, const double* W, const double* v, double* part, int nblk);
cudaError_t launch_ca_pack(cudaStream_t st, int t, int s, const double* Rinv, double* pack);
cudaError_t launch_ca_update(cudaStream_t st, int64_t n, int t, int s, const CaPtrs& P, const double* alpha,
                             double* x, const double* r, double* rnew, double* part, int nblk);

// ---- one-synch CGS2 (reading R36): Bg[0..t·t) = B1 − C2ᵀC2 (symmetric), Bg[t·t..t·t+t) = g1 − Σ_{q ≥ qcur}
// C2_qᵀ α̃_q (abase = α̃ of window block qcur, contiguous per block; NULL: g = g1).  C2 is (nq·t)×t
// row-major, Bg1 = [B1 (upper read) | g1].
cudaError_t launch_onesynch_fix(cudaStream_t st, int t, int nq, int qcur, const double* C, const double* Bg1,
                                const double* abase, double* Bg);

// ---- vector kernels
// out = b − Ax (y holds A·x): r = b − y; partial Σ r² per CTA
cudaError_t launch_residual(cudaStream_t st, int64_t n, const double* b, const double* y, double* r,
                            double* part, int nblk);
// partial Σ v² per CTA
cudaError_t launch_sumsq(cudaStream_t st, int64_t n, const double* v, double* part, int nblk);

// ---- (a6) device-resident loop control (P:146/"while ρ > ε ρ0 and k < k_max"):
// the state of a steady-state solve that runs as ONE CUDA graph (a while node around a switch
// over the captured outer-iteration phases, eks_options.use_graph = 2).  After each outer
// iteration k_loop_check reads ρ² (scal[1]) and the breakdown flag, appends ρ to hist, and sets
// the while condition (ρ > thr and k < kmax and no breakdown and ρ finite) and the next phase.
struct LoopState {
  int k;        // next outer-iteration index (host's k): hist[k] receives ρ_k
  int kmax;     // k_max
  int nphase;   // phases of the captured period
  int phase;    // phase of the next iteration
  int iters;    // outer iterations executed in the graph (the breakdown one included)
  int stop;     // 0 running, 1 converged or k_max, 2 breakdown (flag in fl), 3 non-finite ρ
  int fl;       // breakdown flag value (block index baked into the phase graph)
  int pad;
  double thr;   // ε ρ0
};
cudaError_t launch_loop_check(cudaStream_t st, unsigned long long hwhile, unsigned long long hswitch,
                              LoopState* state, const double* scal, const int* flag, double* hist);

}  // namespace eks
