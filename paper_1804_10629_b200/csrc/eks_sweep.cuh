// eks_sweep.cuh — DMMA + cp.async-pipelined tall-skinny sweeps (eks_sweep.cu), T ∈ {8,16,32,64}.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace eks {

constexpr int kSweepMaxBlocks = 8;
struct SweepPtrs {
  const double* q[kSweepMaxBlocks];  // update blocks Q_j (Zout = Zin − Σ_j Q_j C_j)
  const double* l[kSweepMaxBlocks];  // left blocks L_j of the partial products L_jᵀ R
};

bool sweep_supported(int t);
bool sweep_fused_supported(int t, int nq);  // fused update + coefficients fits in shared memory
// Largest number of blocks one sweep launch handles for this t (update or partial products).
int sweep_max_blocks(int t);
size_t sweep_part_stride(int t, int nl, bool v);
// Grid (= number of per-CTA partials) used by the last launch_sweep / launch_apply_tc on this thread:
// min(nblk, SMs × resident CTAs per SM), i.e. exactly one wave.
int sweep_last_grid();

// One streaming pass over the rows:
//   R = Zin − Σ_{j<nq} Q_j C_j  (nq > 0: R written to Zout; C is (nq·t)×t row-major)   else R = Zin
//   part[b] = Σ_{rows of CTA b} [L_0 … L_{nl-1}]ᵀ R  (+ L_0ᵀ vec when v)        (nl > 0)
// Supported (nq, nl): (k,0) for k ≤ sweep_max_blocks(t); (0,k) for k a power of two
// ≤ sweep_max_blocks(t); (0,1)+v; (1,1); (2,2).
cudaError_t launch_sweep(cudaStream_t st, int t, int nq, int nl, bool v, int64_t n, const double* Zin, double* Zout,
                         const SweepPtrs& P, const double* C, const double* vec, double* part, int nblk);

// Fused Y = A·X (rows [0,n), CSR with ext-indexed columns, every row ≤ spmm_gram_max_row() entries)
// and per-CTA partials of [XᵀY | Xᵀr] (layout of sweep_part_stride(t,1,true); r may be NULL).
int spmm_gram_max_row();
cudaError_t launch_spmm_gram(cudaStream_t st, int t, int64_t n, const int* rp, const int* col, const double* val,
                             const double* Xext, const double* Xloc, double* Y, const double* r, double* part,
                             int nblk);

// W = Z2·Rinv, AW = AZ2·Rinv in place + fused per-block x/r update (same contract as launch_apply).
// c1n > 0 additionally writes per-CTA partials (layout [c1n][t][t]) of the next block's CGS pass-1
// coefficients [AW_prev, AW]ᵀ AW (c1n = 2) or AWᵀAW (c1n = 1) into c1part — the SRE-CG window.
bool apply_c1_supported(int t, int c1n);
cudaError_t launch_apply_tc(cudaStream_t st, int t, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                            const double* alpha, double* x, double* dx, const double* r, double* rnew,
                            double* rho_part, const int* flag, int mode, int nblk, int c1n = 0,
                            const double* AWprev = nullptr, double* c1part = nullptr);

}  // namespace eks
