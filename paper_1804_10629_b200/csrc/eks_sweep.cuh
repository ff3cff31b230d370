// eks_sweep.cuh — DMMA + cp.async-pipelined tall-skinny sweeps (eks_sweep.cu), T ∈ {8,16,32,64}.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "eks_device.cuh"

namespace eks {

constexpr int kSweepMaxBlocks = 8;
struct SweepPtrs {
  const double* q[kSweepMaxBlocks];  // update blocks Q_j (Zout = Zin − Σ_j Q_j C_j)
  const double* l[kSweepMaxBlocks];  // left blocks L_j of the partial products L_jᵀ R
  // lazy basis blocks (W_j = Z2_j R_j⁻¹ never formed): q[j] holds Z2_j and rq[j] its R_j⁻¹ (t×t,
  // upper triangular); the sweep uses the coefficient R_j⁻¹ C_j (folded in its prologue).  NULL: q[j] is W_j.
  const double* rq[kSweepMaxBlocks];
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
// With tl.cnt set (nl > 0) the grid's last CTAs also reduce the partials into tl.out (see Tail).
cudaError_t launch_sweep(cudaStream_t st, int t, int nq, int nl, bool v, int64_t n, const double* Zin, double* Zout,
                         const SweepPtrs& P, const double* C, const double* vec, double* part, int nblk,
                         const Tail& tl = Tail{});

// Fused Y = A·X (rows [0,n), CSR with columns into Xext; row i's diagonal is column xoff+i)
// and per-CTA partials of [XᵀY | Xᵀr] (layout of sweep_part_stride(t,1,true); r may be NULL),
// reduced into tl.out (t·t + t) when tl.cnt is set; with ch.on (t ∈ {8,16}) the last CTA then
// factors B = RᵀR and writes R, R⁻¹, α̃ = R⁻ᵀ(Xᵀr) like launch_chol.
bool spmm_gram_fused_chol(int t);
// ELL copy of A for rows of ≤ 8 entries (eks_setup_csr): tiles of kEllTR rows, slot k of
// row tile·kEllTR + rr at (tile·w + k)·kEllTR + rr; padding: value 0, a valid column.
constexpr int kEllTR = 64;
int ell_width(int maxrow);  // 5, 7 or 8; 0: rows too long for the ELL path
// tmax[tile] = the largest X row (ext index) a tile gathers (drives the L2 prefetch); n_ext = rows of Xext.
cudaError_t launch_spmm_gram_ell(cudaStream_t st, int t, int64_t n, const int* ecol, const double* eval, int w,
                                 const int* tmax, int64_t n_ext, const double* Xext, int64_t xoff, double* Y,
                                 const double* r, double* part, int nblk, const Tail& tl, const CholArgs& ch);
// Segment plan of the TMA-staged SpMM+Gram (eks_setup_csr, plan tiles of kSegPT rows): per plan
// tile up to kSegMax runs of X rows (first ext row, rows), (0,0)-terminated; rows = Σ run rows;
// own = buffer row of the tile's first own row; every entry's column rewritten as a uint16 row
// of the tile's buffer: lidx holds 8 per row (16 bytes), val (w+1)&~1 per row, both row-major
// (padding: value 0, index of the row's own X row).
constexpr int kSegPT = 16, kSegMax = 8;
struct SegPlan {
  const int* seg = nullptr;              // [ntp][kSegMax][2]
  const int* rows = nullptr;             // [ntp]
  const int* own = nullptr;              // [ntp]
  const unsigned short* lidx = nullptr;  // [ntp][kSegPT][8]
  const double* val = nullptr;           // [ntp][kSegPT][(w+1)&~1]
  int cap = 0;                           // max rows of a plan tile's buffer
};
bool spmm_seg_fits(int t, int w, int cap);
cudaError_t launch_spmm_seg(cudaStream_t st, int t, int64_t n, const SegPlan& pl, int w, const double* Xext,
                            double* Y, const double* r, double* part, int nblk, const Tail& tl, const CholArgs& ch);
// Stencil-structured A (eks_grid.cu): nx × ny × nz lexicographic grid (2D: ny = 1, "planes" are
// x-lines), every entry at offset 0, ±1, ±nx (3D), ±nx·ny inside the grid; sv holds per row the
// w = 7 (3D) or 5 (2D) stencil values in ascending column order, 0 in absent slots, padded to
// (w+1)&~1 doubles per row (row-major: a line's values are one contiguous run).  (A slot-pair-major
// layout — conflict-free value loads, but VS/2 small bulk copies per line — measured 8–20 % slower.)
// Several ranks: the slab is whole planes; X points at the first LOCAL row and the ghost planes
// z = -1 (gb = 1) and z = nz (ga = 1) of the neighbouring ranks sit right before / after the local
// rows (the extended layout of eks.cu), so the kernel reads them like local planes.
struct GridPlan {
  int nx = 0, ny = 0, nz = 0, w = 0;
  int gb = 0, ga = 0;  // ghost planes before / after the local ones (0 or 1)
  const double* sv = nullptr;
};
bool spmm_grid_fits(int t, const GridPlan& gp);
// The A-CholQR Gram [XᵀY (upper 8×8 tiles, lower mirrored) | Xᵀv] as a separate sweep over X and Y
// (t ∈ {32, 64}; per-CTA partials of layout sweep_part_stride(t,1,v), tail-reduced into tl.out).
cudaError_t launch_gram_upper(cudaStream_t st, int t, int64_t n, const double* X, const double* Y, const double* v,
                              double* part, int nblk, const Tail& tl);
// Setup: stencil values per row (layout of GridPlan::sv) scattered from the uploaded CSR (int32 row
// pointers, extended-layout columns); *bad (zeroed by the caller) is set when an entry is not a stencil slot.
cudaError_t launch_grid_sv(cudaStream_t st, int64_t n, const int* rp, const int* col, const double* val,
                           int64_t row_begin, int64_t halo_before, int64_t nx, int64_t ny, int64_t b, int64_t c, int w,
                           double* sv, int* bad, int sms);
bool spmm_grid_fused_chol(int t);  // ch.on allowed: the last CTA runs the solve-path Cholesky
// gram = false: Y = A·X only (no Y scratch, no DMMA, no partials; part and tl unused) — the plain
// SpMM of the CA monomial powers, the store-Q-only CGS2 products and the residual.
cudaError_t launch_spmm_grid(cudaStream_t st, int t, const GridPlan& gp, const double* X, double* Y, const double* r,
                             double* part, int nblk, const Tail& tl, const CholArgs& ch, bool gram = true);
// maxrow = longest CSR row (selects the register-resident fast path; longer rows still work).
cudaError_t launch_spmm_gram(cudaStream_t st, int t, int64_t n, const int* rp, const int* col, const double* val,
                             int maxrow, const double* Xext, int64_t xoff, double* Y, const double* r, double* part,
                             int nblk, const Tail& tl, const CholArgs& ch);

// W = Z2·Rinv, AW = AZ2·Rinv in place + fused per-block x/r update (same contract as launch_apply).
// Per-CTA partials in `part` (stride c1n·t·t + 2): the next block's CGS pass-1 coefficients
// [AW_prev, AW]ᵀ AW (c1n = 2) or AWᵀAW (c1n = 1) — the SRE-CG window — then ‖rnew‖² (last block).
// They are reduced by the grid's tail into tl (tl.count = c1n·t·t [+1]); tl.cnt == NULL: none.
bool apply_c1_supported(int t, int c1n);
// mode bit 8 (lazy basis, SRE-CG): W = Z2·R⁻¹ is NOT written (Z2 stays the stored block); x += Z2 (R⁻¹α̃);
// with bit 4 (no x/r update) Z2 is not even read.  AW = AZ2·R⁻¹ is always formed (in place).
cudaError_t launch_apply_tc(cudaStream_t st, int t, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                            const double* alpha, double* x, double* dx, const double* r, double* rnew, const int* flag,
                            int mode, int nblk, int c1n, const double* AWprev, double* part, const Tail& tl);

}  // namespace eks
