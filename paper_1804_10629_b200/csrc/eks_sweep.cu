// eks_sweep.cu — the tall-skinny fp64 sweeps of the hot path for T ∈ {8,16,32,64}:
//   CGS2 coefficients C = (AQ)ᵀZ, the CGS update Z − Q·C (fused with the next
//   pass's coefficients), the A-CholQR Gram Z2ᵀ(AZ2) with Z2ᵀr, and W = Z2·R⁻¹
//   fused with the x/r update.  (readings R3/R4/R24.)
//
// B200 design: each CTA owns a contiguous chunk of rows and streams TR-row tiles
// of every input block through an NS-stage shared-memory ring filled with
// 16-byte cp.async (LDGSTS) copies, so HBM stays busy while the tile in hand is
// processed.  Shared-memory rows are padded to T+4 doubles, which makes every
// fragment access below bank-conflict free.  The small dense products run on the
// fp64 tensor cores with mma.sync.m8n8k4.f64 (DMMA; tcgen05 has no fp64 kind).
// Per-CTA partial sums go to a per-CTA slot and are reduced in a fixed order
// afterwards (no fp64 atomics, bitwise reproducible).
#include "eks_device.cuh"
#include "eks_kernels.cuh"
#include "eks_sweep.cuh"

#include <climits>
#include <cstdint>
#include <cstdlib>

namespace eks {

namespace {

// 16-byte async copy global → shared; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// CTA b's rows start at a multiple of 8 (16-byte alignment of every int32/fp64 row-indexed copy).
__device__ __forceinline__ int64_t chunk_lo(int64_t n, int b, int nb) {
  return b >= nb ? n : (((int64_t)b * n / nb) & ~(int64_t)7);
}

// Copy rows [row, row+rows) of a row-major n×T block into a padded smem tile
// (row stride S doubles); rows rows..TR-1 are zero-filled.  All threads take part.
template <int T, int S, int TR>
__device__ __forceinline__ void tile_async(double* dst, const double* src, int64_t row, int rows) {
  constexpr int CPR = T / 2;  // 16-byte chunks per row
  for (int e = threadIdx.x; e < TR * CPR; e += blockDim.x) {
    const int r = e / CPR, c = (e % CPR) * 2;
    const bool ok = r < rows;
    cp16(dst + r * S + c, ok ? (const void*)(src + (row + r) * T + c) : (const void*)src, ok ? 16 : 0);
  }
}

// Copy v[row .. row+rows) (8-byte cp.async) into dst[0..TR), zero-filling the rest.
template <int TR>
__device__ __forceinline__ void vec_async(double* dst, const double* src, int64_t row, int rows) {
  for (int e = threadIdx.x; e < TR; e += blockDim.x) {
    const bool ok = e < rows;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(saddr(dst + e)),
                 "l"(ok ? (const void*)(src + row + e) : (const void*)src), "r"(ok ? 8 : 0)
                 : "memory");
  }
}

}  // namespace

// ----------------------------------------------------------------------------
// Compile-time configuration of one sweep kernel.
//   NQ: blocks in the update R = Zin − Σ_q Q_q C_q (0: R = Zin, no update; Zin == nullptr: 0)
//   NL: left blocks of the partial Lᵀ R (0: none);  V: also L_0ᵀ v
// ----------------------------------------------------------------------------
// AL: the last left block is Zin itself (SRE-CG: Z = A·W_{j−1} = AQ_last), so it is streamed
// once and R goes to a separate (unstaged) tile.
// UP (NQ = 0, NL = 1): only the upper 8×8 tiles of L_0ᵀR (the A-CholQR Gram, whose lower triangle is never
// read, reading R4), the lower ones mirrored into the partial.
template <int T, int NQ, int NL, bool V, bool AL = false, bool UP = false>
struct SwCfg {
  static constexpr int TR = (T == 8) ? 64 : 32;  // rows per tile
  static constexpr int S = T + 4;                // padded smem row stride (doubles)
  static constexpr int TILE = TR * S;            // doubles per block tile
  static constexpr int NARR = 1 + NQ + NL - (AL ? 1 : 0);  // streamed blocks
  static constexpr int STAGE = NARR * TILE + (V ? TR : 0);  // doubles per stage
  static constexpr int SC = T + 4;               // padded stride of C
  static constexpr int CDBL = NQ * T * SC + (AL ? TILE : 0);  // C, and the R tile when AL
  // Stages: as many as fit in ~100 KB (two CTAs per SM), else ~200 KB (one CTA per SM);
  // the ring keeps NS-1 tiles of every input in flight to cover HBM latency.
  static constexpr int NSA = (100 * 1024 / 8 - CDBL) / STAGE;
  static constexpr int NS0 = NSA >= 3 ? NSA : (200 * 1024 / 8 - CDBL) / STAGE;
  static constexpr int NS = NS0 > 8 ? 8 : (NS0 < 2 ? 2 : NS0);
  // update: output tiles (TR/8)×(T/8) over 8 warps
  static constexpr int UT = (TR / 8) * (T / 8);
  static constexpr int UPW = UT / 8;
  // partial products: NL·(T/8)² output tiles; WS row slices when fewer than 8
  static constexpr int MT = T / 8;
  static constexpr int OT = UP ? MT * (MT + 1) / 2 : NL * MT * MT;
  static constexpr int WS = (NL == 0) ? 1 : (OT >= 8 ? 1 : 8 / OT);
  static constexpr int TPW = (NL == 0) ? 0 : (OT >= 8 ? (OT + 7) / 8 : 1);
  static_assert(!UP || (NQ == 0 && NL == 1 && OT >= 8), "upper Gram: one left block, t >= 32");
  static constexpr int PER = NL * T * T + (V ? T : 0);  // partial doubles per CTA
  static constexpr int RED = (WS > 1 ? 8 * NL * T * T : 0) + (V ? 8 * T : 0);
  static constexpr int SMEM0 = NS * STAGE + CDBL;
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;  // doubles
  // the update's B fragments (C) held in registers when they are few (else read from sC per tile)
  static constexpr int NCF = UPW * NQ * (T / 4);
  static constexpr bool CREG = NQ > 0 && NCF <= 16;
};

// upper 8×8 tile number u (row-major over mi ≤ ni) → (mi, ni)
__device__ __forceinline__ void upper_tile(int u, int mt, int& mi, int& ni) {
  mi = 0;
  while (u >= mt - mi) {
    u -= mt - mi;
    ++mi;
  }
  ni = mi + u;
}

template <int T, int NQ, int NL, bool V, bool AL = false, bool UP = false>
__global__ void __launch_bounds__(256, 1)
    k_sweep(int64_t n, const double* Zin, double* Zout, const SweepPtrs P,
            const double* __restrict__ Cm, const double* __restrict__ v, double* __restrict__ part, const Tail tl) {
  using K = SwCfg<T, NQ, NL, V, AL, UP>;
  static_assert(!AL || (NQ > 0 && NL > 0 && !V), "alias needs an update and left blocks");
  pdl_enter();
  constexpr int S = K::S;
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + K::TR - 1) / K::TR);
  double* sC = sm + K::NS * K::STAGE;
  double* sRb = sC + NQ * T * K::SC;  // R tile (AL only)

  if constexpr (NQ > 0) {
    for (int e = tid; e < NQ * T * T; e += 256) sC[(e / T) * K::SC + e % T] = Cm[e];
    // lazy basis blocks: C_j ← R_j⁻¹ C_j (R⁻¹ upper triangular, ascending k, fma), the stage area as
    // scratch before the first tiles are issued — every CTA computes the same folded coefficients
    bool lazy = false;
#pragma unroll
    for (int j = 0; j < NQ; ++j) lazy = lazy || P.rq[j] != nullptr;
    if (lazy) {
      double* tR = sm;
      double* tO = sm + T * T;
#pragma unroll 1
      for (int j = 0; j < NQ; ++j) {
        if (P.rq[j] == nullptr) continue;
        __syncthreads();
        for (int e = tid; e < T * T; e += 256) tR[e] = P.rq[j][e];
        __syncthreads();
        for (int e = tid; e < T * T; e += 256) {
          const int i = e / T, c = e % T;
          double v = 0.0;
          for (int k = i; k < T; ++k) v = fma(tR[i * T + k], sC[(j * T + k) * K::SC + c], v);
          tO[e] = v;
        }
        __syncthreads();
        for (int e = tid; e < T * T; e += 256) sC[(j * T + e / T) * K::SC + e % T] = tO[e];
      }
      __syncthreads();
    }
  }
  double cf[K::CREG ? K::NCF : 1];
  if constexpr (K::CREG) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < K::UPW; ++u) {
      const int ni = (warp * K::UPW + u) % (T / 8);
#pragma unroll
      for (int j = 0; j < NQ; ++j)
#pragma unroll
        for (int kk = 0; kk < T; kk += 4)
          cf[(u * NQ + j) * (T / 4) + kk / 4] = sC[j * T * K::SC + (kk + q4) * K::SC + ni * 8 + g];
    }
  }

  auto issue = [&](int i) {
    if (i < ntiles) {
      const int s = i % K::NS;
      const int64_t row = lo + (int64_t)i * K::TR;
      const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
      double* st = sm + s * K::STAGE;
      if (Zin != nullptr) tile_async<T, S, K::TR>(st, Zin, row, rows);  // nullptr: R starts from 0
#pragma unroll
      for (int j = 0; j < NQ; ++j) tile_async<T, S, K::TR>(st + (1 + j) * K::TILE, P.q[j], row, rows);
#pragma unroll
      for (int j = 0; j < NL - (AL ? 1 : 0); ++j) tile_async<T, S, K::TR>(st + (1 + NQ + j) * K::TILE, P.l[j], row, rows);
      if constexpr (V) vec_async<K::TR>(st + K::NARR * K::TILE, v, row, rows);
    }
    cp_commit();
  };
#pragma unroll
  for (int i = 0; i < K::NS - 1; ++i) issue(i);

  double acc[K::TPW > 0 ? K::TPW : 1][2];
#pragma unroll
  for (int j = 0; j < (K::TPW > 0 ? K::TPW : 1); ++j) acc[j][0] = acc[j][1] = 0.0;
  double accv[2] = {0.0, 0.0};
  int umi[UP ? K::TPW : 1], uni[UP ? K::TPW : 1];  // UP: this warp's upper tiles, decoded once
  if constexpr (UP) {
#pragma unroll
    for (int u = 0; u < K::TPW; ++u) {
      const int tile = (warp / K::WS) * K::TPW + u;
      upper_tile(tile < K::OT ? tile : 0, K::MT, umi[u], uni[u]);
    }
  }

  for (int i = 0; i < ntiles; ++i) {
    cp_wait<K::NS - 2>();
    __syncthreads();  // tile i visible to all; stage (i-1)%NS free for refill
    issue(i + K::NS - 1);
    double* st = sm + (i % K::NS) * K::STAGE;
    double* sZ = st;
    const int64_t row = lo + (int64_t)i * K::TR;
    const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
    // ---------------- update: R = Zin − Σ_q Q_q C_q, written in place into sZ and to Zout
    if constexpr (NQ > 0) {
#pragma unroll
      for (int u = 0; u < K::UPW; ++u) {
        const int tile = warp * K::UPW + u;
        const int mi = tile / (T / 8), ni = tile % (T / 8);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const double* sQ = st + (1 + j) * K::TILE;
          const double* Cj = sC + j * T * K::SC;
#pragma unroll
          for (int kk = 0; kk < T; kk += 4)
            dmma(d0, d1, sQ[(mi * 8 + g) * S + kk + q4],
                 K::CREG ? cf[(u * NQ + j) * (T / 4) + kk / 4] : Cj[(kk + q4) * K::SC + ni * 8 + g]);
        }
        const int r = mi * 8 + g, c = ni * 8 + 2 * q4;
        const double z0 = (Zin != nullptr ? sZ[r * S + c] : 0.0) - d0;
        const double z1 = (Zin != nullptr ? sZ[r * S + c + 1] : 0.0) - d1;
        double* sOut = AL ? sRb : sZ;
        sOut[r * S + c] = z0;
        sOut[r * S + c + 1] = z1;
        if (r < rows) *reinterpret_cast<double2*>(Zout + (row + r) * T + c) = make_double2(z0, z1);
      }
      if constexpr (NL > 0) __syncthreads();
    }
    // ---------------- partial products Σ_rows L_lᵀ R  (+ L_0ᵀ v)
    if constexpr (NL > 0) {
      const int slice = warp % K::WS;
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = (warp / K::WS) * K::TPW + u;
        int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        if constexpr (UP) {
          if (tile >= K::OT) continue;
          l = 0;
          mi = umi[u];
          ni = uni[u];
        }
        const double* sL = (AL && l == NL - 1) ? sZ : st + (1 + NQ + l) * K::TILE;
        const double* sR = AL ? sRb : sZ;
        double d0 = acc[u][0], d1 = acc[u][1];
#pragma unroll
        for (int kk = slice * 4; kk < K::TR; kk += 4 * K::WS)
          dmma(d0, d1, sL[(kk + q4) * S + mi * 8 + g], sR[(kk + q4) * S + ni * 8 + g]);
        acc[u][0] = d0;
        acc[u][1] = d1;
      }
      if constexpr (V) {
        const double* sL0 = st + (1 + NQ) * K::TILE;
        const double* sv = st + K::NARR * K::TILE;
        for (int r = warp; r < rows; r += 8) {
          const double vr = sv[r];
          if (lane < T) accv[0] = fma(sL0[r * S + lane], vr, accv[0]);
          if (lane + 32 < T) accv[1] = fma(sL0[r * S + lane + 32], vr, accv[1]);
        }
      }
    }
  }
  cp_wait<0>();

  // ---------------- per-CTA partial → part[blockIdx.x] (fixed order)
  if constexpr (NL > 0) {
    double* out = part + (size_t)blockIdx.x * K::PER;
    double* red = sm;
    __syncthreads();  // all warps done with the stages (red reuses them)
    if constexpr (K::WS == 1) {
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = warp * K::TPW + u;
        int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        if constexpr (UP) {
          if (tile >= K::OT) continue;
          l = 0;
          upper_tile(tile, K::MT, mi, ni);
          if (mi < ni) {  // mirrored lower tile
            out[(ni * 8 + 2 * q4) * T + mi * 8 + g] = acc[u][0];
            out[(ni * 8 + 2 * q4 + 1) * T + mi * 8 + g] = acc[u][1];
          }
        }
        *reinterpret_cast<double2*>(out + l * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4) =
            make_double2(acc[u][0], acc[u][1]);
      }
    } else {
      {
        const int tile = warp / K::WS;
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        double* dst = red + (size_t)warp * NL * T * T + l * T * T;
        dst[(mi * 8 + g) * T + ni * 8 + 2 * q4] = acc[0][0];
        dst[(mi * 8 + g) * T + ni * 8 + 2 * q4 + 1] = acc[0][1];
      }
      __syncthreads();
      for (int e = tid; e < NL * T * T; e += 256) {
        const int l = e / (T * T), m = (e / T) % T, nn = e % T;
        const int tile = l * K::MT * K::MT + (m / 8) * K::MT + nn / 8;
        double s = 0.0;
        for (int w = tile * K::WS; w < tile * K::WS + K::WS; ++w) s += red[(size_t)w * NL * T * T + e];
        out[e] = s;
      }
    }
    if constexpr (V) {
      double* rv = red + (K::WS > 1 ? 8 * NL * T * T : 0);
      if (lane < T) rv[warp * T + lane] = accv[0];
      if (lane + 32 < T) rv[warp * T + lane + 32] = accv[1];
      __syncthreads();
      for (int e = tid; e < T; e += 256) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += rv[w * T + e];
        out[NL * T * T + e] = s;
      }
    }
    if (tl.cnt != nullptr) tail_reduce(part, K::PER, tl);
  }
}

// ----------------------------------------------------------------------------
// W = Z2·R⁻¹, AW = AZ2·R⁻¹ (in place) and the fused x/r update of the block
// (see launch_apply).  Same pipeline; both products on DMMA.
// ----------------------------------------------------------------------------
// ZT = false: the lazy basis without x/r update (mode bits 4 | 8): no Z2 tile and no vectors in a stage,
// so more stages fit (more bytes in flight per SM)
template <int T, int C1N, bool ZT = true>
struct ApCfg {
  static constexpr int TR = 64;  // 8 warps × 8 rows: every warp owns complete rows
  static constexpr int S = T + 4;
  static constexpr int TILE = TR * S;
  // [Z2 tile (ZT)], AZ2 tile, [AW_prev tile (C1N == 2)], [r_in, dx, x vectors (ZT)]
  static constexpr int NTL = (C1N == 2 ? 3 : 2) - (ZT ? 0 : 1);
  static constexpr int OY = ZT ? TILE : 0, OPREV = OY + TILE, VOFF = NTL * TILE;
  static constexpr int STAGE = NTL * TILE + (ZT ? 3 * TR : 0);
  static constexpr int NSA = (100 * 1024 / 8 - T * (T + 4)) / STAGE;
  static constexpr int NS0 = NSA >= 3 ? NSA : (200 * 1024 / 8 - T * (T + 4)) / STAGE;
  static constexpr int NS = NS0 > 8 ? 8 : (NS0 < 2 ? 2 : NS0);
  static constexpr int NT = T / 8;  // column tiles per row group (all in the same warp)
  // fused next-pass coefficients C1 = [AW_prev, AW]ᵀ AW: C1N·(T/8)² output tiles over 8 warps
  static constexpr int MT = T / 8;
  static constexpr int OT = C1N * MT * MT;
  static constexpr int WS = (C1N == 0) ? 1 : (OT >= 8 ? 1 : 8 / OT);
  static constexpr int TPW = (C1N == 0) ? 1 : (OT >= 8 ? OT / 8 : 1);
  // WOWN (T ≤ 16): every warp accumulates ALL C1 tiles over its own 8 rows (k-steps of 4 rows) from
  // fragments loaded once per k-step (AW column tiles serve as both operands of the AWᵀAW tiles) — no
  // CTA barrier between the R⁻¹ product and C1, ≈2.5× fewer shared loads; per-warp partials summed at the end
  static constexpr bool WOWN = T <= 32 && C1N > 0;
  static constexpr int NAW = WOWN ? (C1N == 2 ? MT * MT : 0) + MT * (MT + 1) / 2 : 0;
  static constexpr int RED = WOWN ? 8 * C1N * T * T : (WS > 1 ? 8 * C1N * T * T : 0);
  static constexpr int SMEM0 = NS * STAGE + T * (T + 4) + T;
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;
};

template <int T, int C1N, bool ZT = true>
__global__ void __launch_bounds__(256, (T <= 16 ? 2 : 1))
    k_apply_tc(int64_t n, double* Z2W, double* AZ2AW, const double* __restrict__ Rinv,
               const double* __restrict__ alpha, double* __restrict__ x, double* __restrict__ dx,
               const double* __restrict__ r, double* __restrict__ rnew, const int* __restrict__ flag, int mode,
               const double* __restrict__ AWprev, double* __restrict__ part, const Tail tl) {
  using K = ApCfg<T, C1N, ZT>;
  pdl_enter();
  constexpr int PS = C1N * T * T + 2;  // per-CTA partial: [C1 (C1N·T·T) | ‖rnew‖² | pad] (16-byte rows)
  constexpr int S = K::S, SR = T + 4;
  extern __shared__ __align__(128) double sm[];
  __shared__ double sred[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + K::TR - 1) / K::TR);
  double* sRi = sm + K::NS * K::STAGE;
  double* sA = sRi + T * SR;
  const bool first = mode & 1, last = mode & 2, basis = mode & 4, lazy = mode & 8;
  const bool skip = basis || (flag != nullptr && *flag != INT_MAX);
  for (int e = tid; e < T * T; e += 256) sRi[(e / T) * SR + e % T] = Rinv[e];
  // lazy: x += W α̃ = Z2 β with β = R⁻¹ α̃ (R⁻¹ upper triangular)
  for (int e = tid; e < T; e += 256) {
    double v = 0.0;
    if (alpha && lazy)
      for (int k = e; k < T; ++k) v = fma(Rinv[e * T + k], alpha[k], v);
    else if (alpha)
      v = alpha[e];
    sA[e] = v;
  }
  const bool zread = ZT && !(lazy && basis);  // Z2 tiles are needed for W (eager) or for x += Z2 β (lazy)
  constexpr int VOFF = K::VOFF;  // vectors after the tiles
  auto issue = [&](int i) {
    if (i < ntiles) {
      const int s = i % K::NS;
      const int64_t row = lo + (int64_t)i * K::TR;
      const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
      double* st = sm + s * K::STAGE;
      if (zread) tile_async<T, S, K::TR>(st, Z2W, row, rows);
      tile_async<T, S, K::TR>(st + K::OY, AZ2AW, row, rows);
      if constexpr (C1N == 2) tile_async<T, S, K::TR>(st + K::OPREV, AWprev, row, rows);
      if (ZT && !skip) {
        double* sv = st + VOFF;
        vec_async<K::TR>(sv, first ? r : rnew, row, rows);
        if (!first) vec_async<K::TR>(sv + K::TR, dx, row, rows);
        if (last) vec_async<K::TR>(sv + 2 * K::TR, x, row, rows);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int i = 0; i < K::NS - 1; ++i) issue(i);
  // R⁻¹ B fragments and α pairs in registers for T ≤ 16 (8 + 4 values), else from shared memory
  constexpr bool RREG = T <= 16;
  double rf[RREG ? K::NT * (T / 4) : 1], af[RREG ? 2 * K::NT : 1];
  if constexpr (RREG) {
    __syncthreads();
#pragma unroll
    for (int ni = 0; ni < K::NT; ++ni) {
#pragma unroll
      for (int kk = 0; kk < T; kk += 4) rf[ni * (T / 4) + kk / 4] = sRi[(kk + q4) * SR + ni * 8 + g];
      af[2 * ni] = sA[ni * 8 + 2 * q4];
      af[2 * ni + 1] = sA[ni * 8 + 2 * q4 + 1];
    }
  }

  double rr_acc = 0.0;
  constexpr int NACC = K::WOWN ? K::NAW : K::TPW;
  double acc[NACC][2];
#pragma unroll
  for (int u = 0; u < NACC; ++u) acc[u][0] = acc[u][1] = 0.0;
  for (int i = 0; i < ntiles; ++i) {
    cp_wait<K::NS - 2>();
    __syncthreads();
    issue(i + K::NS - 1);
    double* sZ = sm + (i % K::NS) * K::STAGE;
    double* sY = sZ + K::OY;
    const double* sv = sZ + VOFF;
    const int64_t row = lo + (int64_t)i * K::TR;
    const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
    // warp `warp` owns rows 8·warp … 8·warp+7 of the tile, all NT column tiles
    const int rr = warp * 8 + g;
    double pu = 0.0, pq = 0.0;  // row dot products with alpha, summed over column tiles in order
    double yk[K::NT][2];
#pragma unroll
    for (int ni = 0; ni < K::NT; ++ni) {
      double w0 = 0.0, w1 = 0.0, y0 = 0.0, y1 = 0.0;
      // R⁻¹ is upper triangular: rows k > 8·ni + 7 of column tile ni are exact zeros (skipped: the
      // same result, 1/4 (t = 16) to 7/16 (t = 64) fewer DMMAs)
#pragma unroll
      for (int kk = 0; kk < (T < 8 * (ni + 1) ? T : 8 * (ni + 1)); kk += 4) {
        const double b = RREG ? rf[ni * (T / 4) + kk / 4] : sRi[(kk + q4) * SR + ni * 8 + g];
        if (ZT && !lazy) dmma(w0, w1, sZ[rr * S + kk + q4], b);
        dmma(y0, y1, sY[rr * S + kk + q4], b);
      }
      const int c = ni * 8 + 2 * q4;
      if (ZT && lazy && zread) {  // the x update multiplies Z2 by β (no W)
        w0 = sZ[rr * S + c];
        w1 = sZ[rr * S + c + 1];
      }
      if (rr < rows) {
        if (ZT && !lazy) *reinterpret_cast<double2*>(Z2W + (row + rr) * T + c) = make_double2(w0, w1);
        *reinterpret_cast<double2*>(AZ2AW + (row + rr) * T + c) = make_double2(y0, y1);
      }
      yk[ni][0] = y0;
      yk[ni][1] = y1;
      if (!skip) {  // (warp-uniform) the row products with α̃ / β of the x and r updates
        const double a0 = RREG ? af[2 * ni] : sA[c], a1 = RREG ? af[2 * ni + 1] : sA[c + 1];
        // r −= AW α̃; lazy: a = β = R⁻¹α̃, so the residual update takes AZ2 (the sY tile, still unchanged) · β
        const double q0 = lazy ? sY[rr * S + c] : y0, q1 = lazy ? sY[rr * S + c + 1] : y1;
        double tu = fma(w0, a0, w1 * a1);
        double tq = fma(q0, a0, q1 * a1);
        tu += __shfl_xor_sync(0xffffffffu, tu, 1);
        tq += __shfl_xor_sync(0xffffffffu, tq, 1);
        tu += __shfl_xor_sync(0xffffffffu, tu, 2);
        tq += __shfl_xor_sync(0xffffffffu, tq, 2);
        pu += tu;
        pq += tq;
      }
    }
    if (!skip && q4 == 0 && rr < rows) {
      const int64_t rg = row + rr;
      const double dxi = first ? pu : sv[K::TR + rr] + pu;
      const double rn = sv[rr] - pq;
      rnew[rg] = rn;
      if (last) {
        x[rg] = sv[2 * K::TR + rr] + dxi;
        rr_acc = fma(rn, rn, rr_acc);
      } else {
        dx[rg] = dxi;
      }
    }
    if constexpr (C1N > 0) {
      // AW tile replaces the AZ2 tile in place (each warp owns its rows), then
      // C1 partial += [AW_prev, AW]ᵀ AW over the tile (next block's CGS pass 1)
#pragma unroll
      for (int ni = 0; ni < K::NT; ++ni) {
        sY[rr * S + ni * 8 + 2 * q4] = yk[ni][0];
        sY[rr * S + ni * 8 + 2 * q4 + 1] = yk[ni][1];
      }
      if constexpr (K::WOWN) {
        __syncwarp();  // the warp's own rows only
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int kr = warp * 8 + ks * 4 + q4;
          double fa[K::MT], fp[K::MT];
#pragma unroll
          for (int i2 = 0; i2 < K::MT; ++i2) {
            fa[i2] = sY[kr * S + i2 * 8 + g];
            fp[i2] = C1N == 2 ? sZ[K::OPREV + kr * S + i2 * 8 + g] : 0.0;
          }
          int u = 0;
          if constexpr (C1N == 2) {
#pragma unroll
            for (int mi = 0; mi < K::MT; ++mi)
#pragma unroll
              for (int ni = 0; ni < K::MT; ++ni, ++u) dmma(acc[u][0], acc[u][1], fp[mi], fa[ni]);
          }
#pragma unroll
          for (int mi = 0; mi < K::MT; ++mi)
#pragma unroll
            for (int ni = mi; ni < K::MT; ++ni, ++u) dmma(acc[u][0], acc[u][1], fa[mi], fa[ni]);
        }
        continue;
      }
      __syncthreads();
      const int slice = warp % K::WS;
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = (warp / K::WS) * K::TPW + u;
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        if (K::WS == 1 && l == C1N - 1 && mi > ni) continue;  // AWᵀAW is symmetric: upper tiles, mirrored below
        const double* sL = (C1N == 2 && l == 0) ? sZ + K::OPREV : sY;
        double d0 = acc[u][0], d1 = acc[u][1];
#pragma unroll
        for (int kk = slice * 4; kk < K::TR; kk += 4 * K::WS)
          dmma(d0, d1, sL[(kk + q4) * S + mi * 8 + g], sY[(kk + q4) * S + ni * 8 + g]);
        acc[u][0] = d0;
        acc[u][1] = d1;
      }
    }
  }
  cp_wait<0>();
  if (tl.cnt == nullptr) return;  // nothing to reduce (no fused C1, not the last block)
  if (last) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rr_acc += __shfl_down_sync(0xffffffffu, rr_acc, o);
    if (lane == 0) sred[warp] = rr_acc;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < 8; ++w) sacc += sred[w];
      part[(size_t)blockIdx.x * PS + C1N * T * T] = sacc;
    }
  }
  if constexpr (C1N > 0) {
    double* out = part + (size_t)blockIdx.x * PS;
    __syncthreads();
    if constexpr (K::WOWN) {  // per-warp partials (lower half of AWᵀAW mirrored), summed in warp order
      double* red = sm;
      double* dst = red + (size_t)warp * C1N * T * T;
      int u = 0;
      if constexpr (C1N == 2) {
#pragma unroll
        for (int mi = 0; mi < K::MT; ++mi)
#pragma unroll
          for (int ni = 0; ni < K::MT; ++ni, ++u)
            *reinterpret_cast<double2*>(dst + (mi * 8 + g) * T + ni * 8 + 2 * q4) = make_double2(acc[u][0], acc[u][1]);
      }
      double* d1 = dst + (C1N - 1) * T * T;
#pragma unroll
      for (int mi = 0; mi < K::MT; ++mi)
#pragma unroll
        for (int ni = mi; ni < K::MT; ++ni, ++u) {
          *reinterpret_cast<double2*>(d1 + (mi * 8 + g) * T + ni * 8 + 2 * q4) = make_double2(acc[u][0], acc[u][1]);
          if (mi < ni) {
            d1[(ni * 8 + 2 * q4) * T + mi * 8 + g] = acc[u][0];
            d1[(ni * 8 + 2 * q4 + 1) * T + mi * 8 + g] = acc[u][1];
          }
        }
      __syncthreads();
      for (int e = tid; e < C1N * T * T; e += 256) {
        double sacc = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc += red[(size_t)w * C1N * T * T + e];
        out[e] = sacc;
      }
    } else if constexpr (K::WS == 1) {
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = warp * K::TPW + u;
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        if (l == C1N - 1 && mi > ni) continue;  // written by its mirror tile
        if (l == C1N - 1 && mi < ni) {
          out[l * T * T + (ni * 8 + 2 * q4) * T + mi * 8 + g] = acc[u][0];
          out[l * T * T + (ni * 8 + 2 * q4 + 1) * T + mi * 8 + g] = acc[u][1];
        }
        *reinterpret_cast<double2*>(out + l * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4) =
            make_double2(acc[u][0], acc[u][1]);
      }
    } else {
      double* red = sm;
      {
        const int tile = warp / K::WS;
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        double* dst = red + (size_t)warp * C1N * T * T + l * T * T;
        dst[(mi * 8 + g) * T + ni * 8 + 2 * q4] = acc[0][0];
        dst[(mi * 8 + g) * T + ni * 8 + 2 * q4 + 1] = acc[0][1];
      }
      __syncthreads();
      for (int e = tid; e < C1N * T * T; e += 256) {
        const int l = e / (T * T), m = (e / T) % T, nn = e % T;
        const int tile = l * K::MT * K::MT + (m / 8) * K::MT + nn / 8;
        double sacc = 0.0;
        for (int w = tile * K::WS; w < tile * K::WS + K::WS; ++w) sacc += red[(size_t)w * C1N * T * T + e];
        out[e] = sacc;
      }
    }
  }
  tail_reduce(part, PS, tl);
}

// ----------------------------------------------------------------------------
// Epilogue of the fused SpMM+Gram kernels: the CTA's partial [XᵀY | Xᵀr] (layout
// of k_sweep<T,0,1,true>), the tail reduction into tl.out and, for T ≤ 16 on one
// rank, the Cholesky of the reduced Gram by the last CTA (chol_warp, registers).
// ----------------------------------------------------------------------------
template <int T, int MT, int WS, int TPW, int NW = 8>
__device__ __forceinline__ void gram_epilogue(double* part, const double (&acc)[TPW][2], const double (&accv)[2],
                                              double* sm, const Tail& tl, const CholArgs& ch, bool has_r) {
  constexpr int PER = T * T + T, NT = NW * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  double* out = part + (size_t)blockIdx.x * PER;
  double* red = sm;
  if constexpr (WS == 1) {
#pragma unroll
    for (int uu = 0; uu < TPW; ++uu) {
      const int ot = warp * TPW + uu;
      const int mi = ot / MT, ni = ot % MT;
      *reinterpret_cast<double2*>(out + (mi * 8 + g) * T + ni * 8 + 2 * q4) = make_double2(acc[uu][0], acc[uu][1]);
    }
  } else {
    {
      const int ot = warp / WS;
      const int mi = ot / MT, ni = ot % MT;
      red[(size_t)warp * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4] = acc[0][0];
      red[(size_t)warp * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4 + 1] = acc[0][1];
    }
    __syncthreads();
    for (int e = tid; e < T * T; e += NT) {
      const int m = e / T, nn = e % T;
      const int ot = (m / 8) * MT + nn / 8;
      double s = 0.0;
      for (int w = ot * WS; w < ot * WS + WS; ++w) s += red[(size_t)w * T * T + e];
      out[e] = s;
    }
  }
  double* rv = red + (WS > 1 ? NW * T * T : 0);
  if (lane < T) rv[warp * T + lane] = accv[0];
  if (lane + 32 < T) rv[warp * T + lane + 32] = accv[1];
  __syncthreads();
  for (int e = tid; e < T; e += NT) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += rv[w * T + e];
    out[T * T + e] = s;
  }
  if (tl.cnt != nullptr) {
    const bool last = tail_reduce(part, PER, tl);
    if constexpr (T <= 16) {
      if (last && ch.on && warp == 0)
        chol_warp<T>(tl.out, has_r ? tl.out + T * T : nullptr, ch.R, ch.Rinv, ch.alpha, ch.flag, ch.gblock);
    }
  }
}

// ----------------------------------------------------------------------------
// Fused SpMM + Gram (A-CholQR's B = Z2ᵀ(A Z2) and Z2ᵀr; Y = A·X).
// Tiles of TR rows are dealt round-robin to the CTAs (tile = blockIdx + k·grid), so
// at any moment the whole grid works on one contiguous window of rows and the
// stencil neighbours of X (rows ±1, ±N, ±N²) are re-read from L2 rather than HBM.
// G = T/2 threads per row, each owning 2 columns (16-byte gathers of the row-major
// X rows).  A tile is processed in PASSES units of RPP rows; a unit's (col, val)
// entries are loaded cooperatively, one entry per lane (SL slots per lane), and
// handed out by shuffles.  Software pipeline over units: while unit u's X gathers
// are in flight, the entries of unit u+1 and the row pointers of unit u+2 are
// loaded, so the gathers are the only exposed latency.  The diagonal entry's
// gather is the row's own X row (every row has a diagonal, checked at setup): the
// Gram needs no extra read of X.  The tile's X and Y rows are kept in shared memory
// and XᵀY, Xᵀr accumulate on DMMA.  Accumulation order of every Y entry: p
// ascending, fma from 0.0 — bitwise equal to k_spmm and to the oracle (R20).  Rows
// longer than NZ take a plain loop.  The per-CTA partials are reduced by the grid's
// last CTAs (Tail) and, on one rank, the very last CTA factors B = RᵀR (T ≤ 16).
// ----------------------------------------------------------------------------
template <int T, int NZ>
struct SgCfg {
  static constexpr int TR = 64;
  static constexpr int S = T + 4;
  static constexpr int G = T / 2;       // threads per row (2 columns each)
  static constexpr int RPP = 256 / G;    // rows per unit
  static constexpr int PASSES = TR / RPP;
  static constexpr int SL = (NZ + G - 1) / G;  // (col, val) slots per lane
  static constexpr int MT = T / 8;
  static constexpr int OT = MT * MT;
  static constexpr int WS = OT >= 8 ? 1 : 8 / OT;
  static constexpr int TPW = OT >= 8 ? OT / 8 : 1;
  static constexpr int PER = T * T + T;
  static constexpr int RED = (WS > 1 ? 8 * T * T : 0) + 8 * T;
  static constexpr int SMEM0 = 2 * TR * S + TR;
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;
};

template <int T, int NZ>
__global__ void __launch_bounds__(256, (T >= 64 ? 2 : 3))
    k_spmm_gram(int64_t n, const int* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                const double* __restrict__ Xext, int64_t xoff, double* __restrict__ Y, const double* __restrict__ r,
                double* __restrict__ part, const Tail tl, const CholArgs ch) {
  using K = SgCfg<T, NZ>;
  pdl_enter();
  constexpr int S = K::S, G = K::G, SL = K::SL, P = K::PASSES, RPP = K::RPP;
  extern __shared__ __align__(128) double sm[];
  double* sX = sm;
  double* sY = sm + K::TR * S;
  double* sr = sm + 2 * K::TR * S;
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int grp = tid / G, gl = tid % G;
  const int64_t ntiles = (n + K::TR - 1) / K::TR;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nunits = my_tiles * P;
  // global row of this thread in unit u (may be >= n)
  auto row_of = [&](int64_t u) { return (blockIdx.x + (u / P) * gridDim.x) * K::TR + (u % P) * RPP + grp; };
  auto load_rp = [&](int64_t u, int& p0, int& len) {
    p0 = 0;
    len = 0;
    const int64_t i = row_of(u);
    if (u < nunits && i < n) {
      p0 = __ldg(rp + i);
      len = __ldg(rp + i + 1) - p0;
    }
  };
  auto load_cv = [&](int p0, int len, int (&c)[SL], double (&v)[SL]) {
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int k = s * G + gl;
      c[s] = 0;
      v[s] = 0.0;
      if (k < len && k < NZ) {
        c[s] = __ldg(col + p0 + k);
        v[s] = __ldg(val + p0 + k);
      }
    }
  };

  double acc[K::TPW][2];
#pragma unroll
  for (int j = 0; j < K::TPW; ++j) acc[j][0] = acc[j][1] = 0.0;
  double accv[2] = {0.0, 0.0};

  // pipeline state: unit u (entries ready), unit u+1 (row pointers ready)
  int p0c, lenc, p0n, lenn, cc[SL];
  double cv[SL];
  load_rp(0, p0c, lenc);
  load_rp(1, p0n, lenn);
  load_cv(p0c, lenc, cc, cv);
  for (int64_t u = 0; u < nunits; ++u) {
    const int ps = (int)(u % P);
    const int64_t tile = blockIdx.x + (u / P) * gridDim.x;
    const int64_t row0 = tile * K::TR;
    const int rr = ps * RPP + grp;
    const int64_t i = row0 + rr;
    int p0nn, lennn, cn[SL];
    double vn[SL];
    load_rp(u + 2, p0nn, lennn);
    double2 y = make_double2(0.0, 0.0), xd = make_double2(0.0, 0.0);
    if (__all_sync(FULL, lenc <= NZ)) {
      const int dcol = (int)(xoff + i);
      double2 xv[NZ];
      unsigned dm = 0;  // bit k: entry k is the diagonal
#pragma unroll
      for (int k = 0; k < NZ; ++k) {
        const int c = __shfl_sync(FULL, cc[k / G], k % G, G);
        dm |= (c == dcol ? 1u : 0u) << k;
        if (k < lenc) xv[k] = __ldg(reinterpret_cast<const double2*>(Xext + (int64_t)c * T) + gl);
      }
      load_cv(p0n, lenn, cn, vn);  // next unit's entries, behind this unit's gathers
#pragma unroll
      for (int k = 0; k < NZ; ++k) {
        const double a = __shfl_sync(FULL, cv[k / G], k % G, G);
        if (k < lenc) {
          y.x = __fma_rn(a, xv[k].x, y.x);
          y.y = __fma_rn(a, xv[k].y, y.y);
          if ((dm >> k) & 1u) xd = xv[k];
        }
      }
    } else {
      load_cv(p0n, lenn, cn, vn);
      const int dcol = (int)(xoff + i);
      for (int p = p0c; p < p0c + lenc; ++p) {  // long rows: plain loop, same order
        const int c = __ldg(col + p);
        const double2 xv = __ldg(reinterpret_cast<const double2*>(Xext + (int64_t)c * T) + gl);
        const double a = __ldg(val + p);
        y.x = __fma_rn(a, xv.x, y.x);
        y.y = __fma_rn(a, xv.y, y.y);
        if (c == dcol) xd = xv;
      }
    }
    if (i < n) *reinterpret_cast<double2*>(Y + i * T + 2 * gl) = y;
    *reinterpret_cast<double2*>(sY + rr * S + 2 * gl) = y;  // rows beyond the end stay 0 in the Gram
    *reinterpret_cast<double2*>(sX + rr * S + 2 * gl) = xd;
    p0c = p0n;
    lenc = lenn;
    p0n = p0nn;
    lenn = lennn;
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      cc[s] = cn[s];
      cv[s] = vn[s];
    }
    if (ps == P - 1) {
      // ---------------- Gram partial Xᵀ Y and Xᵀ r of the tile
      const int rows = (int)((n - row0) < K::TR ? (n - row0) : K::TR);
      if (r != nullptr)
        for (int e = tid; e < K::TR; e += 256) sr[e] = e < rows ? __ldg(r + row0 + e) : 0.0;
      __syncthreads();
      const int slice = warp % K::WS;
#pragma unroll
      for (int uu = 0; uu < K::TPW; ++uu) {
        const int ot = (warp / K::WS) * K::TPW + uu;
        const int mi = ot / K::MT, ni = ot % K::MT;
        double d0 = acc[uu][0], d1 = acc[uu][1];
#pragma unroll
        for (int kk = slice * 4; kk < K::TR; kk += 4 * K::WS)
          dmma(d0, d1, sX[(kk + q4) * S + mi * 8 + g], sY[(kk + q4) * S + ni * 8 + g]);
        acc[uu][0] = d0;
        acc[uu][1] = d1;
      }
      if (r != nullptr)
        for (int q = warp; q < rows; q += 8) {
          const double vr = sr[q];
          if (lane < T) accv[0] = fma(sX[q * S + lane], vr, accv[0]);
          if (lane + 32 < T) accv[1] = fma(sX[q * S + lane + 32], vr, accv[1]);
        }
      __syncthreads();
    }
  }
  gram_epilogue<T, K::MT, K::WS, K::TPW>(part, acc, accv, sm, tl, ch, r != nullptr);
}

// ----------------------------------------------------------------------------
// The same fused SpMM + Gram on the ELL copy of A that eks_setup_csr builds when
// every row has ≤ 8 entries (all stencil operators): tiles of kEllTR = 64 rows,
// slot k of row tile·64 + rr at index (tile·W + k)·64 + rr, padded slots holding
// value 0 and a valid column.  Every address is computed, not loaded; no
// predication, no shuffles.  Tiles are dealt round-robin to the CTAs so the grid
// sweeps one window of rows (far neighbours ±N² are L2 hits, A and X leave HBM
// once).  The tile's own X rows are streamed into shared memory with cp.async one
// tile ahead (double buffer); entries whose column falls inside the tile (the
// diagonal and the ±1 neighbours of a stencil) read that copy, only the others are
// 16-byte global gathers — and that copy is also the X of the Gram.  The columns of
// the next unit are loaded while this unit's gathers are in flight.  Padded slots
// add fma(0, x, y) = y exactly (y is never −0 from a +0 start), so Y stays bitwise
// equal to the ascending-p CSR accumulation (R20).
// ----------------------------------------------------------------------------
template <int T, int W>
struct SeCfg {
  static constexpr int TR = kEllTR;
  static constexpr int S = T + 4;
  static constexpr int G = T / 2;       // threads per row (2 columns each)
  static constexpr int RPP = 256 / G;    // rows per unit
  static constexpr int PASSES = TR / RPP;
  static constexpr int MT = T / 8;
  static constexpr int OT = MT * MT;
  static constexpr int WS = OT >= 8 ? 1 : 8 / OT;
  static constexpr int TPW = OT >= 8 ? OT / 8 : 1;
  static constexpr int RED = (WS > 1 ? 8 * T * T : 0) + 8 * T;
  static constexpr int SMEM0 = 3 * TR * S + TR;  // 2 X tiles, Y tile, r
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;
};

template <int T, int W, int MINB = (T >= 64 ? 2 : 3)>
__global__ void __launch_bounds__(256, MINB)
    k_spmm_gram_ell(int64_t n, const int* __restrict__ ecol, const double* __restrict__ eval,
                    const double* __restrict__ Xext, int64_t xoff, double* __restrict__ Y,
                    const double* __restrict__ r, double* __restrict__ part, const Tail tl, const CholArgs ch) {
  using K = SeCfg<T, W>;
  pdl_enter();
  constexpr int S = K::S, G = K::G, P = K::PASSES, RPP = K::RPP, TR = K::TR, H = T / 2;
  extern __shared__ __align__(128) double sm[];
  double* sY = sm + 2 * TR * S;
  double* sr = sm + 3 * TR * S;
  const double2* __restrict__ X2 = reinterpret_cast<const double2*>(Xext);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int grp = tid / G, gl = tid % G;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto load_xtile = [&](int64_t tile, double* dst) {  // own X rows of a tile, zero-filled past n
    const int64_t row0 = tile * TR;
    const int rows = (int)((n - row0) < TR ? (n - row0) : TR);
    for (int e = tid; e < TR * H; e += 256) {
      const int q = e / H, c = (e % H) * 2;
      const bool ok = q < rows;
      cp16(dst + q * S + c, ok ? (const void*)(Xext + (xoff + row0 + q) * T + c) : (const void*)Xext, ok ? 16 : 0);
    }
    cp_commit();
  };

  double acc[K::TPW][2];
#pragma unroll
  for (int j = 0; j < K::TPW; ++j) acc[j][0] = acc[j][1] = 0.0;
  double accv[2] = {0.0, 0.0};

  int cc[W];
#pragma unroll
  for (int k = 0; k < W; ++k) cc[k] = 0;
  if (my_tiles > 0) {
    const int64_t e = (int64_t)blockIdx.x * (TR * W) + grp;
#pragma unroll
    for (int k = 0; k < W; ++k) cc[k] = __ldg(ecol + e + k * TR);
    load_xtile(blockIdx.x, sm);
  }
  for (int64_t j = 0; j < my_tiles; ++j) {
    const int64_t tile = blockIdx.x + j * gridDim.x;
    const int64_t row0 = tile * TR, xrow0 = xoff + row0;
    const int rows = (int)((n - row0) < TR ? (n - row0) : TR);
    const bool more = j + 1 < my_tiles;
    double* sX = sm + (j & 1) * TR * S;
    if (more) load_xtile(tile + gridDim.x, sm + ((j + 1) & 1) * TR * S);
    else cp_commit();
    cp_wait<1>();     // this tile's X rows have landed
    __syncthreads();  // … and are visible to every thread
#pragma unroll
    for (int ps = 0; ps < P; ++ps) {
      const int rr = ps * RPP + grp;
      const int64_t i = row0 + rr;
      const int64_t e = tile * (TR * W) + rr;
      double2 xv[W];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int64_t lc = (int64_t)cc[k] - xrow0;
        if ((uint64_t)lc < (uint64_t)TR) xv[k] = *reinterpret_cast<const double2*>(sX + lc * S + 2 * gl);
        else xv[k] = __ldg(X2 + (int64_t)cc[k] * H + gl);
      }
      double a[W];
#pragma unroll
      for (int k = 0; k < W; ++k) a[k] = __ldg(eval + e + k * TR);
      if (ps + 1 < P || more) {  // next unit's columns, behind this unit's gathers
        const int64_t e1 = ps + 1 < P ? e + RPP : (tile + gridDim.x) * (TR * W) + grp;
#pragma unroll
        for (int k = 0; k < W; ++k) cc[k] = __ldg(ecol + e1 + k * TR);
      }
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < W; ++k) {
        y.x = __fma_rn(a[k], xv[k].x, y.x);
        y.y = __fma_rn(a[k], xv[k].y, y.y);
      }
      if (i < n) reinterpret_cast<double2*>(Y)[i * H + gl] = y;
      *reinterpret_cast<double2*>(sY + rr * S + 2 * gl) = y;  // padded rows are 0 in the Gram
    }
    // ---------------- Gram partial Xᵀ Y and Xᵀ r of the tile
    if (r != nullptr)
      for (int q = tid; q < TR; q += 256) sr[q] = q < rows ? __ldg(r + row0 + q) : 0.0;
    __syncthreads();
    const int slice = warp % K::WS;
#pragma unroll
    for (int uu = 0; uu < K::TPW; ++uu) {
      const int ot = (warp / K::WS) * K::TPW + uu;
      const int mi = ot / K::MT, ni = ot % K::MT;
      double d0 = acc[uu][0], d1 = acc[uu][1];
#pragma unroll
      for (int kk = slice * 4; kk < TR; kk += 4 * K::WS)
        dmma(d0, d1, sX[(kk + q4) * S + mi * 8 + g], sY[(kk + q4) * S + ni * 8 + g]);
      acc[uu][0] = d0;
      acc[uu][1] = d1;
    }
    if (r != nullptr)
      for (int q = warp; q < rows; q += 8) {
        const double vr = sr[q];
        if (lane < T) accv[0] = fma(sX[q * S + lane], vr, accv[0]);
        if (lane + 32 < T) accv[1] = fma(sX[q * S + lane + 32], vr, accv[1]);
      }
    __syncthreads();  // sX / sY / sr are rewritten by the next tile
  }
  cp_wait<0>();
  gram_epilogue<T, K::MT, K::WS, K::TPW>(part, acc, accv, sm, tl, ch, r != nullptr);
}

// ----------------------------------------------------------------------------
// Segment-staged fused SpMM + Gram (TMA bulk copies + mbarrier ring).
// eks_setup_csr plans, for every 16-row plan tile, the few contiguous runs of X
// rows ("segments") its entries reference — for a stencil: the tile's own rows
// with the ±1 halo, and the slabs at ±N (and ±N²) — and rewrites every entry's
// column as a row index into the concatenation of those segments (uint16).  A CTA
// (one per SM, persistent) then streams macro tiles of M plan tiles: one elected
// thread issues cp.async.bulk copies of the macro tile's values, local indices and
// X segments into a stage of an NS-deep shared-memory ring, completing on that
// stage's mbarrier; all 8 warps multiply out of shared memory.  Nothing in flight
// occupies registers, so the ring keeps ~(NS−1)·40 KB per SM in flight and the
// kernel streams at the L2/HBM limit instead of the gather latency limit.  Each Y
// entry is accumulated in the ELL order (p ascending, padded slots add fma(0,x,y)
// = y), bitwise equal to the oracle (R20); the Gram/α̃ epilogue is the same as
// the other SpMM+Gram kernels.
// ----------------------------------------------------------------------------
template <int T>
struct SsCfg {
  static constexpr int NWC = T <= 16 ? 16 : 8, NTH = 32 * (NWC + 1);  // consumer warps + 1 producer warp
  static constexpr int M = T == 8 ? 8 : (T == 16 ? 4 : 2);  // plan tiles per macro tile (~40-80 KB of X)
  static constexpr int TR = kSegPT * M;                      // rows per macro tile
  static constexpr int RW = T == 8 ? 8 : 4;                  // rows per warp unit (= DMMA k-steps × 4)
  static constexpr int G = 32 / RW;                          // threads per row
  static constexpr int C = T / G;                            // columns per thread (2, 2, 4, 8)
  static constexpr int U = TR / RW;                          // units per macro tile
  static constexpr int UPW = U / NWC;                        // units per consumer warp per macro tile
  static constexpr int S = T + 4;                            // row stride of the per-warp Y scratch
  static constexpr int MT = T / 8;
  static constexpr int NUT = MT * (MT + 1) / 2;              // upper-triangular 8×8 output tiles
  static_assert(U % NWC == 0 && kSegPT % RW == 0, "tile shape");
};
__host__ __device__ constexpr int seg_vs(int w) { return (w + 1) & ~1; }  // value slots per row (16-byte rows)

// Bytes of one ring stage: X segments of M plan tiles (`cap` rows each), values (VS per
// row), local indices (8 × uint16 per row), own-row offsets, r — 128-byte aligned.
template <int T, int W>
__host__ __device__ constexpr size_t seg_stage_bytes(int cap) {
  using K = SsCfg<T>;
  return ((size_t)K::M * cap * T * 8 + (size_t)K::TR * seg_vs(W) * 8 + (size_t)K::TR * 16 + 16 * K::M +
          (size_t)K::TR * 8 + 127) &
         ~(size_t)127;
}
template <int T>
__host__ __device__ constexpr size_t seg_fixed_bytes() {
  using K = SsCfg<T>;
  return (size_t)K::NWC * K::RW * K::S * 8 + 16 * 8 + 128;  // per-warp Y scratch, mbarriers, slack
}
constexpr size_t kSegSmem = 220 * 1024;

template <int T, int W>
__global__ void __launch_bounds__(SsCfg<T>::NTH, 1)
    k_spmm_seg(int64_t n, const SegPlan pl, const double* __restrict__ Xext, double* __restrict__ Y,
               const double* __restrict__ r, double* __restrict__ part, const Tail tl, const CholArgs ch, int NS,
               int probe) {
  using K = SsCfg<T>;
  pdl_enter();
  constexpr int S = K::S, G = K::G, C = K::C, RW = K::RW, TR = K::TR, M = K::M, PT = kSegPT, NWC = K::NWC;
  constexpr int VS = seg_vs(W), MT = K::MT;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int cap = pl.cap;
  const size_t SB = seg_stage_bytes<T, W>(cap);
  double* sYw = reinterpret_cast<double*>(smraw + (size_t)NS * SB);  // [NWC][RW][S]
  uint64_t* full = reinterpret_cast<uint64_t*>(sYw + NWC * RW * S);
  uint64_t* empty = full + 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t ntp = (n + PT - 1) / PT;  // plan tiles
  const int64_t nmt = (ntp + M - 1) / M;  // macro tiles
  const int64_t my = nmt > blockIdx.x ? (nmt - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const size_t oV = (size_t)M * cap * T * 8, oL = oV + (size_t)TR * VS * 8, oO = oL + (size_t)TR * 16,
               oR = oO + 16 * M;
  auto stage = [&](int s) { return smraw + (size_t)s * SB; };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWC) {
    // ================= producer warp: stage j%NS ← macro tile blockIdx + j·grid.  The lanes
    // hold the tile's segment table (loaded one tile ahead), a segmented scan places every
    // segment in the stage buffer, lane 0 arms the full barrier with the byte count and
    // every lane issues the bulk copies of its own segments.
    constexpr int NE = M * kSegMax, EPL = (NE + 31) / 32;
    int2 msg[EPL];
    int mown = 0;
    auto load_meta = [&](int64_t j) {
      const int64_t p0 = (blockIdx.x + j * gridDim.x) * M;
      const int pm = j < my ? (int)((ntp - p0) < M ? (ntp - p0) : M) : 0;
      const int2* sg0 = reinterpret_cast<const int2*>(pl.seg) + p0 * kSegMax;
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int e = lane + 32 * u;
        msg[u] = (e < NE && e / kSegMax < pm) ? __ldg(sg0 + e) : make_int2(0, 0);
      }
      mown = lane < pm ? __ldg(pl.own + p0 + lane) : 0;
    };
    load_meta(0);
    for (int64_t j = 0; j < my; ++j) {
      const int s = (int)(j % NS);
      if (j >= NS) mbar_wait(empty + s, (uint32_t)((j / NS - 1) & 1));  // consumers released the stage
      const int64_t mt = blockIdx.x + j * gridDim.x, p0 = mt * M, row0 = mt * TR;
      const int pm = (int)((ntp - p0) < M ? (ntp - p0) : M);
      const int rows = (int)((n - row0) < TR ? (n - row0) : TR);
      unsigned char* st = stage(s);
      uint32_t mine = 0;
#pragma unroll
      for (int u = 0; u < EPL; ++u) mine += (uint32_t)msg[u].y;
      if (lane < pm) reinterpret_cast<int*>(st + oO)[lane] = mown;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
      const int rb = r != nullptr ? (rows & ~1) : 0;  // r rows moved by the bulk copy (16-byte multiple)
      if (lane == 0) {
        if (r != nullptr && (rows & 1)) reinterpret_cast<double*>(st + oR)[rows - 1] = r[row0 + rows - 1];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(full + s, (uint32_t)(pm * PT * VS * 8 + pm * PT * 16 + rb * 8) + mine * T * 8);
        bulk_g2s(st + oV, pl.val + p0 * PT * VS, (uint32_t)(pm * PT * VS * 8), full + s);
        bulk_g2s(st + oL, pl.lidx + p0 * PT * 8, (uint32_t)(pm * PT * 16), full + s);
        if (rb > 0) bulk_g2s(st + oR, r + row0, (uint32_t)rb * 8, full + s);
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int q = lane % kSegMax;  // exclusive scan of run lengths per plan tile (8 lanes)
        int off = msg[u].y;
#pragma unroll
        for (int d = 1; d < kSegMax; d <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, off, d, kSegMax);
          if (q >= d) off += v;
        }
        off -= msg[u].y;
        const int e = lane + 32 * u;
        if (msg[u].y > 0)
          bulk_g2s(reinterpret_cast<double*>(st) + ((size_t)(e / kSegMax) * cap + off) * T,
                   Xext + (int64_t)msg[u].x * T, (uint32_t)msg[u].y * T * 8, full + s);
      }
      load_meta(j + 1);
    }
    // the producer warp still takes part in the epilogue's barriers (zero partial)
  }

  // ================= consumer warps: Y rows, then this warp's rows of XᵀY and Xᵀr on DMMA
  double acc[K::NUT][2];
#pragma unroll
  for (int u = 0; u < K::NUT; ++u) acc[u][0] = acc[u][1] = 0.0;
  double accv[2] = {0.0, 0.0};
  if (warp < NWC) {
    const int rw = lane / G, gl = lane % G;
    double* yw = sYw + (size_t)warp * RW * S;
    for (int64_t j = 0; j < my; ++j) {
      const int s = (int)(j % NS);
      const int64_t mt = blockIdx.x + j * gridDim.x, row0 = mt * TR;
      const int rows = (int)((n - row0) < TR ? (n - row0) : TR);
      const unsigned char* st = stage(s);
      const double* sX = reinterpret_cast<const double*>(st);
      const double* sV = reinterpret_cast<const double*>(st + oV);
      const uint4* sL = reinterpret_cast<const uint4*>(st + oL);
      const int* sO = reinterpret_cast<const int*>(st + oO);
      const double* sR = reinterpret_cast<const double*>(st + oR);
      mbar_wait(full + s, (uint32_t)((j / NS) & 1));
#pragma unroll
      for (int uu = 0; uu < (probe ? 0 : K::UPW); ++uu) {
        const int r0u = (warp + uu * NWC) * RW;  // first row of the unit in the macro tile
        const int rr = r0u + rw;
        const int m = rr / PT;
        const double* xb = sX + (size_t)m * cap * T + gl * C;
        // ---- Y row rr, columns gl·C … gl·C+C-1 (ELL order: p ascending); rows past n: 0
        const uint4 lv = rr < rows ? sL[rr] : make_uint4(0u, 0u, 0u, 0u);
        const unsigned lw[4] = {lv.x, lv.y, lv.z, lv.w};
        int li[W];
#pragma unroll
        for (int k = 0; k < W; ++k) li[k] = (int)((lw[k >> 1] >> (16 * (k & 1))) & 0xffffu);
        double a[VS];
#pragma unroll
        for (int k = 0; k < VS; k += 2) {
          const double2 av =
              rr < rows ? *reinterpret_cast<const double2*>(sV + (size_t)rr * VS + k) : make_double2(0.0, 0.0);
          a[k] = av.x;
          a[k + 1] = av.y;
        }
#pragma unroll
        for (int c2 = 0; c2 < C / 2; ++c2) {
          double2 xv[W];
#pragma unroll
          for (int k = 0; k < W; ++k)  // (rows past n read buffer row 0 of plan tile 0, always present)
            xv[k] = *reinterpret_cast<const double2*>((rr < rows ? xb : sX + gl * C) + (size_t)li[k] * T + 2 * c2);
          double2 y = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < W; ++k) {
            y.x = __fma_rn(a[k], xv[k].x, y.x);
            y.y = __fma_rn(a[k], xv[k].y, y.y);
          }
          if (rr >= rows) y = make_double2(0.0, 0.0);
          else *reinterpret_cast<double2*>(Y + (row0 + rr) * T + gl * C + 2 * c2) = y;
          *reinterpret_cast<double2*>(yw + rw * S + gl * C + 2 * c2) = y;
        }
        __syncwarp();
        // ---- Gram: XᵀY over the unit's RW rows (upper 8×8 tiles), Xᵀr
        const int mu = r0u / PT, qb = r0u % PT;
        const double* xo = sX + ((size_t)mu * cap + sO[mu] + qb) * T;  // own X rows of the unit
#pragma unroll
        for (int ks = 0; ks < RW / 4; ++ks) {
          const int rq = ks * 4 + q4;
          const bool ok = r0u + rq < rows;
          double xa[MT], yb[MT];
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            xa[i] = ok ? xo[rq * T + i * 8 + g] : 0.0;
            yb[i] = yw[rq * S + i * 8 + g];
          }
          int ut = 0;
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int ni = mi; ni < MT; ++ni, ++ut) dmma(acc[ut][0], acc[ut][1], xa[mi], yb[ni]);
        }
        if (r != nullptr) {
#pragma unroll
          for (int rq = 0; rq < RW; ++rq)
            if (r0u + rq < rows) {
              const double vr = sR[r0u + rq];
              if (lane < T) accv[0] = fma(xo[rq * T + lane], vr, accv[0]);
              if (lane + 32 < T) accv[1] = fma(xo[rq * T + lane + 32], vr, accv[1]);
            }
        }
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(empty + s);
    }
  }
  // ================= epilogue: consumer warps' partials summed in warp order, lower half mirrored
  __syncthreads();
  double* red = reinterpret_cast<double*>(smraw);  // T·T + T (stages are drained)
  constexpr int PER = T * T + T;
  for (int w = 0; w < NWC; ++w) {
    if (warp == w) {
      int ut = 0;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = mi; ni < MT; ++ni, ++ut) {
          double* d = red + (mi * 8 + g) * T + ni * 8 + 2 * q4;
          d[0] = w == 0 ? acc[ut][0] : d[0] + acc[ut][0];
          d[1] = w == 0 ? acc[ut][1] : d[1] + acc[ut][1];
        }
      if (lane < T) red[T * T + lane] = w == 0 ? accv[0] : red[T * T + lane] + accv[0];
      if (lane + 32 < T) red[T * T + lane + 32] = w == 0 ? accv[1] : red[T * T + lane + 32] + accv[1];
    }
    __syncthreads();
  }
  double* out = part + (size_t)blockIdx.x * PER;
  for (int e = tid; e < T * T; e += K::NTH) {
    const int rI = e / T, cI = e % T;
    out[e] = (rI / 8 <= cI / 8) ? red[e] : red[cI * T + rI];
  }
  for (int e = tid; e < T; e += K::NTH) out[T * T + e] = red[T * T + e];
  if (tl.cnt != nullptr) {
    const bool last = tail_reduce(part, PER, tl);
    if constexpr (T <= 16) {
      if (last && ch.on && warp == 0)
        chol_warp<T>(tl.out, r != nullptr ? tl.out + T * T : nullptr, ch.R, ch.Rinv, ch.alpha, ch.flag, ch.gblock);
    }
  }
}

// ----------------------------------------------------------------------------
// The SRE-CG fused CGS pass at T = 16 (k_sweep<16,2,2,·,AL> semantics: Z1 = Zin − Q_0C_0 − Q_1C_1 written
// to Zout, per-CTA partial [L_0, Zin]ᵀ Z1 with Zin = A·Q_1 the last left block) restructured for B200:
//  * tiles of 64 rows, warp w owns rows 8w..8w+7 of every tile: its update DMMAs (both column tiles from
//    one A fragment), its Z1 rows (kept in its own rows of the Q_0 tile) and its partial-product k-steps
//    use only its rows — one CTA barrier per tile (the ring), none between the update and the products;
//  * rows stored unpadded (128 B) with the 16-byte chunks XOR-swizzled by f(r) = ((r&1)<<2)|(r&2): every
//    cp.async chunk row is one aligned 128-byte line and every fragment / double2 access is conflict-free;
//  * 3 stages of 4 tiles (96 KB) → 2 CTAs per SM.
// The arithmetic (DMMA k order, Z1 = Zin − D) is that of k_sweep; the partial sums are accumulated per warp
// over its rows and summed over the 8 warps in order (a fixed order: run-to-run reproducible).
// ----------------------------------------------------------------------------
template <int T>
__device__ __forceinline__ int swz(int r, int c) {  // element (r, c) of an unpadded swizzled T-column tile
  return r * T + (((c >> 1) ^ (((r & 1) << 2) | (r & 2))) << 1) + (c & 1);
}

template <int T>
struct UcCfg {
  static constexpr int NS = 3, TR = 64, TILE = TR * T, STAGE = 4 * TILE, SC = T + 4;
  static constexpr int SMEM = NS * STAGE + 2 * T * SC;  // doubles: ring + C (padded)
  static constexpr int NT = T / 8, KS = T / 4;          // column tiles, k-steps per window block
};

template <int T>
__global__ void __launch_bounds__(256, (T == 16 ? 2 : 1))
    k_upcoef_w(int64_t n, const double* Zin, double* Zout, const SweepPtrs P, const double* __restrict__ Cm,
               double* __restrict__ part, const Tail tl) {
  using K = UcCfg<T>;
  constexpr int TR = K::TR, TILE = K::TILE, STAGE = K::STAGE, NS = K::NS, SC = K::SC, NT = K::NT, KS = K::KS;
  pdl_enter();
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + TR - 1) / TR);
  double* sC = sm + NS * STAGE;
  // C (2T×T); lazy blocks: C_j ← R_j⁻¹ C_j (as k_sweep), the ring as scratch before the first copies
  for (int e = tid; e < 2 * T * T; e += 256) sC[(e / T) * SC + e % T] = Cm[e];
  if (P.rq[0] != nullptr || P.rq[1] != nullptr) {
    double* tR = sm;
    double* tO = sm + T * T;
#pragma unroll 1
    for (int j = 0; j < 2; ++j) {
      if (P.rq[j] == nullptr) continue;
      __syncthreads();
      for (int e = tid; e < T * T; e += 256) tR[e] = P.rq[j][e];
      __syncthreads();
      for (int e = tid; e < T * T; e += 256) {
        const int i = e / T, c = e % T;
        double v = 0.0;
        for (int k = i; k < T; ++k) v = fma(tR[i * T + k], sC[(j * T + k) * SC + c], v);
        tO[e] = v;
      }
      __syncthreads();
      for (int e = tid; e < T * T; e += 256) sC[(j * T + e / T) * SC + e % T] = tO[e];
    }
  }
  __syncthreads();
  // B fragments of the update in registers for t = 16 (cf[j][ni][ks] = C_j[4ks + q4][8ni + g]); t = 32 reads
  // them from the padded sC (64 more registers would spill next to the 32 partial tiles)
  constexpr bool CREG = T <= 16;
  double cf[2][CREG ? NT : 1][CREG ? KS : 1];
  if constexpr (CREG) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) cf[j][ni][ks] = sC[(j * T + ks * 4 + q4) * SC + ni * 8 + g];
  }
  __syncthreads();  // the scratch rows of the ring are reused by the copies below

  const double* src[4] = {Zin, P.q[0], P.q[1], P.l[0]};
  auto issue = [&](int i) {
    if (i < ntiles) {
      const int64_t row = lo + (int64_t)i * TR;
      const int rows = (int)((hi - row) < TR ? (hi - row) : TR);
      double* st = sm + (i % NS) * STAGE;
      constexpr int CPR = T / 2;  // 16-byte chunks per row
      for (int e = tid; e < TR * CPR; e += 256) {
        const int r = e / CPR, j = e % CPR;
        const bool ok = r < rows;
        const int d = r * T + ((j ^ (((r & 1) << 2) | (r & 2))) << 1);
#pragma unroll
        for (int a = 0; a < 4; ++a)
          cp16(st + a * TILE + d, ok ? (const void*)(src[a] + (row + r) * T + 2 * j) : (const void*)src[a], ok ? 16 : 0);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) issue(i);

  double acc[2][NT][NT][2];  // [L_0ᵀZ1 | Zinᵀ Z1] tiles (mi, ni)
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int mi = 0; mi < NT; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) acc[l][mi][ni][0] = acc[l][mi][ni][1] = 0.0;
  const int r = warp * 8 + g;  // this lane's update row
  for (int i = 0; i < ntiles; ++i) {
    cp_wait<NS - 2>();
    __syncthreads();
    issue(i + NS - 1);
    double* st = sm + (i % NS) * STAGE;
    const double* sZ = st;
    double* sQ0 = st + TILE;
    const double* sQ1 = st + 2 * TILE;
    const double* sL = st + 3 * TILE;
    const int64_t row = lo + (int64_t)i * TR;
    const int rows = (int)((hi - row) < TR ? (hi - row) : TR);
    // ---- update: D = Q_0 C_0 + Q_1 C_1 over the warp's 8 rows (every column tile per A fragment)
    double d[NT][2];
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) d[ni][0] = d[ni][1] = 0.0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double* sQ = j ? sQ1 : sQ0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double a = sQ[swz<T>(r, ks * 4 + q4)];
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
          dmma(d[ni][0], d[ni][1], a, CREG ? cf[j][CREG ? ni : 0][CREG ? ks : 0] : sC[(j * T + ks * 4 + q4) * SC + ni * 8 + g]);
      }
    }
    __syncwarp();  // the warp's Q_0 rows are read: they now take its Z1 rows
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int c = ni * 8 + 2 * q4;
      const double2 z = *reinterpret_cast<const double2*>(sZ + swz<T>(r, c));
      const double2 z1 = make_double2(z.x - d[ni][0], z.y - d[ni][1]);
      *reinterpret_cast<double2*>(sQ0 + swz<T>(r, c)) = z1;
      if (r < rows) *reinterpret_cast<double2*>(Zout + (row + r) * T + c) = z1;
    }
    __syncwarp();
    // ---- partial [L_0, Zin]ᵀ Z1 over the warp's rows: k-steps of 4 rows
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kr = warp * 8 + ks * 4 + q4;
      double fl[NT], fz[NT], fy[NT];
#pragma unroll
      for (int mi = 0; mi < NT; ++mi) {
        fl[mi] = sL[swz<T>(kr, mi * 8 + g)];
        fz[mi] = sZ[swz<T>(kr, mi * 8 + g)];
        fy[mi] = sQ0[swz<T>(kr, mi * 8 + g)];
      }
#pragma unroll
      for (int mi = 0; mi < NT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          dmma(acc[0][mi][ni][0], acc[0][mi][ni][1], fl[mi], fy[ni]);
          dmma(acc[1][mi][ni][0], acc[1][mi][ni][1], fz[mi], fy[ni]);
        }
    }
  }
  cp_wait<0>();
  // ---- per-CTA partial: the warps' sums in warp order
  constexpr int PER = 2 * T * T;
  __syncthreads();
  double* red = sm;
  {
    double* dst = red + (size_t)warp * PER;
#pragma unroll
    for (int l = 0; l < 2; ++l)
#pragma unroll
      for (int mi = 0; mi < NT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
          *reinterpret_cast<double2*>(dst + l * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4) =
              make_double2(acc[l][mi][ni][0], acc[l][mi][ni][1]);
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * PER;
  for (int e = tid; e < PER; e += 256) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[(size_t)w * PER + e];
    out[e] = v;
  }
  if (tl.cnt != nullptr) tail_reduce(part, PER, tl);
}

// ----------------------------------------------------------------------------
// The A-CholQR Gram [XᵀY (upper 8×8 tiles, lower mirrored) | Xᵀv] of the t = 64 split SpMM step (R35) with
// warp-owned rows: warp w owns rows 8w..8w+7 of every 64-row tile and accumulates ALL 36 upper tiles over
// them, Xᵀv by plain FMAs on the X fragments (k-steps of 4 rows; each X / Y column-tile fragment loaded
// once feeds up to 8 DMMAs: 16 shared loads per 36 DMMAs instead of 2 per DMMA); swizzled unpadded rows (aligned cp.async lines,
// conflict-free fragments); 3 stages of 2 tiles = 192 KB → 1 CTA per SM.  The warps' sums are added in warp
// order (fixed: run-to-run reproducible).
// ----------------------------------------------------------------------------
template <int T>
struct GwCfg {
  static constexpr int NS = 3, TR = 64, TILE = TR * T, STAGE = 2 * TILE + TR;
  static constexpr int MT = T / 8, NUT = MT * (MT + 1) / 2;
  static constexpr int SMEM = NS * STAGE > T * T + T ? NS * STAGE : T * T + T;
};

template <int T, bool V>
__global__ void __launch_bounds__(256, 1)
    k_gram_w(int64_t n, const double* __restrict__ X, const double* __restrict__ Y, const double* __restrict__ v,
             double* __restrict__ part, const Tail tl) {
  using K = GwCfg<T>;
  constexpr int TR = K::TR, TILE = K::TILE, STAGE = K::STAGE, NS = K::NS, MT = K::MT, NUT = K::NUT;
  pdl_enter();
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + TR - 1) / TR);
  auto issue = [&](int i) {
    if (i < ntiles) {
      const int64_t row = lo + (int64_t)i * TR;
      const int rows = (int)((hi - row) < TR ? (hi - row) : TR);
      double* st = sm + (i % NS) * STAGE;
      constexpr int CPR = T / 2;
      for (int e = tid; e < TR * CPR; e += 256) {
        const int r = e / CPR, j = e % CPR;
        const bool ok = r < rows;
        const int d = r * T + ((j ^ (((r & 1) << 2) | (r & 2))) << 1);
        cp16(st + d, ok ? (const void*)(X + (row + r) * T + 2 * j) : (const void*)X, ok ? 16 : 0);
        cp16(st + TILE + d, ok ? (const void*)(Y + (row + r) * T + 2 * j) : (const void*)Y, ok ? 16 : 0);
      }
      if constexpr (V) vec_async<TR>(st + 2 * TILE, v, row, rows);
    }
    cp_commit();
  };
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) issue(i);
  double acc[NUT][2], accv[MT][2];
#pragma unroll
  for (int u = 0; u < NUT; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
  for (int u = 0; u < MT; ++u) accv[u][0] = accv[u][1] = 0.0;
  for (int i = 0; i < ntiles; ++i) {
    cp_wait<NS - 2>();
    __syncthreads();
    issue(i + NS - 1);
    const double* st = sm + (i % NS) * STAGE;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kr = warp * 8 + ks * 4 + q4;
      double fx[MT], fy[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        fx[m] = st[swz<T>(kr, m * 8 + g)];
        fy[m] = st[TILE + swz<T>(kr, m * 8 + g)];
      }
      int u = 0;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = mi; ni < MT; ++ni, ++u) dmma(acc[u][0], acc[u][1], fx[mi], fy[ni]);
      if constexpr (V) {
        // Xᵀv on the FMA pipe: the lane's X fragment fx[m] = X[kr][8m+g] times v[kr] (8 DFMA instead of
        // 8 DMMA with v as column 0 of a tile: a DMMA costs the fp64 pipe ≈ 7 DFMA issue slots)
        const double bv = st[2 * TILE + kr];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) accv[mi][0] = fma(fx[mi], bv, accv[mi][0]);
      }
    }
  }
  if constexpr (V) {  // rows kr = … + q4: sum the 4 lanes of a group (fixed order)
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      accv[mi][0] += __shfl_xor_sync(0xffffffffu, accv[mi][0], 1);
      accv[mi][0] += __shfl_xor_sync(0xffffffffu, accv[mi][0], 2);
    }
  }
  cp_wait<0>();
  // ---- per-CTA partial: the warps' tiles added into shared memory in warp order, lower half mirrored
  constexpr int PER = T * T + (V ? T : 0);
  double* red = sm;
  __syncthreads();
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
      int u = 0;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = mi; ni < MT; ++ni, ++u) {
          double* d = red + (mi * 8 + g) * T + ni * 8 + 2 * q4;
          d[0] = w == 0 ? acc[u][0] : d[0] + acc[u][0];
          d[1] = w == 0 ? acc[u][1] : d[1] + acc[u][1];
        }
      if constexpr (V) {
        if (q4 == 0)
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) {
            double* d = red + T * T + mi * 8 + g;
            *d = w == 0 ? accv[mi][0] : *d + accv[mi][0];
          }
      }
    }
    __syncthreads();
  }
  double* out = part + (size_t)blockIdx.x * PER;
  for (int e = tid; e < T * T; e += 256) {
    const int rI = e / T, cI = e % T;
    out[e] = (rI / 8 <= cI / 8) ? red[e] : red[cI * T + rI];
  }
  if constexpr (V)
    for (int e = tid; e < T; e += 256) out[T * T + e] = red[T * T + e];
  if (tl.cnt != nullptr) tail_reduce(part, PER, tl);
}

static bool gramw_env() {
  static const bool on = [] {  // EKS_GRAMW=0: the generic k_sweep<64,0,1,·,·,UP> Gram (A/B measurements)
    const char* e = getenv("EKS_GRAMW");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

static bool upcoef16_env() {
  static const bool on = [] {  // EKS_UPCOEF16=0: the generic k_sweep<T,2,2,·,AL> at t = 16/32 (A/B measurements)
    const char* e = getenv("EKS_UPCOEF16");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static thread_local int t_last_grid = 0;
int sweep_last_grid() { return t_last_grid; }

// One wave: min(requested, SMs × resident CTAs per SM).
static int grid_for(int nblk_max, int occ) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int g = sms * occ;
  return g < nblk_max ? g : nblk_max;
}
template <int T>
static cudaError_t launch_upcoef_w(cudaStream_t st, int64_t n, const double* Zin, double* Zout, const SweepPtrs& P,
                                   const double* C, double* part, int nblk, const Tail& tl) {
  const size_t sm = (size_t)UcCfg<T>::SMEM * 8;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_upcoef_w<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_upcoef_w<T>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  return launch_k(k_upcoef_w<T>, nblk, 256, sm, st, n, Zin, Zout, P, C, part, tl);
}

template <int T, int NQ, int NL, bool V, bool AL = false, bool UP = false>
static cudaError_t launch_sweep_t(cudaStream_t st, int64_t n, const double* Zin, double* Zout, const SweepPtrs& P,
                                  const double* C, const double* v, double* part, int nblk, const Tail& tl) {
  using K = SwCfg<T, NQ, NL, V, AL, UP>;
  const size_t sm = (size_t)K::SMEM * 8;
  if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_sweep<T, NQ, NL, V, AL, UP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep<T, NQ, NL, V, AL, UP>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  return launch_k(k_sweep<T, NQ, NL, V, AL, UP>, nblk, 256, sm, st, n, Zin, Zout, P, C, v, part,
                  NL > 0 ? tl : Tail{});
}

cudaError_t launch_gram_upper(cudaStream_t st, int t, int64_t n, const double* X, const double* Y, const double* v,
                              double* part, int nblk, const Tail& tl) {
  SweepPtrs P{};
  P.l[0] = X;
  switch (t) {
    case 32: return v ? launch_sweep_t<32, 0, 1, true, false, true>(st, n, Y, nullptr, P, nullptr, v, part, nblk, tl)
                      : launch_sweep_t<32, 0, 1, false, false, true>(st, n, Y, nullptr, P, nullptr, v, part, nblk, tl);
    case 64:
      if (gramw_env()) {
        const size_t sm = (size_t)GwCfg<64>::SMEM * 8;
        auto kern = v ? k_gram_w<64, true> : k_gram_w<64, false>;
        static int occ = 0;
        if (!occ) {
          cudaFuncSetAttribute(k_gram_w<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          cudaFuncSetAttribute(k_gram_w<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gram_w<64, true>, 256, sm);
          if (occ < 1) occ = 1;
        }
        nblk = grid_for(nblk, occ);
        t_last_grid = nblk;
        return launch_k(kern, nblk, 256, sm, st, n, X, Y, v, part, tl);
      }
      return v ? launch_sweep_t<64, 0, 1, true, false, true>(st, n, Y, nullptr, P, nullptr, v, part, nblk, tl)
                      : launch_sweep_t<64, 0, 1, false, false, true>(st, n, Y, nullptr, P, nullptr, v, part, nblk, tl);
    default: return cudaErrorInvalidValue;
  }
}

#define EKS_SW_T(t, ...)                                   \
  switch (t) {                                             \
    case 8: { constexpr int T = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int T = 16; __VA_ARGS__; } break; \
    case 32: { constexpr int T = 32; __VA_ARGS__; } break; \
    case 64: { constexpr int T = 64; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;                 \
  }

bool sweep_supported(int t) { return t == 8 || t == 16 || t == 32 || t == 64; }

// The fused update + coefficient sweep keeps 2·nq+1 blocks per stage plus C in shared memory.
bool sweep_fused_supported(int t, int nq) {
  switch (t) {
    case 8: return nq == 1 ? SwCfg<8, 1, 1, false>::SMEM * 8 <= 227 * 1024 : nq == 2;
    case 16: return nq == 1 || nq == 2;
    case 32: return (nq == 1 || nq == 2) && SwCfg<32, 2, 2, false>::SMEM * 8 <= 227 * 1024;
    case 64: return nq == 1;
    default: return false;
  }
}

int sweep_max_blocks(int t) { return t <= 16 ? 8 : (t == 32 ? 4 : 2); }

size_t sweep_part_stride(int t, int nl, bool v) { return (size_t)nl * t * t + (v ? t : 0); }

template <int T, int K>
static cudaError_t sweep_k(cudaStream_t st, bool upd, int64_t n, const double* Zin, double* Zout, const SweepPtrs& P,
                           const double* C, const double* vec, double* part, int nblk, const Tail& tl) {
  if constexpr (K <= 8 && (T <= 16 || (T == 32 && K <= 4) || (T == 64 && K <= 2))) {
    if (upd) return launch_sweep_t<T, K, 0, false>(st, n, Zin, Zout, P, C, vec, part, nblk, tl);
    // partial products need NL·(T/8)² to be a multiple or divisor of the 8 warps
    if constexpr ((K & (K - 1)) == 0)
      return launch_sweep_t<T, 0, K, false>(st, n, Zin, Zout, P, C, vec, part, nblk, tl);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_sweep(cudaStream_t st, int t, int nq, int nl, bool v, int64_t n, const double* Zin, double* Zout,
                         const SweepPtrs& P, const double* C, const double* vec, double* part, int nblk,
                         const Tail& tl) {
  if (nq > sweep_max_blocks(t) || nl > sweep_max_blocks(t)) return cudaErrorInvalidValue;
  EKS_SW_T(t, {
    if (nq == 0 && nl == 1 && v) return launch_sweep_t<T, 0, 1, true>(st, n, Zin, Zout, P, C, vec, part, nblk, tl);
    if (v) return cudaErrorInvalidValue;
    if (nq == 1 && nl == 1) return launch_sweep_t<T, 1, 1, false>(st, n, Zin, Zout, P, C, vec, part, nblk, tl);
    if (nq == 2 && nl == 2) {
      if constexpr (T == 16 || T == 32)
        if (P.l[1] == Zin && upcoef16_env()) return launch_upcoef_w<T>(st, n, Zin, Zout, P, C, part, nblk, tl);
      if (P.l[1] == Zin) return launch_sweep_t<T, 2, 2, false, true>(st, n, Zin, Zout, P, C, vec, part, nblk, tl);
      return launch_sweep_t<T, 2, 2, false>(st, n, Zin, Zout, P, C, vec, part, nblk, tl);
    }
    if (nq > 0 && nl > 0) return cudaErrorInvalidValue;
    const bool upd = nq > 0;
    switch (upd ? nq : nl) {
      case 1: return sweep_k<T, 1>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 2: return sweep_k<T, 2>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 3: return sweep_k<T, 3>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 4: return sweep_k<T, 4>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 5: return sweep_k<T, 5>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 6: return sweep_k<T, 6>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 7: return sweep_k<T, 7>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      case 8: return sweep_k<T, 8>(st, upd, n, Zin, Zout, P, C, vec, part, nblk, tl);
      default: return cudaErrorInvalidValue;
    }
  });
  return cudaErrorInvalidValue;
}

bool spmm_gram_fused_chol(int t) { return t == 8 || t == 16; }

template <int T, int NZ>
static cudaError_t spmm_gram_t(cudaStream_t st, int64_t n, const int* rp, const int* col, const double* val,
                               const double* Xext, int64_t xoff, double* Y, const double* r, double* part, int nblk,
                               const Tail& tl, const CholArgs& ch) {
  using K = SgCfg<T, NZ>;
  const size_t sm = (size_t)K::SMEM * 8;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_spmm_gram<T, NZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmm_gram<T, NZ>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  return launch_k(k_spmm_gram<T, NZ>, nblk, 256, sm, st, n, rp, col, val, Xext, xoff, Y, r, part, tl, ch);
}

template <int T, int W, int MINB = (T >= 64 ? 2 : 3)>
static cudaError_t spmm_gram_ell_t(cudaStream_t st, int64_t n, const int* ecol, const double* eval, const int* tmax,
                                   int64_t n_ext, const double* Xext, int64_t xoff, double* Y, const double* r,
                                   double* part, int nblk, const Tail& tl, const CholArgs& ch) {
  using K = SeCfg<T, W>;
  const size_t sm = (size_t)K::SMEM * 8;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_spmm_gram_ell<T, W, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmm_gram_ell<T, W, MINB>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  (void)tmax;
  (void)n_ext;
  return launch_k(k_spmm_gram_ell<T, W, MINB>, nblk, 256, sm, st, n, ecol, eval, Xext, xoff, Y, r, part, tl, ch);
}

int ell_width(int maxrow) { return maxrow <= 5 ? 5 : (maxrow <= 7 ? 7 : (maxrow <= 8 ? 8 : 0)); }

cudaError_t launch_spmm_gram_ell(cudaStream_t st, int t, int64_t n, const int* ecol, const double* eval, int w,
                                 const int* tmax, int64_t n_ext, const double* Xext, int64_t xoff, double* Y,
                                 const double* r, double* part, int nblk, const Tail& tl, const CholArgs& ch) {
  if (ch.on && !spmm_gram_fused_chol(t)) return cudaErrorInvalidValue;
  EKS_SW_T(t, {
    // 4 CTAs/SM (≤ 64 registers) hides more gather latency when X streams from HBM; when the
    // block is L2-resident the 3-CTA build (more registers, fewer spills) is faster (measured)
    static const int mbe = getenv("EKS_ELL_MINB") ? atoi(getenv("EKS_ELL_MINB")) : 0;
    const int mb = mbe ? mbe : ((double)n * T * 8 > 64e6 ? 4 : 3);
    if constexpr (T == 16) {
      if (mb == 4 && w == 5) return spmm_gram_ell_t<T, 5, 4>(st, n, ecol, eval, tmax, n_ext, Xext, xoff, Y, r, part, nblk, tl, ch);
      if (mb == 4 && w == 7) return spmm_gram_ell_t<T, 7, 4>(st, n, ecol, eval, tmax, n_ext, Xext, xoff, Y, r, part, nblk, tl, ch);
    }
    if (w == 5) return spmm_gram_ell_t<T, 5>(st, n, ecol, eval, tmax, n_ext, Xext, xoff, Y, r, part, nblk, tl, ch);
    if (w == 7) return spmm_gram_ell_t<T, 7>(st, n, ecol, eval, tmax, n_ext, Xext, xoff, Y, r, part, nblk, tl, ch);
    if (w == 8) return spmm_gram_ell_t<T, 8>(st, n, ecol, eval, tmax, n_ext, Xext, xoff, Y, r, part, nblk, tl, ch);
  });
  return cudaErrorInvalidValue;
}

template <int T, int W>
static cudaError_t spmm_seg_t(cudaStream_t st, int64_t n, const SegPlan& pl, const double* Xext, double* Y,
                              const double* r, double* part, int nblk, const Tail& tl, const CholArgs& ch) {
  using K = SsCfg<T>;
  const size_t SB = seg_stage_bytes<T, W>(pl.cap), fixed = seg_fixed_bytes<T>();
  int ns = (int)((kSegSmem - fixed) / SB);
  if (ns > 8) ns = 8;
  if (ns < 2) return cudaErrorInvalidConfiguration;
  size_t sm = (size_t)ns * SB + fixed;
  const size_t red = (size_t)(T * T + T) * 8;
  if (sm < red) sm = red;
  cudaFuncSetAttribute(k_spmm_seg<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  nblk = nblk < sms ? nblk : sms;  // one persistent CTA per SM
  t_last_grid = nblk;
  static const int probe = getenv("EKS_SEG_PROBE") ? atoi(getenv("EKS_SEG_PROBE")) : 0;
  return launch_k(k_spmm_seg<T, W>, nblk, K::NTH, sm, st, n, pl, Xext, Y, r, part, tl, ch, ns, probe);
}

template <int T>
static bool seg_fits_t(int w, int cap) {
  const size_t SB = w <= 5 ? seg_stage_bytes<T, 5>(cap) : (w <= 7 ? seg_stage_bytes<T, 7>(cap) : seg_stage_bytes<T, 8>(cap));
  const size_t fixed = seg_fixed_bytes<T>();
  return fixed < kSegSmem && (kSegSmem - fixed) / SB >= 2;
}

bool spmm_seg_fits(int t, int w, int cap) {
  if (cap < 1 || cap > 65535 || w < 1 || w > 8) return false;
  switch (t) {
    case 8: return seg_fits_t<8>(w, cap);
    case 16: return seg_fits_t<16>(w, cap);
    case 32: return seg_fits_t<32>(w, cap);
    case 64: return seg_fits_t<64>(w, cap);
    default: return false;
  }
}

cudaError_t launch_spmm_seg(cudaStream_t st, int t, int64_t n, const SegPlan& pl, int w, const double* Xext,
                            double* Y, const double* r, double* part, int nblk, const Tail& tl, const CholArgs& ch) {
  if (ch.on && !spmm_gram_fused_chol(t)) return cudaErrorInvalidValue;
  EKS_SW_T(t, {
    if (w == 5) return spmm_seg_t<T, 5>(st, n, pl, Xext, Y, r, part, nblk, tl, ch);
    if (w == 7) return spmm_seg_t<T, 7>(st, n, pl, Xext, Y, r, part, nblk, tl, ch);
    if (w == 8) return spmm_seg_t<T, 8>(st, n, pl, Xext, Y, r, part, nblk, tl, ch);
  });
  return cudaErrorInvalidValue;
}

cudaError_t launch_spmm_gram(cudaStream_t st, int t, int64_t n, const int* rp, const int* col, const double* val,
                             int maxrow, const double* Xext, int64_t xoff, double* Y, const double* r, double* part,
                             int nblk, const Tail& tl, const CholArgs& ch) {
  if (ch.on && !spmm_gram_fused_chol(t)) return cudaErrorInvalidValue;
  EKS_SW_T(t, {
    (void)maxrow;  // rows of any length (the ELL kernel covers rows of ≤ 8 entries)
    return spmm_gram_t<T, 8>(st, n, rp, col, val, Xext, xoff, Y, r, part, nblk, tl, ch);
  });
  return cudaErrorInvalidValue;
}

template <int T, int C1N, bool ZT = true>
static cudaError_t apply_t(cudaStream_t st, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                           const double* alpha, double* x, double* dx, const double* r, double* rnew, const int* flag,
                           int mode, const double* AWprev, double* part, int nblk, const Tail& tl) {
  if (ZT && (mode & 12) == 12)  // lazy basis without update: the stage layout without Z2 and vectors
    return apply_t<T, C1N, false>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, flag, mode, AWprev, part, nblk, tl);
  using K = ApCfg<T, C1N, ZT>;
  const size_t sm = (size_t)K::SMEM * 8;
  if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_apply_tc<T, C1N, ZT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply_tc<T, C1N, ZT>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  return launch_k(k_apply_tc<T, C1N, ZT>, nblk, 256, sm, st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, flag, mode,
                  AWprev, part, tl);
}

bool apply_c1_supported(int t, int c1n) {
  if (!sweep_supported(t) || c1n < 0 || c1n > 2) return false;
  switch (t) {
    case 8: return ApCfg<8, 2>::SMEM * 8 <= 227 * 1024;
    case 16: return ApCfg<16, 2>::SMEM * 8 <= 227 * 1024;
    case 32: return ApCfg<32, 2>::SMEM * 8 <= 227 * 1024;
    default: return c1n == 0 || ApCfg<64, 2>::SMEM * 8 <= 227 * 1024;
  }
}

cudaError_t launch_apply_tc(cudaStream_t st, int t, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                            const double* alpha, double* x, double* dx, const double* r, double* rnew, const int* flag,
                            int mode, int nblk, int c1n, const double* AWprev, double* part, const Tail& tl) {
  EKS_SW_T(t, {
    if (c1n == 0) return apply_t<T, 0>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, flag, mode, AWprev, part, nblk, tl);
    if (c1n == 1) return apply_t<T, 1>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, flag, mode, AWprev, part, nblk, tl);
    if (c1n == 2) return apply_t<T, 2>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, flag, mode, AWprev, part, nblk, tl);
  });
  return cudaErrorInvalidValue;
}

}  // namespace eks
