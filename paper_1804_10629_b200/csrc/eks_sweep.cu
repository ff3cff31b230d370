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
#include "eks_kernels.cuh"
#include "eks_sweep.cuh"

#include <climits>
#include <cstdint>

namespace eks {

namespace {

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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

// D(8×8) += A(8×4, row) · B(4×8, col): lane (g = lane>>2, q = lane&3) holds
// a = A[g][q], b = B[q][g], d = {D[g][2q], D[g][2q+1]}.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
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
//   NQ: blocks in the update R = Zin − Σ_q Q_q C_q (0: R = Zin, no update)
//   NL: left blocks of the partial Lᵀ R (0: none);  V: also L_0ᵀ v
// ----------------------------------------------------------------------------
template <int T, int NQ, int NL, bool V>
struct SwCfg {
  static constexpr int TR = (T == 8) ? 64 : 32;  // rows per tile
  static constexpr int S = T + 4;                // padded smem row stride (doubles)
  static constexpr int TILE = TR * S;            // doubles per block tile
  static constexpr int NARR = 1 + NQ + NL;       // streamed blocks
  static constexpr int STAGE = NARR * TILE + (V ? TR : 0);  // doubles per stage
  static constexpr int SC = T + 4;               // padded stride of C
  static constexpr int CDBL = NQ * T * SC;
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
  static constexpr int OT = NL * MT * MT;
  static constexpr int WS = (NL == 0) ? 1 : (OT >= 8 ? 1 : 8 / OT);
  static constexpr int TPW = (NL == 0) ? 0 : (OT >= 8 ? OT / 8 : 1);
  static constexpr int PER = NL * T * T + (V ? T : 0);  // partial doubles per CTA
  static constexpr int RED = (WS > 1 ? 8 * NL * T * T : 0) + (V ? 8 * T : 0);
  static constexpr int SMEM0 = NS * STAGE + CDBL;
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;  // doubles
};

template <int T, int NQ, int NL, bool V>
__global__ void __launch_bounds__(256, 1)
    k_sweep(int64_t n, const double* Zin, double* Zout, const SweepPtrs P,
            const double* __restrict__ Cm, const double* __restrict__ v, double* __restrict__ part) {
  using K = SwCfg<T, NQ, NL, V>;
  constexpr int S = K::S;
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + K::TR - 1) / K::TR);
  double* sC = sm + K::NS * K::STAGE;

  if constexpr (NQ > 0)
    for (int e = tid; e < NQ * T * T; e += 256) sC[(e / T) * K::SC + e % T] = Cm[e];

  auto issue = [&](int i) {
    if (i < ntiles) {
      const int s = i % K::NS;
      const int64_t row = lo + (int64_t)i * K::TR;
      const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
      double* st = sm + s * K::STAGE;
      tile_async<T, S, K::TR>(st, Zin, row, rows);
#pragma unroll
      for (int j = 0; j < NQ; ++j) tile_async<T, S, K::TR>(st + (1 + j) * K::TILE, P.q[j], row, rows);
#pragma unroll
      for (int j = 0; j < NL; ++j) tile_async<T, S, K::TR>(st + (1 + NQ + j) * K::TILE, P.l[j], row, rows);
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
            dmma(d0, d1, sQ[(mi * 8 + g) * S + kk + q4], Cj[(kk + q4) * K::SC + ni * 8 + g]);
        }
        const int r = mi * 8 + g, c = ni * 8 + 2 * q4;
        const double z0 = sZ[r * S + c] - d0, z1 = sZ[r * S + c + 1] - d1;
        sZ[r * S + c] = z0;
        sZ[r * S + c + 1] = z1;
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
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        const double* sL = st + (1 + NQ + l) * K::TILE;
        double d0 = acc[u][0], d1 = acc[u][1];
#pragma unroll
        for (int kk = slice * 4; kk < K::TR; kk += 4 * K::WS)
          dmma(d0, d1, sL[(kk + q4) * S + mi * 8 + g], sZ[(kk + q4) * S + ni * 8 + g]);
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
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
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
  }
}

// ----------------------------------------------------------------------------
// W = Z2·R⁻¹, AW = AZ2·R⁻¹ (in place) and the fused x/r update of the block
// (see launch_apply).  Same pipeline; both products on DMMA.
// ----------------------------------------------------------------------------
template <int T, int C1N>
struct ApCfg {
  static constexpr int TR = 64;  // 8 warps × 8 rows: every warp owns complete rows
  static constexpr int S = T + 4;
  static constexpr int TILE = TR * S;
  // Z2, AZ2 tiles (+ AW_prev tile when C1N == 2) + r_in, dx, x vectors
  static constexpr int STAGE = (C1N == 2 ? 3 : 2) * TILE + 3 * TR;
  static constexpr int NSA = (100 * 1024 / 8 - T * (T + 4)) / STAGE;
  static constexpr int NS0 = NSA >= 3 ? NSA : (200 * 1024 / 8 - T * (T + 4)) / STAGE;
  static constexpr int NS = NS0 > 8 ? 8 : (NS0 < 2 ? 2 : NS0);
  static constexpr int NT = T / 8;  // column tiles per row group (all in the same warp)
  // fused next-pass coefficients C1 = [AW_prev, AW]ᵀ AW: C1N·(T/8)² output tiles over 8 warps
  static constexpr int MT = T / 8;
  static constexpr int OT = C1N * MT * MT;
  static constexpr int WS = (C1N == 0) ? 1 : (OT >= 8 ? 1 : 8 / OT);
  static constexpr int TPW = (C1N == 0) ? 1 : (OT >= 8 ? OT / 8 : 1);
  static constexpr int RED = (WS > 1 ? 8 * C1N * T * T : 0);
  static constexpr int SMEM0 = NS * STAGE + T * (T + 4) + T;
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;
};

template <int T, int C1N>
__global__ void __launch_bounds__(256, 1)
    k_apply_tc(int64_t n, double* Z2W, double* AZ2AW, const double* __restrict__ Rinv,
               const double* __restrict__ alpha, double* __restrict__ x, double* __restrict__ dx,
               const double* __restrict__ r, double* __restrict__ rnew, double* __restrict__ rho_part,
               const int* __restrict__ flag, int mode, const double* __restrict__ AWprev,
               double* __restrict__ c1part) {
  using K = ApCfg<T, C1N>;
  constexpr int S = K::S, SR = T + 4;
  extern __shared__ __align__(128) double sm[];
  __shared__ double sred[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + K::TR - 1) / K::TR);
  double* sRi = sm + K::NS * K::STAGE;
  double* sA = sRi + T * SR;
  const bool first = mode & 1, last = mode & 2, basis = mode & 4;
  const bool skip = basis || (flag != nullptr && *flag != INT_MAX);
  for (int e = tid; e < T * T; e += 256) sRi[(e / T) * SR + e % T] = Rinv[e];
  for (int e = tid; e < T; e += 256) sA[e] = alpha ? alpha[e] : 0.0;
  constexpr int VOFF = (C1N == 2 ? 3 : 2) * K::TILE;  // vectors after the tiles
  auto issue = [&](int i) {
    if (i < ntiles) {
      const int s = i % K::NS;
      const int64_t row = lo + (int64_t)i * K::TR;
      const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
      double* st = sm + s * K::STAGE;
      tile_async<T, S, K::TR>(st, Z2W, row, rows);
      tile_async<T, S, K::TR>(st + K::TILE, AZ2AW, row, rows);
      if constexpr (C1N == 2) tile_async<T, S, K::TR>(st + 2 * K::TILE, AWprev, row, rows);
      if (!skip) {
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
  double rr_acc = 0.0;
  double acc[K::TPW][2];
#pragma unroll
  for (int u = 0; u < K::TPW; ++u) acc[u][0] = acc[u][1] = 0.0;
  for (int i = 0; i < ntiles; ++i) {
    cp_wait<K::NS - 2>();
    __syncthreads();
    issue(i + K::NS - 1);
    double* sZ = sm + (i % K::NS) * K::STAGE;
    double* sY = sZ + K::TILE;
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
#pragma unroll
      for (int kk = 0; kk < T; kk += 4) {
        const double b = sRi[(kk + q4) * SR + ni * 8 + g];
        dmma(w0, w1, sZ[rr * S + kk + q4], b);
        dmma(y0, y1, sY[rr * S + kk + q4], b);
      }
      const int c = ni * 8 + 2 * q4;
      if (rr < rows) {
        *reinterpret_cast<double2*>(Z2W + (row + rr) * T + c) = make_double2(w0, w1);
        *reinterpret_cast<double2*>(AZ2AW + (row + rr) * T + c) = make_double2(y0, y1);
      }
      yk[ni][0] = y0;
      yk[ni][1] = y1;
      double tu = fma(w0, sA[c], w1 * sA[c + 1]);
      double tq = fma(y0, sA[c], y1 * sA[c + 1]);
      tu += __shfl_xor_sync(0xffffffffu, tu, 1);
      tq += __shfl_xor_sync(0xffffffffu, tq, 1);
      tu += __shfl_xor_sync(0xffffffffu, tu, 2);
      tq += __shfl_xor_sync(0xffffffffu, tq, 2);
      pu += tu;
      pq += tq;
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
      __syncthreads();
      const int slice = warp % K::WS;
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = (warp / K::WS) * K::TPW + u;
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
        const double* sL = (C1N == 2 && l == 0) ? sZ + 2 * K::TILE : sY;
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
  if (last && rho_part != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rr_acc += __shfl_down_sync(0xffffffffu, rr_acc, o);
    if (lane == 0) sred[warp] = rr_acc;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < 8; ++w) sacc += sred[w];
      rho_part[blockIdx.x] = sacc;
    }
  }
  if constexpr (C1N > 0) {
    double* out = c1part + (size_t)blockIdx.x * C1N * T * T;
    __syncthreads();
    if constexpr (K::WS == 1) {
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = warp * K::TPW + u;
        const int l = tile / (K::MT * K::MT), mi = (tile / K::MT) % K::MT, ni = tile % K::MT;
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
}

// ----------------------------------------------------------------------------
// Fused SpMM + Gram (A-CholQR's B = Z2ᵀ(A Z2) and Z2ᵀr; Y = A·X).
// Per TR-row tile the CTA streams, through the cp.async ring: the tile's CSR row
// pointers, its (col, val) entries, its own X rows and r.  Only the X gathers of
// neighbour rows remain dependent loads (mostly L2 hits for stencils).  Y is
// written to HBM and kept in shared memory, and the Gram partial XᵀY, Xᵀr of the
// tile is accumulated on DMMA.  Accumulation order of every Y entry: p
// ascending, fma from 0.0 — bitwise equal to k_spmm and to the oracle (R20).
// ----------------------------------------------------------------------------
template <int T>
struct SgCfg {
  static constexpr int TR = 64;
  static constexpr int S = T + 4;
  static constexpr int G = T / 2;         // threads per row (2 columns each)
  static constexpr int RPP = 256 / G;      // rows per pass
  static constexpr int PASSES = TR / RPP;
  static constexpr int MAXROW = 8;         // entries per row supported by the staged path
  static constexpr int ECAP = TR * MAXROW + 4;  // + alignment slack of the 16-byte copies
  // stage layout (doubles): X tile | r tile | val[ECAP] | col[ECAP] (ints) | rp[TR+4] (ints)
  static constexpr int STAGE = TR * S + TR + ECAP + (ECAP + TR + 4) / 2 + 2;
  static constexpr int YT = TR * S;        // Y tile (single buffer)
  static constexpr int NSA = (100 * 1024 / 8 - YT) / STAGE;
  static constexpr int NS = NSA > 6 ? 6 : (NSA < 3 ? 3 : NSA);
  static constexpr int MT = T / 8;
  static constexpr int OT = MT * MT;
  static constexpr int WS = OT >= 8 ? 1 : 8 / OT;
  static constexpr int TPW = OT >= 8 ? OT / 8 : 1;
  static constexpr int PER = T * T + T;
  static constexpr int RED = (WS > 1 ? 8 * T * T : 0) + 8 * T;
  static constexpr int SMEM0 = NS * STAGE + YT;
  static constexpr int SMEM = SMEM0 > RED ? SMEM0 : RED;
};

template <int T>
__global__ void __launch_bounds__(256, (T <= 16 ? 3 : 2))
    k_spmm_gram(int64_t n, const int* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                const double* __restrict__ Xext, const double* __restrict__ Xloc, double* __restrict__ Y,
                const double* __restrict__ r, double* __restrict__ part) {
  using K = SgCfg<T>;
  constexpr int S = K::S;
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int ntiles = (int)((hi - lo + K::TR - 1) / K::TR);
  double* sY = sm + K::NS * K::STAGE;
  static_assert(K::NS >= 3, "the L2 prefetch of tile i+1 needs two landed stages");
  auto row0_of = [&](int i) { return lo + (int64_t)i * K::TR; };

  // (p_begin, p_end) of tile i, prefetched one iteration ahead of its issue
  auto bounds = [&](int i, int& pb, int& pe) {
    if (i < ntiles) {
      const int64_t row = lo + (int64_t)i * K::TR;
      const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
      pb = __ldg(rp + row);
      pe = __ldg(rp + row + rows);
    }
  };
  auto issue = [&](int i, int pb, int pe) {
    if (i < ntiles) {
      const int s = i % K::NS;
      const int64_t row = lo + (int64_t)i * K::TR;
      const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
      double* st = sm + s * K::STAGE;
      tile_async<T, S, K::TR>(st, Xloc, row, rows);
      if (r != nullptr) vec_async<K::TR>(st + K::TR * S, r, row, rows);
      double* sval = st + K::TR * S + K::TR;
      int* scol = reinterpret_cast<int*>(sval + K::ECAP);
      int* srp = scol + K::ECAP;
      // 16-byte chunks of the aligned-down ranges (the device CSR arrays are padded by 16 bytes)
      const int pv = pb & ~1, pc = pb & ~3;
      const int nv = (pe - pv + 1) >> 1, nc = (pe - pc + 3) >> 2, nr = (rows + 4) >> 2;
      for (int e = tid; e < nv + nc + nr; e += 256) {
        if (e < nv) cp16(sval + 2 * e, val + pv + 2 * e, 16);
        else if (e < nv + nc) cp16(scol + 4 * (e - nv), col + pc + 4 * (e - nv), 16);
        else cp16(srp + 4 * (e - nv - nc), rp + row + 4 * (e - nv - nc), 16);
      }
    }
    cp_commit();
  };
  int nb[K::NS][2];
#pragma unroll
  for (int i = 0; i < K::NS; ++i) {
    nb[i][0] = nb[i][1] = 0;
    bounds(i, nb[i][0], nb[i][1]);
  }
#pragma unroll
  for (int i = 0; i < K::NS - 1; ++i) issue(i, nb[i][0], nb[i][1]);
  int pend_b = nb[K::NS - 1][0], pend_e = nb[K::NS - 1][1];  // bounds of the next tile to issue

  double acc[K::TPW][2];
#pragma unroll
  for (int j = 0; j < K::TPW; ++j) acc[j][0] = acc[j][1] = 0.0;
  double accv[2] = {0.0, 0.0};
  const int grp = tid / K::G, gl = tid % K::G;

  for (int i = 0; i < ntiles; ++i) {
    cp_wait<K::NS - 3>();  // tiles i and i+1 have landed
    __syncthreads();
    issue(i + K::NS - 1, pend_b, pend_e);
    int nbb = 0, nbe = 0;
    bounds(i + K::NS, nbb, nbe);  // prefetch for the next issue
    if (i + 1 < ntiles) {
      // warm L2 with the out-of-tile X rows tile i+1 will gather
      const double* sn = sm + ((i + 1) % K::NS) * K::STAGE + K::TR * S + K::TR;
      const int* ncol = reinterpret_cast<const int*>(sn + K::ECAP);
      const int* nrp = ncol + K::ECAP;
      const int64_t nrow = row0_of(i + 1);
      const int nrows = (int)((hi - nrow) < K::TR ? (hi - nrow) : K::TR);
      const int ne = nrp[nrows] - nrp[0], nco = nrp[0] & 3;
      constexpr int LPR = (T * 8 + 127) / 128;  // 128-byte lines per X row
      for (int e = tid; e < ne * LPR; e += 256) {
        const int c = ncol[nco + e / LPR];
        if (c < nrow || c >= nrow + nrows)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(Xext + (int64_t)c * T + (e % LPR) * 16));
      }
    }
    const double* st = sm + (i % K::NS) * K::STAGE;
    const double* sX = st;
    const double* sr = st + K::TR * S;
    const double* sval = sr + K::TR;
    const int* scol = reinterpret_cast<const int*>(sval + K::ECAP);
    const int* srp = scol + K::ECAP;
    const int64_t row = lo + (int64_t)i * K::TR;
    const int rows = (int)((hi - row) < K::TR ? (hi - row) : K::TR);
    const int pbase = srp[0], vo = pbase & 1, co = pbase & 3;  // offsets of the aligned copies
    // ---------------- Y rows of the tile
#pragma unroll
    for (int ps = 0; ps < K::PASSES; ++ps) {
      const int rr = ps * K::RPP + grp;
      double ax = 0.0, ay = 0.0;
      if (rr < rows) {
        const int q0 = srp[rr] - pbase, q1 = srp[rr + 1] - pbase;
        double a[K::MAXROW];
        double2 xv[K::MAXROW];
#pragma unroll
        for (int k = 0; k < K::MAXROW; ++k)
          if (q0 + k < q1) {
            a[k] = sval[vo + q0 + k];
            xv[k] = __ldg(reinterpret_cast<const double2*>(Xext + (int64_t)scol[co + q0 + k] * T) + gl);
          }
#pragma unroll
        for (int k = 0; k < K::MAXROW; ++k)
          if (q0 + k < q1) {
            ax = __fma_rn(a[k], xv[k].x, ax);
            ay = __fma_rn(a[k], xv[k].y, ay);
          }
        *reinterpret_cast<double2*>(Y + (row + rr) * T + 2 * gl) = make_double2(ax, ay);
      }
      sY[rr * S + 2 * gl] = ax;  // rows beyond the tile end stay 0 in the Gram
      sY[rr * S + 2 * gl + 1] = ay;
    }
    __syncthreads();
    // ---------------- Gram partial Xᵀ Y and Xᵀ r of the tile (X rows beyond `rows` are zero-filled)
    {
      const int slice = warp % K::WS;
#pragma unroll
      for (int u = 0; u < K::TPW; ++u) {
        const int tile = (warp / K::WS) * K::TPW + u;
        const int mi = tile / K::MT, ni = tile % K::MT;
        double d0 = acc[u][0], d1 = acc[u][1];
#pragma unroll
        for (int kk = slice * 4; kk < K::TR; kk += 4 * K::WS)
          dmma(d0, d1, sX[(kk + q4) * S + mi * 8 + g], sY[(kk + q4) * S + ni * 8 + g]);
        acc[u][0] = d0;
        acc[u][1] = d1;
      }
      for (int rr = warp; r != nullptr && rr < rows; rr += 8) {
        const double vr = sr[rr];
        if (lane < T) accv[0] = fma(sX[rr * S + lane], vr, accv[0]);
        if (lane + 32 < T) accv[1] = fma(sX[rr * S + lane + 32], vr, accv[1]);
      }
    }
    pend_b = nbb;
    pend_e = nbe;
  }
  cp_wait<0>();
  // ---------------- per-CTA partial (same layout as k_sweep<T,0,1,true>)
  double* out = part + (size_t)blockIdx.x * K::PER;
  double* red = sm;
  __syncthreads();
  if constexpr (K::WS == 1) {
#pragma unroll
    for (int u = 0; u < K::TPW; ++u) {
      const int tile = warp * K::TPW + u;
      const int mi = tile / K::MT, ni = tile % K::MT;
      *reinterpret_cast<double2*>(out + (mi * 8 + g) * T + ni * 8 + 2 * q4) = make_double2(acc[u][0], acc[u][1]);
    }
  } else {
    {
      const int tile = warp / K::WS;
      const int mi = tile / K::MT, ni = tile % K::MT;
      red[(size_t)warp * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4] = acc[0][0];
      red[(size_t)warp * T * T + (mi * 8 + g) * T + ni * 8 + 2 * q4 + 1] = acc[0][1];
    }
    __syncthreads();
    for (int e = tid; e < T * T; e += 256) {
      const int m = e / T, nn = e % T;
      const int tile = (m / 8) * K::MT + nn / 8;
      double s = 0.0;
      for (int w = tile * K::WS; w < tile * K::WS + K::WS; ++w) s += red[(size_t)w * T * T + e];
      out[e] = s;
    }
  }
  double* rv = red + (K::WS > 1 ? 8 * T * T : 0);
  if (lane < T) rv[warp * T + lane] = accv[0];
  if (lane + 32 < T) rv[warp * T + lane + 32] = accv[1];
  __syncthreads();
  for (int e = tid; e < T; e += 256) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += rv[w * T + e];
    out[T * T + e] = s;
  }
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
template <int T, int NQ, int NL, bool V>
static cudaError_t launch_sweep_t(cudaStream_t st, int64_t n, const double* Zin, double* Zout, const SweepPtrs& P,
                                  const double* C, const double* v, double* part, int nblk) {
  using K = SwCfg<T, NQ, NL, V>;
  const size_t sm = (size_t)K::SMEM * 8;
  if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_sweep<T, NQ, NL, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep<T, NQ, NL, V>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  k_sweep<T, NQ, NL, V><<<nblk, 256, sm, st>>>(n, Zin, Zout, P, C, v, part);
  return cudaGetLastError();
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
                           const double* C, const double* vec, double* part, int nblk) {
  if constexpr (K <= 8 && (T <= 16 || (T == 32 && K <= 4) || (T == 64 && K <= 2))) {
    if (upd) return launch_sweep_t<T, K, 0, false>(st, n, Zin, Zout, P, C, vec, part, nblk);
    // partial products need NL·(T/8)² to be a multiple or divisor of the 8 warps
    if constexpr ((K & (K - 1)) == 0) return launch_sweep_t<T, 0, K, false>(st, n, Zin, Zout, P, C, vec, part, nblk);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_sweep(cudaStream_t st, int t, int nq, int nl, bool v, int64_t n, const double* Zin, double* Zout,
                         const SweepPtrs& P, const double* C, const double* vec, double* part, int nblk) {
  if (nq > sweep_max_blocks(t) || nl > sweep_max_blocks(t)) return cudaErrorInvalidValue;
  EKS_SW_T(t, {
    if (nq == 0 && nl == 1 && v) return launch_sweep_t<T, 0, 1, true>(st, n, Zin, Zout, P, C, vec, part, nblk);
    if (v) return cudaErrorInvalidValue;
    if (nq == 1 && nl == 1) return launch_sweep_t<T, 1, 1, false>(st, n, Zin, Zout, P, C, vec, part, nblk);
    if (nq == 2 && nl == 2) return launch_sweep_t<T, 2, 2, false>(st, n, Zin, Zout, P, C, vec, part, nblk);
    if (nq > 0 && nl > 0) return cudaErrorInvalidValue;
    const bool upd = nq > 0;
    switch (upd ? nq : nl) {
      case 1: return sweep_k<T, 1>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 2: return sweep_k<T, 2>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 3: return sweep_k<T, 3>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 4: return sweep_k<T, 4>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 5: return sweep_k<T, 5>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 6: return sweep_k<T, 6>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 7: return sweep_k<T, 7>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      case 8: return sweep_k<T, 8>(st, upd, n, Zin, Zout, P, C, vec, part, nblk);
      default: return cudaErrorInvalidValue;
    }
  });
  return cudaErrorInvalidValue;
}

int spmm_gram_max_row() { return 8; }

cudaError_t launch_spmm_gram(cudaStream_t st, int t, int64_t n, const int* rp, const int* col, const double* val,
                             const double* Xext, const double* Xloc, double* Y, const double* r, double* part,
                             int nblk) {
  EKS_SW_T(t, {
    using K = SgCfg<T>;
    static_assert(K::MAXROW == 8, "spmm_gram_max_row");
    const size_t sm = (size_t)K::SMEM * 8;
    static int occ = 0;
    if (!occ) {
      cudaFuncSetAttribute(k_spmm_gram<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmm_gram<T>, 256, sm);
      if (occ < 1) occ = 1;
    }
    nblk = grid_for(nblk, occ);
    t_last_grid = nblk;
    k_spmm_gram<T><<<nblk, 256, sm, st>>>(n, rp, col, val, Xext, Xloc, Y, r, part);
  });
  return cudaGetLastError();
}

template <int T, int C1N>
static cudaError_t apply_t(cudaStream_t st, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                           const double* alpha, double* x, double* dx, const double* r, double* rnew,
                           double* rho_part, const int* flag, int mode, const double* AWprev, double* c1part,
                           int nblk) {
  using K = ApCfg<T, C1N>;
  const size_t sm = (size_t)K::SMEM * 8;
  if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_apply_tc<T, C1N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply_tc<T, C1N>, 256, sm);
    if (occ < 1) occ = 1;
  }
  nblk = grid_for(nblk, occ);
  t_last_grid = nblk;
  k_apply_tc<T, C1N><<<nblk, 256, sm, st>>>(n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, rho_part, flag, mode,
                                            AWprev, c1part);
  return cudaGetLastError();
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
                            const double* alpha, double* x, double* dx, const double* r, double* rnew,
                            double* rho_part, const int* flag, int mode, int nblk, int c1n, const double* AWprev,
                            double* c1part) {
  EKS_SW_T(t, {
    if (c1n == 0) return apply_t<T, 0>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, rho_part, flag, mode, AWprev,
                                       c1part, nblk);
    if (c1n == 1) return apply_t<T, 1>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, rho_part, flag, mode, AWprev,
                                       c1part, nblk);
    if (c1n == 2) return apply_t<T, 2>(st, n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, rho_part, flag, mode, AWprev,
                                       c1part, nblk);
  });
  return cudaErrorInvalidValue;
}

}  // namespace eks
