// eks_kernels.cu — sm_100a CUDA kernels of the s-step enlarged CG hot path
// (arXiv:1804.10629, Alg 3/4/6).  fp64 throughout (the paper's MATLAB precision).
// Blocks are row-major n×T, T a power of two ≤ 64.  No fp64 atomics: every
// reduction is a fixed-order two-stage tree (per-CTA partials, then
// launch_reduce), so results are bitwise reproducible run to run.
#include "eks_device.cuh"
#include "eks_kernels.cuh"

#include <climits>
#include <cstdio>
#include <cstdlib>

namespace eks {

bool pdl_enabled() {
  static const int on = getenv("EKS_PDL") ? atoi(getenv("EKS_PDL")) : 1;
  return on != 0;
}

// Upper bound on CTAs (= per-CTA partial slots) of the row-sweep kernels; each
// launcher uses min(this, SMs × resident CTAs per SM), i.e. one full wave.
int sweep_ctas(int sms) { return 4 * sms; }

#define EKS_DISPATCH_T(t, ...)                          \
  switch (t) {                                          \
    case 1: { constexpr int T = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int T = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int T = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int T = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int T = 16; __VA_ARGS__; } break; \
    case 32: { constexpr int T = 32; __VA_ARGS__; } break; \
    case 64: { constexpr int T = 64; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;              \
  }

static inline int ilog2(int t) { int l = 0; while ((1 << l) < t) ++l; return l; }

__device__ __forceinline__ int64_t chunk_lo(int64_t n, int b, int nb) { return (int64_t)b * n / nb; }

// Sum a per-thread double over the CTA in a fixed order (warp shuffle tree, then warps in order).
__device__ __forceinline__ double block_sum(double v, double* sbuf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sbuf[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sbuf[i];
  return s;
}

// ============================================================================
// (a1) T(r) — P:41 ("T(r_0) … splits r_0 into t vectors").
// ============================================================================
__global__ void k_split(int t, int lt, int64_t n_local, int64_t row0, int64_t n_global,
                        const double* __restrict__ r, double* __restrict__ Z) {
  const int64_t total = n_local * t;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e >> lt;
    const int c = (int)(e & (t - 1));
    const int64_t g = row0 + i;
    // D_c = [floor(c n / t), floor((c+1) n / t))  (reading R1); t is a power of two
    const int64_t lo = ((int64_t)c * n_global) >> lt, hi = ((int64_t)(c + 1) * n_global) >> lt;
    Z[e] = (g >= lo && g < hi) ? r[i] : 0.0;
  }
}

cudaError_t launch_split(cudaStream_t st, int t, int64_t n_local, int64_t row0, int64_t n_global,
                         const double* r, double* Z) {
  if (n_local <= 0) return cudaSuccess;
  int64_t total = n_local * t;
  int blocks = (int)((total + kThreads - 1) / kThreads);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_split<<<blocks, kThreads, 0, st>>>(t, ilog2(t), n_local, row0, n_global, r, Z);
  return cudaGetLastError();
}

// ============================================================================
// (a2) SpMM Y = A·X — P:54.  G = T/2 threads per row, each
// owning two consecutive columns (16-byte loads of the row-major X rows).
// Accumulation: p ascending, fma, from 0.0 — bitwise equal to the oracle (R20).
// ============================================================================
template <int T>
__global__ void __launch_bounds__(kThreads) k_spmm(int r0, int r1, const int* __restrict__ rp,
                                                   const int* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ X, double* __restrict__ Y) {
  constexpr int VEC = T >= 2 ? 2 : 1;
  constexpr int G = T / VEC;
  const int lane = threadIdx.x % G;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  constexpr int B = 8;  // entries fetched per batch: all (val, col) loads, then all X gathers in flight
  for (int64_t i = r0 + grp; i < r1; i += ngrp) {
    const int p0 = __ldg(rp + i), p1 = __ldg(rp + i + 1);
    if constexpr (VEC == 2) {
      double ax = 0.0, ay = 0.0;
      int p = p0;
      for (; p + B <= p1; p += B) {
        double a[B];
        int c[B];
        double2 xv[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
          a[k] = __ldg(val + p + k);
          c[k] = __ldg(col + p + k);
        }
#pragma unroll
        for (int k = 0; k < B; ++k) xv[k] = __ldg(reinterpret_cast<const double2*>(X + (int64_t)c[k] * T) + lane);
#pragma unroll
        for (int k = 0; k < B; ++k) {
          ax = __fma_rn(a[k], xv[k].x, ax);
          ay = __fma_rn(a[k], xv[k].y, ay);
        }
      }
      if (p < p1) {  // tail (< B entries; a 5/7-point stencil row lands here entirely)
        const int m = p1 - p;
        double a[B];
        int c[B];
        double2 xv[B];
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (k < m) {
            a[k] = __ldg(val + p + k);
            c[k] = __ldg(col + p + k);
          }
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (k < m) xv[k] = __ldg(reinterpret_cast<const double2*>(X + (int64_t)c[k] * T) + lane);
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (k < m) {
            ax = __fma_rn(a[k], xv[k].x, ax);
            ay = __fma_rn(a[k], xv[k].y, ay);
          }
        p = p1;
      }
      for (; p < p1; ++p) {
        const double a = __ldg(val + p);
        const int c = __ldg(col + p);
        const double2 xv = __ldg(reinterpret_cast<const double2*>(X + (int64_t)c * T) + lane);
        ax = __fma_rn(a, xv.x, ax);
        ay = __fma_rn(a, xv.y, ay);
      }
      reinterpret_cast<double2*>(Y + i * T)[lane] = make_double2(ax, ay);
    } else {
      double ax = 0.0;
      for (int p = p0; p < p1; ++p) ax = __fma_rn(__ldg(val + p), __ldg(X + __ldg(col + p)), ax);
      Y[i] = ax;
    }
  }
}

cudaError_t launch_spmm(cudaStream_t st, int t, int r0, int r1, const int* rp, const int* col,
                        const double* val, const double* Xext, double* Y, int sms) {
  if (r1 <= r0) return cudaSuccess;
  EKS_DISPATCH_T(t, {
    constexpr int G = (T >= 2 ? T / 2 : 1);
    int64_t threads = (int64_t)(r1 - r0) * G;
    int64_t blocks = (threads + kThreads - 1) / kThreads;
    int64_t cap = (int64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    k_spmm<T><<<(int)blocks, kThreads, 0, st>>>(r0, r1, rp, col, val, Xext, Y);
  });
  return cudaGetLastError();
}

// ============================================================================
// Tall-skinny Lᵀ·R partial products (CGS2 coefficients, Gram matrices).
// Each CTA owns a contiguous row chunk, streams TR-row tiles of R and of up to
// GL left blocks through shared memory, and accumulates a TA×TA register tile
// per thread; KS row slices are summed in a fixed order at the end.
// ============================================================================
constexpr int kMaxList = 32;
struct PtrList { const double* p[kMaxList]; };

template <int T>
struct TnCfg {
  static constexpr int TA = T >= 64 ? 8 : (T >= 16 ? 4 : (T >= 2 ? 2 : 1));
  static constexpr int NA = T / TA;
  static constexpr int TPS = NA * NA;
  static constexpr int KS = kThreads / TPS;
  static constexpr int TR = KS > 32 ? KS : 32;
  static constexpr int ACC = TA * TA;
  static constexpr int TILE = TR * T;  // doubles per tile
  static constexpr int GLa = ACC >= 32 ? 1 : 32 / ACC;
  static constexpr int GLb = (32768 / (TILE * 8)) > 0 ? 32768 / (TILE * 8) : 1;
  static constexpr int GL = GLa < GLb ? GLa : GLb;
};

size_t tn_partials_stride(int t, int nl, bool has_v) { return (size_t)nl * t * t + (has_v ? t : 0); }

template <int T>
__device__ __forceinline__ void load_tile(double* __restrict__ s, const double* __restrict__ g,
                                          int64_t row, int64_t rows_avail, int TR) {
  // copy rows [row, row+TR) (only the first rows_avail exist) of a row-major n×T block
  const int nvalid = (int)(rows_avail < TR ? (rows_avail > 0 ? rows_avail : 0) : TR);
  if constexpr (T >= 2) {
    const double2* src = reinterpret_cast<const double2*>(g + row * T);
    double2* dst = reinterpret_cast<double2*>(s);
    const int nv = nvalid * T / 2, ntot = TR * T / 2;
    for (int e = threadIdx.x; e < ntot; e += blockDim.x)
      dst[e] = e < nv ? __ldg(src + e) : make_double2(0.0, 0.0);
  } else {
    for (int e = threadIdx.x; e < TR; e += blockDim.x) s[e] = e < nvalid ? __ldg(g + row + e) : 0.0;
  }
}

template <int T>
__global__ void __launch_bounds__(kThreads) k_tn_partials(int64_t n, int nl, PtrList L, const double* __restrict__ R,
                                                          const double* __restrict__ v, double* __restrict__ part,
                                                          size_t stride, int j0) {
  using C = TnCfg<T>;
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int ks = tid / C::TPS, tin = tid % C::TPS;
  const int ia = tin / C::NA, ib = tin % C::NA;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  double* sR = smem;
  double* sL = smem + C::TILE;
  double* sV = sL + C::GL * C::TILE;  // TR doubles (only if v)
  const bool has_v = v != nullptr;
  double* outb = part + (size_t)blockIdx.x * stride;

  for (int g0 = 0; g0 < nl; g0 += C::GL) {
    const int gn = (nl - g0) < C::GL ? (nl - g0) : C::GL;
    const bool vhere = has_v && g0 == 0;
    double acc[C::GL][C::TA][C::TA];
    double accv[C::TA];
#pragma unroll
    for (int j = 0; j < C::GL; ++j)
#pragma unroll
      for (int x = 0; x < C::TA; ++x)
#pragma unroll
        for (int y = 0; y < C::TA; ++y) acc[j][x][y] = 0.0;
#pragma unroll
    for (int x = 0; x < C::TA; ++x) accv[x] = 0.0;

    for (int64_t row = lo; row < hi; row += C::TR) {
      const int64_t avail = hi - row;
      load_tile<T>(sR, R, row, avail, C::TR);
      for (int j = 0; j < gn; ++j) load_tile<T>(sL + j * C::TILE, L.p[g0 + j], row, avail, C::TR);
      if (vhere)
        for (int e = tid; e < C::TR; e += blockDim.x) sV[e] = e < avail ? __ldg(v + row + e) : 0.0;
      __syncthreads();
      for (int rr = ks; rr < C::TR; rr += C::KS) {
        double rv[C::TA];
#pragma unroll
        for (int y = 0; y < C::TA; ++y) rv[y] = sR[rr * T + ib * C::TA + y];
#pragma unroll
        for (int j = 0; j < C::GL; ++j) {
          if (j < gn) {
            double lv[C::TA];
#pragma unroll
            for (int x = 0; x < C::TA; ++x) lv[x] = sL[j * C::TILE + rr * T + ia * C::TA + x];
#pragma unroll
            for (int x = 0; x < C::TA; ++x)
#pragma unroll
              for (int y = 0; y < C::TA; ++y) acc[j][x][y] = __fma_rn(lv[x], rv[y], acc[j][x][y]);
            if (j == 0 && vhere && ib == 0) {
              const double vv = sV[rr];
#pragma unroll
              for (int x = 0; x < C::TA; ++x) accv[x] = __fma_rn(lv[x], vv, accv[x]);
            }
          }
        }
      }
      __syncthreads();
    }
    // fixed-order reduction of the KS slices through shared memory; block j of
    // this group lands at (g0+j)*T*T, the v part (only with nl == 1) at nl*T*T.
    const int per = gn * T * T + (vhere ? T : 0);
    const int RB = (4160 / per) > 0 ? 4160 / per : 1;
    double* sred = smem;  // reuse of the tile area (>= 4160 doubles, see tn_smem_bytes)
    for (int c0 = 0; c0 < C::KS; c0 += RB) {
      if (ks >= c0 && ks < c0 + RB) {
        double* dst = sred + (size_t)(ks - c0) * per;
#pragma unroll
        for (int j = 0; j < C::GL; ++j)
          if (j < gn)
#pragma unroll
            for (int x = 0; x < C::TA; ++x)
#pragma unroll
              for (int y = 0; y < C::TA; ++y) dst[j * T * T + (ia * C::TA + x) * T + ib * C::TA + y] = acc[j][x][y];
        if (vhere && ib == 0)
#pragma unroll
          for (int x = 0; x < C::TA; ++x) dst[gn * T * T + ia * C::TA + x] = accv[x];
      }
      __syncthreads();
      const int nk = (C::KS - c0) < RB ? (C::KS - c0) : RB;
      for (int e = tid; e < per; e += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nk; ++k) s += sred[(size_t)k * per + e];
        const size_t o = e < gn * T * T ? (size_t)g0 * T * T + e : (size_t)nl * T * T + (e - gn * T * T);
        if (c0 == 0) outb[o] = s; else outb[o] += s;
      }
      __syncthreads();
    }
  }
}

template <int T>
static size_t tn_smem_bytes() {
  using C = TnCfg<T>;
  size_t tiles = (size_t)(1 + C::GL) * C::TILE * 8 + (size_t)C::TR * 8;
  size_t red = 4160 * 8;
  return tiles > red ? tiles : red;
}

cudaError_t launch_tn_partials(cudaStream_t st, int t, int64_t n, int nl, const double* const* Lhost,
                               const double* R, const double* v, double* part, int nblk) {
  if (nl <= 0) return cudaSuccess;
  if (v != nullptr && nl != 1) return cudaErrorInvalidValue;  // v only with a single left block
  const size_t stride = tn_partials_stride(t, nl, v != nullptr);
  for (int j0 = 0; j0 < nl; j0 += kMaxList) {
    const int cnt = (nl - j0) < kMaxList ? (nl - j0) : kMaxList;
    PtrList pl{};
    for (int j = 0; j < cnt; ++j) pl.p[j] = Lhost[j0 + j];
    // partial layout per CTA: [nl][T][T] then [T] (v); this launch writes blocks j0..j0+cnt-1
    EKS_DISPATCH_T(t, {
      size_t sm = tn_smem_bytes<T>();
      cudaFuncSetAttribute(k_tn_partials<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      // offset the partial pointer so that block j0 lands at j0; v part only with j0 == 0
      k_tn_partials<T><<<nblk, kThreads, sm, st>>>(n, cnt, pl, R, j0 == 0 ? v : nullptr,
                                                   part + (size_t)j0 * T * T, stride, 0);
    });
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ============================================================================
// Fixed-order reduction of per-CTA partials.
// ============================================================================
__global__ void k_reduce(const double* __restrict__ part, int nblk, size_t stride, size_t count,
                         double* __restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(size_t)b * stride + e];
    out[e] = s;
  }
}

// 32 consecutive entries per CTA (coalesced), the 8 warps split the CTA partials
// (warp w takes b ≡ w mod 8, ascending), then warps are combined in order.
__global__ void __launch_bounds__(256) k_reduce32(const double* __restrict__ part, int nblk, size_t stride,
                                                  size_t count, double* __restrict__ out) {
  __shared__ double s[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t e = (size_t)blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (e < count) {
    // 8 independent loads in flight per lane, then summed in ascending b order
    for (int b0 = w; b0 < nblk; b0 += 64) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int b = b0 + 8 * k;
        v[k] = b < nblk ? __ldg(part + (size_t)b * stride + e) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
  }
  s[w][lane] = acc;
  __syncthreads();
  if (w == 0 && e < count) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += s[k][lane];
    out[e] = t;
  }
}

cudaError_t launch_reduce(cudaStream_t st, const double* part, int nblk, size_t stride, size_t count,
                          double* out) {
  if (count == 0) return cudaSuccess;
  k_reduce32<<<(int)((count + 31) / 32), 256, 0, st>>>(part, nblk, stride, count, out);
  return cudaGetLastError();
}

// ============================================================================
// CGS update Zout = Zin − Σ_j Q_j C_j.  Each thread owns CPT
// consecutive columns of RPT rows of a TRU-row tile; Q_j tiles and the C_j
// blocks are staged in shared memory.
// ============================================================================
template <int T>
struct UpCfg {
  static constexpr int CPT = T >= 64 ? 8 : (T == 32 ? 4 : (T == 16 ? 2 : 1));
  static constexpr int TPR = T / CPT;                 // threads per row
  static constexpr int RPP = kThreads / TPR;          // rows per pass
  static constexpr int TRU = T >= 64 ? 64 : RPP;      // rows per tile
  static constexpr int RPT = TRU / RPP;               // rows per thread
  static constexpr int CJ = (49152 / (T * T * 8)) < kMaxList ? (49152 / (T * T * 8)) : kMaxList;
};

template <int T>
__global__ void __launch_bounds__(kThreads) k_ts_update(int64_t n, int nq, PtrList Q, const double* __restrict__ Cm,
                                                        const double* Zin, double* Zout) {
  using U = UpCfg<T>;
  extern __shared__ double smem[];
  double* sQ = smem;                 // TRU*T
  double* sC = smem + U::TRU * T;    // CJ*T*T
  const int tid = threadIdx.x;
  const int rloc = tid / U::TPR, c0 = (tid % U::TPR) * U::CPT;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const int nchunk = (nq + U::CJ - 1) / U::CJ;
  if (nchunk == 1) {
    for (int e = tid; e < nq * T * T; e += blockDim.x) sC[e] = Cm[e];
    __syncthreads();
  }
  for (int64_t row = lo; row < hi; row += U::TRU) {
    const int64_t avail = hi - row;
    double acc[U::RPT][U::CPT];
#pragma unroll
    for (int q = 0; q < U::RPT; ++q)
#pragma unroll
      for (int c = 0; c < U::CPT; ++c) acc[q][c] = 0.0;
    for (int ch = 0; ch < nchunk; ++ch) {
      const int jb = ch * U::CJ, je = (jb + U::CJ) < nq ? jb + U::CJ : nq;
      if (nchunk > 1) {
        __syncthreads();
        for (int e = tid; e < (je - jb) * T * T; e += blockDim.x) sC[e] = Cm[(size_t)jb * T * T + e];
      }
      for (int j = jb; j < je; ++j) {
        __syncthreads();
        load_tile<T>(sQ, Q.p[j], row, avail, U::TRU);
        __syncthreads();
        const double* Cj = sC + (size_t)(j - jb) * T * T;
#pragma unroll
        for (int q = 0; q < U::RPT; ++q) {
          const int rr = rloc + q * U::RPP;
#pragma unroll 4
          for (int a = 0; a < T; ++a) {
            const double qa = sQ[rr * T + a];
#pragma unroll
            for (int c = 0; c < U::CPT; ++c) acc[q][c] = __fma_rn(qa, Cj[a * T + c0 + c], acc[q][c]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < U::RPT; ++q) {
      const int64_t r = row + rloc + q * U::RPP;
      if (r < hi) {
#pragma unroll
        for (int c = 0; c < U::CPT; ++c) Zout[r * T + c0 + c] = Zin[r * T + c0 + c] - acc[q][c];
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_ts_update(cudaStream_t st, int t, int64_t n, int nq, const double* const* Qhost,
                             const double* C, const double* Zin, double* Zout, int nblk) {
  if (nq <= 0) {
    if (Zin != Zout) return cudaMemcpyAsync(Zout, Zin, sizeof(double) * n * t, cudaMemcpyDeviceToDevice, st);
    return cudaSuccess;
  }
  for (int j0 = 0; j0 < nq; j0 += kMaxList) {
    const int cnt = (nq - j0) < kMaxList ? (nq - j0) : kMaxList;
    PtrList pl{};
    for (int j = 0; j < cnt; ++j) pl.p[j] = Qhost[j0 + j];
    EKS_DISPATCH_T(t, {
      using U = UpCfg<T>;
      size_t sm = (size_t)(U::TRU * T + U::CJ * T * T) * 8;
      cudaFuncSetAttribute(k_ts_update<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_ts_update<T><<<nblk, kThreads, sm, st>>>(n, cnt, pl, C + (size_t)j0 * T * T, j0 == 0 ? Zin : Zout, Zout);
    });
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ============================================================================
// Small Cholesky B = RᵀR (A-CholQR), explicit R⁻¹, alpha = R⁻ᵀ g.
// Right-looking: at step k the trailing entries get B_ij -= R_ki·R_kj (product
// rounded, then subtracted, no fma), so every entry sees exactly the
// subtractions of the oracle's left-looking loop in the same order — R is
// bitwise equal to or_chol for equal B (reading R20), while each step is one
// parallel sweep instead of a serial dot product.  Breakdown: pivot <= t·2^-52·max|B| (R6).
// R⁻¹ by the mirrored right-looking backward substitution.
// ============================================================================
template <int T>
__global__ void __launch_bounds__(256) k_chol(const double* __restrict__ B, const double* __restrict__ g,
                                              double* __restrict__ Rout, double* __restrict__ Rinv,
                                              double* __restrict__ alpha, int* flag, int gblock) {
  extern __shared__ double csm[];
  double(*sA)[T + 1] = reinterpret_cast<double(*)[T + 1]>(csm);                  // trailing matrix
  double(*sR)[T + 1] = reinterpret_cast<double(*)[T + 1]>(csm + T * (T + 1));      // R
  double(*sY)[T + 1] = reinterpret_cast<double(*)[T + 1]>(csm + 2 * T * (T + 1));  // R⁻¹
  __shared__ double sred[8];
  __shared__ double sg[T];
  __shared__ int sfail;
  const int tid = threadIdx.x, nth = blockDim.x;
  double m = 0.0;
  for (int e = tid; e < T * T; e += nth) {
    const int i = e / T, j = e % T;
    const double b = B[e];
    sA[i][j] = b;
    sR[i][j] = 0.0;
    sY[i][j] = (i == j) ? 1.0 : 0.0;
    if (j >= i) m = fmax(m, fabs(b));
  }
  if (g != nullptr && tid < T) sg[tid] = g[tid];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) sred[tid >> 5] = m;
  if (tid == 0) sfail = 0;
  __syncthreads();
  double bm = 0.0;
  for (int w = 0; w < (nth >> 5); ++w) bm = fmax(bm, sred[w]);
  const double thr = __dmul_rn((double)T * 0x1p-52, bm);
  for (int k = 0; k < T; ++k) {
    if (tid == 0) {
      const double d = sA[k][k];
      if (!(d > thr)) sfail = 1;
      sR[k][k] = __dsqrt_rn(d);
    }
    __syncthreads();
    const double rkk = sR[k][k];
    for (int j = k + 1 + tid; j < T; j += nth) sR[k][j] = __ddiv_rn(sA[k][j], rkk);
    __syncthreads();
    const int m1 = T - k - 1;  // trailing upper triangle (i <= j, both > k)
    for (int e = tid; e < m1 * m1; e += nth) {
      const int i = k + 1 + e / m1, j = k + 1 + e % m1;
      if (j >= i) sA[i][j] = __dsub_rn(sA[i][j], __dmul_rn(sR[k][i], sR[k][j]));
    }
    __syncthreads();
  }
  // R X = I, X upper triangular: X_k· = Y_k· / R_kk, then Y_i· -= R_ik X_k· for i < k (k descending)
  for (int k = T - 1; k >= 0; --k) {
    const double rkk = sR[k][k];
    for (int j = k + tid; j < T; j += nth) sY[k][j] = __ddiv_rn(sY[k][j], rkk);
    __syncthreads();
    const int w = T - k;
    for (int e = tid; e < k * w; e += nth) {
      const int i = e / w, j = k + e % w;
      sY[i][j] = __fma_rn(-sR[i][k], sY[k][j], sY[i][j]);
    }
    __syncthreads();
  }
  for (int e = tid; e < T * T; e += nth) {
    if (Rout) Rout[e] = sR[e / T][e % T];
    Rinv[e] = sY[e / T][e % T];
  }
  if (g != nullptr && alpha != nullptr) {
    // alpha = R⁻ᵀ g: alpha_j = Σ_{i<=j} Rinv[i][j] g_i
    for (int j = tid; j < T; j += nth) {
      double a = 0.0;
      for (int i = 0; i <= j; ++i) a = __fma_rn(sY[i][j], sg[i], a);
      alpha[j] = a;
    }
  }
  if (tid == 0 && sfail && flag) atomicMin(flag, gblock);
}

// t ≤ 32: one warp, the factor in registers (chol_warp, eks_device.cuh) — same operations as k_chol.
template <int T>
__global__ void __launch_bounds__(32) k_chol_w(const double* __restrict__ B, const double* __restrict__ g,
                                               double* __restrict__ Rout, double* __restrict__ Rinv,
                                               double* __restrict__ alpha, int* flag, int gblock) {
  chol_warp<T>(B, g, Rout, Rinv, alpha, flag, gblock);
}

// Solve-path Cholesky: chol_warp_fast (rsqrt pivots, R within a few ulps of launch_chol).
template <int T>
__global__ void __launch_bounds__(32) k_chol_fast(const double* __restrict__ B, const double* __restrict__ g,
                                                  double* __restrict__ Rout, double* __restrict__ Rinv,
                                                  double* __restrict__ alpha, int* flag, int gblock) {
  pdl_enter();
  const int j = threadIdx.x;
  double a[T], y[T];
  const bool fail = chol_warp_fast<T>(B, a, y);
  if (j < T) {
#pragma unroll
    for (int i = 0; i < T; ++i) {
      if (Rout) Rout[i * T + j] = (i <= j) ? a[i] : 0.0;
      Rinv[i * T + j] = y[i];
    }
    if (g != nullptr && alpha != nullptr) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < T; ++i)
        if (i <= j) s = __fma_rn(y[i], __ldcg(g + i), s);
      alpha[j] = s;
    }
  }
  if (fail && j == 0 && flag) atomicMin(flag, gblock);
}

cudaError_t launch_chol_fast(cudaStream_t st, int t, const double* B, const double* g, double* R, double* Rinv,
                             double* alpha, int* flag, int gblock) {
  switch (t) {
    case 1: return launch_k(k_chol_fast<1>, 1, 32, 0, st, B, g, R, Rinv, alpha, flag, gblock);
    case 2: return launch_k(k_chol_fast<2>, 1, 32, 0, st, B, g, R, Rinv, alpha, flag, gblock);
    case 4: return launch_k(k_chol_fast<4>, 1, 32, 0, st, B, g, R, Rinv, alpha, flag, gblock);
    case 8: return launch_k(k_chol_fast<8>, 1, 32, 0, st, B, g, R, Rinv, alpha, flag, gblock);
    case 16: return launch_k(k_chol_fast<16>, 1, 32, 0, st, B, g, R, Rinv, alpha, flag, gblock);
    case 32: return launch_k(k_chol_fast<32>, 1, 32, 0, st, B, g, R, Rinv, alpha, flag, gblock);
    default: return launch_chol(st, t, B, g, R, Rinv, alpha, flag, gblock);
  }
}

cudaError_t launch_chol(cudaStream_t st, int t, const double* B, const double* g, double* R, double* Rinv,
                        double* alpha, int* flag, int gblock) {
  switch (t) {
    case 1: k_chol_w<1><<<1, 32, 0, st>>>(B, g, R, Rinv, alpha, flag, gblock); return cudaGetLastError();
    case 2: k_chol_w<2><<<1, 32, 0, st>>>(B, g, R, Rinv, alpha, flag, gblock); return cudaGetLastError();
    case 4: k_chol_w<4><<<1, 32, 0, st>>>(B, g, R, Rinv, alpha, flag, gblock); return cudaGetLastError();
    case 8: k_chol_w<8><<<1, 32, 0, st>>>(B, g, R, Rinv, alpha, flag, gblock); return cudaGetLastError();
    case 16: k_chol_w<16><<<1, 32, 0, st>>>(B, g, R, Rinv, alpha, flag, gblock); return cudaGetLastError();
    case 32: k_chol_w<32><<<1, 32, 0, st>>>(B, g, R, Rinv, alpha, flag, gblock); return cudaGetLastError();
    default: break;
  }
  EKS_DISPATCH_T(t, {
    const size_t sm = (size_t)3 * T * (T + 1) * 8;
    cudaFuncSetAttribute(k_chol<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_chol<T><<<1, 256, sm, st>>>(B, g, R, Rinv, alpha, flag, gblock);
  });
  return cudaGetLastError();
}

// ============================================================================
// Apply R⁻¹ and the x/r update of this block (P:159-161 / P:189-191 / P:340-342,
// α̃_b = R⁻ᵀ(Z2ᵀ r_{k-1}) so that α̃ = Vᵀ r_{k-1} blockwise).
// ============================================================================
template <int T>
__global__ void __launch_bounds__(kThreads) k_apply(int64_t n, double* __restrict__ Z2W, double* __restrict__ AZ2AW,
                                                    const double* __restrict__ Rinv, const double* __restrict__ alpha,
                                                    double* __restrict__ x, double* __restrict__ dx,
                                                    const double* __restrict__ r, double* __restrict__ rnew,
                                                    double* __restrict__ rho_part, const int* __restrict__ flag,
                                                    int mode) {
  using U = UpCfg<T>;
  extern __shared__ double smem[];
  double* sRi = smem;               // T*T
  double* sA = sRi + T * T;         // T
  double* sZ = sA + T;              // TRU*T
  double* sY = sZ + U::TRU * T;     // TRU*T
  __shared__ double sred[32];
  const int tid = threadIdx.x;
  const int rloc = tid / U::TPR, c0 = (tid % U::TPR) * U::CPT;
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  const bool first = mode & 1, last = mode & 2, basis = mode & 4;
  const bool skip = basis || (flag != nullptr && *flag != INT_MAX);
  for (int e = tid; e < T * T; e += blockDim.x) sRi[e] = Rinv[e];
  for (int e = tid; e < T; e += blockDim.x) sA[e] = alpha ? alpha[e] : 0.0;
  double rr_acc = 0.0;
  __syncthreads();
  for (int64_t row = lo; row < hi; row += U::TRU) {
    const int64_t avail = hi - row;
    load_tile<T>(sZ, Z2W, row, avail, U::TRU);
    load_tile<T>(sY, AZ2AW, row, avail, U::TRU);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < U::RPT; ++q) {
      const int rr = rloc + q * U::RPP;
      const int64_t rg = row + rr;
      double w[U::CPT], aw[U::CPT];
#pragma unroll
      for (int c = 0; c < U::CPT; ++c) { w[c] = 0.0; aw[c] = 0.0; }
      for (int a = 0; a < c0 + U::CPT; ++a) {
        const double za = sZ[rr * T + a], ya = sY[rr * T + a];
#pragma unroll
        for (int c = 0; c < U::CPT; ++c) {
          const double ri = sRi[a * T + c0 + c];
          w[c] = __fma_rn(za, ri, w[c]);
          aw[c] = __fma_rn(ya, ri, aw[c]);
        }
      }
      double u = 0.0, qv = 0.0;
#pragma unroll
      for (int c = 0; c < U::CPT; ++c) {
        u = __fma_rn(w[c], sA[c0 + c], u);
        qv = __fma_rn(aw[c], sA[c0 + c], qv);
      }
      // fixed-order sum over the TPR threads of the row (consecutive lanes)
#pragma unroll
      for (int o = U::TPR / 2; o > 0; o >>= 1) {
        u += __shfl_down_sync(0xffffffffu, u, o, U::TPR);
        qv += __shfl_down_sync(0xffffffffu, qv, o, U::TPR);
      }
      if (rg < hi) {
#pragma unroll
        for (int c = 0; c < U::CPT; ++c) {
          Z2W[rg * T + c0 + c] = w[c];
          AZ2AW[rg * T + c0 + c] = aw[c];
        }
        if (!skip && (tid % U::TPR) == 0) {
          double dxi = first ? u : dx[rg] + u;
          double rn = first ? r[rg] - qv : rnew[rg] - qv;
          rnew[rg] = rn;
          if (last) {
            x[rg] += dxi;
            rr_acc = __fma_rn(rn, rn, rr_acc);
          } else {
            dx[rg] = dxi;
          }
        }
      }
    }
    __syncthreads();
  }
  if (last && rho_part != nullptr) {
    double s = block_sum(rr_acc, sred);
    if (tid == 0) rho_part[blockIdx.x] = s;
  }
}

cudaError_t launch_apply(cudaStream_t st, int t, int64_t n, double* Z2W, double* AZ2AW, const double* Rinv,
                         const double* alpha, double* x, double* dx, const double* r, double* rnew,
                         double* rho_part, const int* flag, int mode, int nblk) {
  EKS_DISPATCH_T(t, {
    using U = UpCfg<T>;
    size_t sm = (size_t)(T * T + T + 2 * U::TRU * T) * 8;
    cudaFuncSetAttribute(k_apply<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_apply<T><<<nblk, kThreads, sm, st>>>(n, Z2W, AZ2AW, Rinv, alpha, x, dx, r, rnew, rho_part, flag, mode);
  });
  return cudaGetLastError();
}


// ============================================================================
// Communication-avoiding variants (CA SRE-CG / CA SRE-CG2 / CA MSDO-CG):
// the s·t columns of an outer iteration are A-orthonormalized by ONE CholQR.
// ============================================================================
// Cholesky of the m×m Gram (m = s·t ≤ kCaMax), R⁻¹ and α̃ = R⁻ᵀ g: k_chol's right-looking
// elimination (R bitwise equal to the oracle's or_chol for equal B, reading R20) at run-time size.
template <bool G>
__global__ void __launch_bounds__(1024) k_chol_dyn(int m, const double* __restrict__ B, const double* __restrict__ g,
                                                   double* __restrict__ Rout, double* __restrict__ Rinv,
                                                   double* __restrict__ alpha, int* flag, int gblock, double* gwork) {
  pdl_enter();
  extern __shared__ double csm[];
  const int M1 = m + 1;
  double* sA = gwork ? gwork : csm;  // m × (m+1): shared memory, or global above kCaSmem columns
  double* sY = sA + m * M1;          // m × (m+1)
  __shared__ double sred[32];
  __shared__ int sfail;
  const int tid = threadIdx.x, nth = blockDim.x;
  double mx = 0.0;
  for (int e = tid; e < m * m; e += nth) {
    const int i = e / m, j = e % m;
    const double b = B[e];
    sA[i * M1 + j] = b;
    sY[i * M1 + j] = (i == j) ? 1.0 : 0.0;
    if (j >= i) mx = fmax(mx, fabs(b));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) sred[tid >> 5] = mx;
  if (tid == 0) sfail = 0;
  __syncthreads();
  double bm = 0.0;
  for (int w = 0; w < (nth >> 5); ++w) bm = fmax(bm, sred[w]);
  const double thr = __dmul_rn((double)m * 0x1p-52, bm);
  __shared__ double srkk;
  for (int k = 0; k < m; ++k) {
    if (tid == 0) {
      const double d = sA[k * M1 + k];
      if (!(d > thr)) sfail = 1;
      srkk = __dsqrt_rn(d);
      sA[k * M1 + k] = srkk;
    }
    __syncthreads();
    const double rkk = srkk;
    for (int j = k + 1 + tid; j < m; j += nth) sA[k * M1 + j] = __ddiv_rn(sA[k * M1 + j], rkk);
    __syncthreads();
    const int m1 = m - k - 1;
    for (int e = tid; e < m1 * m1; e += nth) {
      const int i = k + 1 + e / m1, j = k + 1 + e % m1;
      if (j >= i) sA[i * M1 + j] = __dsub_rn(sA[i * M1 + j], __dmul_rn(sA[k * M1 + i], sA[k * M1 + j]));
    }
    __syncthreads();
  }
  for (int k = m - 1; k >= 0; --k) {
    const double rkk = sA[k * M1 + k];
    for (int j = k + tid; j < m; j += nth) sY[k * M1 + j] = __ddiv_rn(sY[k * M1 + j], rkk);
    __syncthreads();
    const int w = m - k;
    for (int e = tid; e < k * w; e += nth) {
      const int i = e / w, j = k + e % w;
      sY[i * M1 + j] = __fma_rn(-sA[i * M1 + k], sY[k * M1 + j], sY[i * M1 + j]);
    }
    __syncthreads();
  }
  for (int e = tid; e < m * m; e += nth) {
    const int i = e / m, j = e % m;
    if (Rout) Rout[e] = j >= i ? sA[i * M1 + j] : 0.0;
    Rinv[e] = sY[i * M1 + j];
  }
  if (G && alpha != nullptr)
    for (int j = tid; j < m; j += nth) {
      double a = 0.0;
      for (int i = 0; i <= j; ++i) a = __fma_rn(sY[i * M1 + j], g[i], a);
      alpha[j] = a;
    }
  if (tid == 0 && sfail && flag) atomicMin(flag, gblock);
}

size_t chol_dyn_work(int m) { return m > kCaSmem ? (size_t)2 * m * (m + 1) : 0; }

cudaError_t launch_chol_dyn(cudaStream_t st, int m, const double* B, const double* g, double* R, double* Rinv,
                            double* alpha, int* flag, int gblock, double* work) {
  if (m < 1 || m > kCaMax) return cudaErrorInvalidValue;
  const bool glob = m > kCaSmem;
  if (glob && !work) return cudaErrorInvalidValue;
  const size_t sm = glob ? 0 : (size_t)2 * m * (m + 1) * 8;
  const int nth = glob ? 1024 : 256;
  if (g) {
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_chol_dyn<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    return launch_k(k_chol_dyn<true>, 1, nth, sm, st, m, B, g, R, Rinv, alpha, flag, gblock, glob ? work : nullptr);
  }
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_chol_dyn<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  return launch_k(k_chol_dyn<false>, 1, nth, sm, st, m, B, g, R, Rinv, alpha, flag, gblock, glob ? work : nullptr);
}

// out_j = Σ_{i ≤ j} in_i · Rinv[i·t.., j·t..] for the s blocks (W = V R⁻¹ and AW = AV R⁻¹ of the
// st-column CholQR, R upper so only i ≤ j contributes).  R⁻¹ in shared memory; a thread owns one
// (row, column) and all s output blocks.
__global__ void __launch_bounds__(256) k_ca_combine(int64_t n, int t, int s, CaPtrs P, const double* __restrict__ Rinv,
                                                    int skip) {
  pdl_enter();
  extern __shared__ double sR[];
  const int m = s * t;
  if (skip != 0 && *reinterpret_cast<const volatile int*>(P.flag) != INT_MAX) return;  // breakdown
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sR[e] = Rinv[e];
  __syncthreads();
  const int rows_per = blockDim.x / t;
  const int c = threadIdx.x % t, rl = threadIdx.x / t;
  if (rl >= rows_per) return;
  for (int64_t row = (int64_t)blockIdx.x * rows_per + rl; row < n; row += (int64_t)gridDim.x * rows_per) {
    for (int j = 0; j < s; ++j) {
      double acc = 0.0;
      for (int i = 0; i <= j; ++i) {
        const double* v = P.in[i] + row * t;
        const double* rr = sR + (size_t)(i * t) * m + j * t + c;
        for (int a = 0; a < t; ++a) acc = __fma_rn(__ldg(v + a), rr[(size_t)a * m], acc);
      }
      P.out[j][row * t + c] = acc;
    }
  }
}

cudaError_t launch_ca_combine(cudaStream_t st, int64_t n, int t, int s, const CaPtrs& P, const double* Rinv,
                              int sms, bool skip_on_breakdown) {
  const int m = s * t;
  if (m > kCaMax || s > kCaMaxBlocks) return cudaErrorInvalidValue;
  const size_t sm = (size_t)m * m * 8;
  cudaFuncSetAttribute(k_ca_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int rows_per = 256 / t;
  int64_t blocks = (n + rows_per - 1) / rows_per;
  if (blocks > (int64_t)sms * 4) blocks = (int64_t)sms * 4;
  return launch_k(k_ca_combine, (int)blocks, 256, sm, st, n, t, s, P, Rinv, skip_on_breakdown ? 1 : 0);
}

// Block-diagonal triangular solve of an n×t block with a level schedule (block-Jacobi IC(0),
// Alg 8-10 M⁻¹ = L⁻ᵗL⁻¹, reading R32): one CTA per preconditioner domain walks its levels in
// order; a level's rows are independent: Y[i][c] = (Z[i][c] − Σ_p val[p]·Y[col[p]][c]) / diag[i]
// (p ascending, fma).  Y may alias Z (row i reads only its own Z entry).  The same kernel runs the
// forward (strict lower L) and the backward (strict upper Lᵗ, levels from the last row) sweep.
__global__ void __launch_bounds__(256) k_trsv_lev(int t, const int* __restrict__ rp, const int* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ diag,
                                                  const int* __restrict__ dom_lev, const int* __restrict__ lev_ptr,
                                                  const int* __restrict__ rows, const double* Z, double* Y) {
  pdl_enter();
  const int d = blockIdx.x;
  for (int lv = dom_lev[d]; lv < dom_lev[d + 1]; ++lv) {
    const int b = lev_ptr[lv], items = (lev_ptr[lv + 1] - b) * t;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int i = rows[b + it / t], c = it % t;
      double v = Z[(int64_t)i * t + c];
      for (int p = rp[i]; p < rp[i + 1]; ++p) v = __fma_rn(-val[p], Y[(int64_t)col[p] * t + c], v);
      Y[(int64_t)i * t + c] = __ddiv_rn(v, diag[i]);
    }
    __syncthreads();
  }
}

// The same for long rows (complete-Cholesky envelopes, hundreds of entries per row): a warp per
// (row, column) item, the lanes split the row's entries, a butterfly reduces them.
__global__ void __launch_bounds__(512) k_trsv_lev_long(int t, const int* __restrict__ rp, const int* __restrict__ col,
                                                       const double* __restrict__ val, const double* __restrict__ diag,
                                                       const int* __restrict__ dom_lev, const int* __restrict__ lev_ptr,
                                                       const int* __restrict__ rows, const double* Z, double* Y) {
  pdl_enter();
  const int d = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int lv = dom_lev[d]; lv < dom_lev[d + 1]; ++lv) {
    const int b = lev_ptr[lv], items = (lev_ptr[lv + 1] - b) * t;
    for (int it = warp; it < items; it += nw) {
      const int i = rows[b + it / t], c = it % t;
      double v = 0.0;
      for (int p = rp[i] + lane; p < rp[i + 1]; p += 32) v = __fma_rn(val[p], Y[(int64_t)col[p] * t + c], v);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) Y[(int64_t)i * t + c] = __ddiv_rn(Z[(int64_t)i * t + c] - v, diag[i]);
    }
    __syncthreads();
  }
}

cudaError_t launch_trsv_lev_long(cudaStream_t st, int ndom, int t, const int* rp, const int* col, const double* val,
                                 const double* diag, const int* dom_lev, const int* lev_ptr, const int* rows,
                                 const double* Z, double* Y) {
  if (ndom < 1 || t < 1) return cudaErrorInvalidValue;
  return launch_k(k_trsv_lev_long, ndom, 512, 0, st, t, rp, col, val, diag, dom_lev, lev_ptr, rows, Z, Y);
}

cudaError_t launch_trsv_lev(cudaStream_t st, int ndom, int t, const int* rp, const int* col, const double* val,
                            const double* diag, const int* dom_lev, const int* lev_ptr, const int* rows,
                            const double* Z, double* Y) {
  if (ndom < 1 || t < 1) return cudaErrorInvalidValue;
  return launch_k(k_trsv_lev, ndom, 256, 0, st, t, rp, col, val, diag, dom_lev, lev_ptr, rows, Z, Y);
}

// The same sweep with the solved rows kept in a shared-memory ring of W rows (slot = row mod W):
// the setup chose W so that a row's slot is rewritten only at a later level than its last reader
// (eks.cu, ring width).  Everything an item needs is addressed by its schedule position: the
// level bounds (staged in shared memory), the flattened schedule (row, output index, #entries,
// diagonal, ≤ E entries) and the input block, which arrives already permuted into schedule order
// (k_perm_gather for the forward sweep; the forward sweep writes its result in the backward
// schedule's order).  So no load waits on another, and every thread keeps the items of the next
// kTrsvD levels in flight: a level costs shared-memory reads and one barrier.
constexpr int kTrsvD = 4;
template <int E>
struct TrsvItem {
  int i, o, ne;
  double z, rd;
  int k[E];
  double v[E];
};

struct TrsvSched {  // flattened schedule of one sweep
  const int* pos_row;
  const int* pos_out;     // output row index (forward: position in the backward schedule; backward: row)
  const int* pos_ne;
  const double* pos_rdiag;  // 1 / L_ii
  const int* pos_col;     // pos * E + e
  const double* pos_val;  // pos * E + e
};

template <int E>
__device__ __forceinline__ void trsv_load(TrsvItem<E>& f, int pos, int c, int t, const TrsvSched& S, const double* Zp) {
  f.i = __ldg(S.pos_row + pos);
  f.o = __ldg(S.pos_out + pos);
  f.ne = __ldg(S.pos_ne + pos);
  f.rd = __ldg(S.pos_rdiag + pos);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    f.k[e] = __ldg(S.pos_col + (size_t)pos * E + e);
    f.v[e] = __ldg(S.pos_val + (size_t)pos * E + e);
  }
  f.z = Zp[(int64_t)pos * t + c];
}

// cl: column within the CTA's column group (ring stride rs), c: global column (Y stride t)
template <int E>
__device__ __forceinline__ void trsv_solve(const TrsvItem<E>& f, int cl, int c, double* ring, int wmask, int rs, int t,
                                           double* Y) {
  double v = f.z;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e < f.ne) v = __fma_rn(-f.v[e], ring[(f.k[e] & wmask) * rs + cl], v);
  v = v * f.rd;
  ring[(f.i & wmask) * rs + cl] = v;
  Y[(int64_t)f.o * t + c] = v;
}

// The t columns of the block are independent right-hand sides: CTA b solves domain b / ngrp for the
// column group (b % ngrp)·cpg … +cpg.  With a level's items (rows × cpg) within one warp the CTA is
// one warp and the per-level barrier is a warp barrier.
template <int E>
__global__ void __launch_bounds__(256) k_trsv_ring(int t, int cpg, int ngrp, int wmask, const TrsvSched S,
                                                   const int* __restrict__ dom_lev,
                                                   const int* __restrict__ lev_ptr, const double* Zp, double* Y) {
  pdl_enter();
  extern __shared__ double ring[];  // (wmask + 1) × cpg doubles, then the domain's level bounds
  int* slev = reinterpret_cast<int*>(ring + (size_t)(wmask + 1) * cpg);
  const int d = blockIdx.x / ngrp, c0 = (blockIdx.x % ngrp) * cpg, tid = threadIdx.x, nth = blockDim.x;
  const int l0 = dom_lev[d], l1 = dom_lev[d + 1];
  for (int e = tid; e <= l1 - l0; e += nth) slev[e] = lev_ptr[l0 + e];
  __syncthreads();
  const int prow = tid / cpg, cl = tid % cpg;  // this thread's (row in level, column) of a level's first nth items
  TrsvItem<E> q[kTrsvD];
  bool h[kTrsvD];
#pragma unroll
  for (int u = 0; u < kTrsvD; ++u) {
    const int L = l0 + u;
    h[u] = L < l1 && prow < slev[L - l0 + 1] - slev[L - l0];
    if (h[u]) trsv_load(q[u], slev[L - l0] + prow, c0 + cl, t, S, Zp);
  }
  for (int lv = l0; lv < l1; lv += kTrsvD) {
#pragma unroll
    for (int u = 0; u < kTrsvD; ++u) {
      const int L = lv + u;
      if (L < l1) {  // uniform across the CTA
        if (h[u]) trsv_solve(q[u], cl, c0 + cl, ring, wmask, cpg, t, Y);
        const int b = slev[L - l0], items = (slev[L - l0 + 1] - b) * cpg;
        for (int it = tid + nth; it < items; it += nth) {  // wide levels: the rest without prefetch
          TrsvItem<E> f;
          trsv_load(f, b + it / cpg, c0 + it % cpg, t, S, Zp);
          trsv_solve(f, it % cpg, c0 + it % cpg, ring, wmask, cpg, t, Y);
        }
        const int Ln = L + kTrsvD;
        h[u] = Ln < l1 && prow < slev[Ln - l0 + 1] - slev[Ln - l0];
        if (h[u]) trsv_load(q[u], slev[Ln - l0] + prow, c0 + cl, t, S, Zp);
        if (nth == 32) __syncwarp();
        else __syncthreads();
      }
    }
  }
}

// Zp[pos] = Z[row(pos)] for every schedule position (the forward sweep's input in its order).
__global__ void __launch_bounds__(256) k_perm_gather(int64_t npos, int t, const int* __restrict__ pos_row,
                                                     const double* __restrict__ Z, double* __restrict__ Zp) {
  pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npos * t; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = e / t;
    const int c = (int)(e % t);
    Zp[e] = Z[(int64_t)__ldg(pos_row + pos) * t + c];
  }
}

cudaError_t launch_perm_gather(cudaStream_t st, int64_t npos, int t, const int* pos_row, const double* Z,
                               double* Zp, int sms) {
  const int64_t total = npos * t;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (blocks < 1) blocks = 1;
  return launch_k(k_perm_gather, (int)blocks, 256, 0, st, npos, t, pos_row, Z, Zp);
}

// columns per CTA: the largest power-of-two divisor of t with a level's items (maxrows × cpg) in one
// warp (EKS_TRSV_CPG overrides, A/B measurements); t itself when even one column's level exceeds a warp
static int trsv_cpg(int t, int maxrows) {
  static const int env = [] {
    const char* e = getenv("EKS_TRSV_CPG");
    return e ? atoi(e) : 0;
  }();
  if (env > 0 && env <= t && t % env == 0) return env;
  int cpg = t;
  while (cpg > 1 && maxrows * cpg > 32) cpg /= 2;
  return maxrows * cpg <= 32 ? cpg : t;
}

size_t trsv_ring_smem(int wrows, int t, int maxlev) { return (size_t)wrows * t * 8 + (size_t)(maxlev + 1) * 4; }

cudaError_t launch_trsv_ring(cudaStream_t st, int ndom, int t, int wrows, int maxlev, int maxrows,
                             const int* pos_row, const int* pos_out, const int* pos_ne, const double* pos_rdiag,
                             const int* pos_col, const double* pos_val, int E, const int* dom_lev, const int* lev_ptr,
                             const double* Zp, double* Y) {
  if (ndom < 1 || t < 1 || wrows < 1 || (wrows & (wrows - 1))) return cudaErrorInvalidValue;
  const int cpg = trsv_cpg(t, maxrows), ngrp = t / cpg;
  const size_t sm = trsv_ring_smem(wrows, cpg, maxlev);
  if (sm > 220 * 1024) return cudaErrorInvalidValue;
  // threads: a level's items (rows × cpg), rounded to warps, at most 256; wider levels loop
  int nth = ((maxrows * cpg + 31) / 32) * 32;
  if (nth > 256) nth = 256;
  if (nth < 32) nth = 32;
  const TrsvSched S{pos_row, pos_out, pos_ne, pos_rdiag, pos_col, pos_val};
#define EKS_TRSV_E(EE)                                                                                            \
  case EE:                                                                                                        \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_trsv_ring<EE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    return launch_k(k_trsv_ring<EE>, ndom * ngrp, nth, sm, st, t, cpg, ngrp, wrows - 1, S, dom_lev, lev_ptr, Zp, Y);
  switch (E) {
    EKS_TRSV_E(1)
    EKS_TRSV_E(2)
    EKS_TRSV_E(3)
    EKS_TRSV_E(4)
    EKS_TRSV_E(8)
    default: return cudaErrorInvalidValue;
  }
#undef EKS_TRSV_E
}

// Per-CTA partials of Wᵀv (t values per CTA, part[b·t + c]) over the CTA's contiguous rows; a
// warp owns 32/L consecutive rows per step (coalesced), fixed-order lane/warp reductions.
__global__ void __launch_bounds__(256) k_wtv(int64_t n, int t, const double* __restrict__ W,
                                             const double* __restrict__ v, double* __restrict__ part) {
  pdl_enter();
  __shared__ double sacc[8][64];
  int L = 1;
  while (2 * L <= t && 2 * L <= 32) L *= 2;
  const int RPW = 32 / L, CPL = (t + L - 1) / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / L, lc = lane % L;
  const int64_t lo = (int64_t)blockIdx.x * n / gridDim.x, hi = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
  double acc[2] = {0.0, 0.0};
  for (int64_t r0 = lo + (int64_t)warp * RPW; r0 < hi; r0 += 8 * RPW) {
    const int64_t i = r0 + sub;
    if (i < hi) {
      const double vi = v[i];
      for (int q = 0; q < CPL; ++q) {
        const int c = lc + q * L;
        if (c < t) acc[q] = __fma_rn(W[i * t + c], vi, acc[q]);
      }
    }
  }
  for (int q = 0; q < CPL; ++q) {
    for (int o = 16; o >= L; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if (sub == 0 && lc + q * L < t) sacc[warp][lc + q * L] = acc[q];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sacc[w][c];
    part[(size_t)blockIdx.x * t + c] = s;
  }
}

cudaError_t launch_wtv(cudaStream_t st, int64_t n, int t, const double* W, const double* v, double* part, int nblk) {
  if (t < 1 || t > 64) return cudaErrorInvalidValue;
  return launch_k(k_wtv, nblk, 256, 0, st, n, t, W, v, part);
}

// One-synch CGS2 (DESIGN reading R36): after the single stacked reduction of
// [C2 | B1 | g1] (C2 = (AQ)ᵀZ1, B1 = Z1ᵀ(A·Z1), g1 = Z1ᵀr), with QᵀAQ = I and QᵀAZ1 = C2:
//   B = Z2ᵀAZ2 = B1 − C2ᵀC2   (upper entries, mirrored),   g = Z2ᵀr = g1 − Σ_{q ≥ qcur} C2_qᵀ α̃_q,
// where α̃_q = W_qᵀ r_{k−1} of the window blocks built in this outer iteration (abase = that of
// window block qcur; the older blocks' Wᵀr_{k−1} = 0).  One warp per output entry; its lanes
// stride the nq·t-long sum and reduce with a fixed butterfly (run-to-run reproducible).
__global__ void __launch_bounds__(256) k_onesynch_fix(int t, int nq, int qcur, const double* __restrict__ C,
                                                      const double* __restrict__ Bg1, const double* __restrict__ abase,
                                                      double* __restrict__ Bg) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int e = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nU = t * (t + 1) / 2, m = nq * t;
  if (e < nU) {
    int a = 0, rem = e;
    while (rem >= t - a) {
      rem -= t - a;
      ++a;
    }
    const int c = a + rem;
    double v = 0.0;
    for (int qa = lane; qa < m; qa += 32) v = fma(C[(size_t)qa * t + a], C[(size_t)qa * t + c], v);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) {
      const double b = Bg1[a * t + c] - v;
      Bg[a * t + c] = b;
      Bg[c * t + a] = b;
    }
  } else if (e < nU + t) {
    const int c = e - nU;
    double v = 0.0;
    if (abase)
      for (int qa = qcur * t + lane; qa < m; qa += 32) v = fma(C[(size_t)qa * t + c], abase[qa - qcur * t], v);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) Bg[t * t + c] = Bg1[t * t + c] - v;
  }
}

cudaError_t launch_onesynch_fix(cudaStream_t st, int t, int nq, int qcur, const double* C, const double* Bg1,
                                const double* abase, double* Bg) {
  const int warps = t * (t + 1) / 2 + t;
  return launch_k(k_onesynch_fix, (warps + 7) / 8, 256, 0, st, t, nq, qcur, C, Bg1, abase, Bg);
}

// Column block j of −R⁻¹ packed for the update sweeps (W_j = 0 − Σ_{i≤j} V_i·(−R⁻¹_ij)):
// pack + (j(j+1)/2)·t·t holds the t×t blocks −R⁻¹_ij, i = 0..j, each row-major (row = column of V_i).
__global__ void __launch_bounds__(256) k_ca_pack(int t, int s, const double* __restrict__ Rinv,
                                                 double* __restrict__ pack) {
  pdl_enter();
  const int m = s * t, tt = t * t;
  const int total = s * (s + 1) / 2 * tt;
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < total; e += blockDim.x * gridDim.x) {
    const int blk = e / tt, a = (e / t) % t, c = e % t;
    int j = 0;
    while ((j + 1) * (j + 2) / 2 <= blk) ++j;
    const int i = blk - j * (j + 1) / 2;
    pack[e] = -Rinv[(size_t)(i * t + a) * m + j * t + c];
  }
}

cudaError_t launch_ca_pack(cudaStream_t st, int t, int s, const double* Rinv, double* pack) {
  if (s * t > kCaMax || s > kCaMaxBlocks) return cudaErrorInvalidValue;
  const int total = s * (s + 1) / 2 * t * t;
  return launch_k(k_ca_pack, (total + 255) / 256, 256, 0, st, t, s, Rinv, pack);
}

// x += Σ_j W_j α_j, r −= Σ_j AW_j α_j (α = α̃ = R⁻ᵀ Vᵀr of the outer iteration), partial ‖r‖² per CTA;
// nothing when the breakdown flag is set (x stays the last completed iterate).
// A warp owns 32/L consecutive rows per step (L = the largest power of two ≤ min(t, 32) lanes per
// row, ⌈t/L⌉ columns per lane):
// coalesced block reads, then a butterfly over the L lanes of a row.
__global__ void __launch_bounds__(256) k_ca_update(int64_t n, int t, int s, CaPtrs P, const double* __restrict__ alpha,
                                                   double* __restrict__ x, const double* __restrict__ r,
                                                   double* __restrict__ rnew, double* __restrict__ part) {
  pdl_enter();
  __shared__ double sa[kCaMax];
  __shared__ double sred[32];
  const int m = s * t;
  const bool skip = *reinterpret_cast<const volatile int*>(P.flag) != INT_MAX;
  for (int e = threadIdx.x; e < m; e += blockDim.x) sa[e] = alpha[e];
  __syncthreads();
  int L = 1;
  while (2 * L <= t && 2 * L <= 32) L *= 2;
  const int RPW = 32 / L, CPL = (t + L - 1) / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int sub = lane / L, lc = lane % L;
  const int64_t lo = (int64_t)blockIdx.x * n / gridDim.x, hi = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
  double acc = 0.0;
  for (int64_t r0 = lo + (int64_t)warp * RPW; r0 < hi; r0 += (int64_t)nw * RPW) {
    const int64_t i = r0 + sub;
    const bool ok = i < hi;
    double dx = 0.0, dr = 0.0;
    if (ok)
      for (int j = 0; j < s; ++j)
        for (int q = 0; q < CPL; ++q) {
          const int c = lc + q * L;
          if (c >= t) break;
          dx = __fma_rn(P.in[j][i * t + c], sa[j * t + c], dx);
          dr = __fma_rn(P.out[j][i * t + c], sa[j * t + c], dr);
        }
    for (int o = L >> 1; o > 0; o >>= 1) {
      dx += __shfl_xor_sync(0xffffffffu, dx, o);
      dr += __shfl_xor_sync(0xffffffffu, dr, o);
    }
    if (ok && lc == 0) {
      double ri = r[i];
      if (!skip) {
        x[i] += dx;
        ri -= dr;
      }
      rnew[i] = ri;
      acc = __fma_rn(ri, ri, acc);
    }
  }
  const double tot = block_sum(acc, sred);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// The same with M = s·⌈t/L⌉ ≤ 4 (block, column) pairs per lane known at compile time and U = 4 row
// groups per warp step: all 2·M·U block loads of a step are issued before the first FMA (memory-
// level parallelism; the generic kernel above waits on each load).
template <int M>
__global__ void __launch_bounds__(256) k_ca_update_m(int64_t n, int t, int s, CaPtrs P, const double* __restrict__ alpha,
                                                     double* __restrict__ x, const double* __restrict__ r,
                                                     double* __restrict__ rnew, double* __restrict__ part) {
  pdl_enter();
  constexpr int U = 4;
  __shared__ double sa[kCaMax];
  __shared__ double sred[32];
  const int m = s * t;
  const bool skip = *reinterpret_cast<const volatile int*>(P.flag) != INT_MAX;
  for (int e = threadIdx.x; e < m; e += blockDim.x) sa[e] = alpha[e];
  __syncthreads();
  int L = 1;
  while (2 * L <= t && 2 * L <= 32) L *= 2;
  const int RPW = 32 / L, CPL = (t + L - 1) / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int sub = lane / L, lc = lane % L;
  const int64_t lo = (int64_t)blockIdx.x * n / gridDim.x, hi = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
  // this lane's (block j, column c) pairs and their α
  int jj[M], cc[M];
  double al[M];
#pragma unroll
  for (int q = 0; q < M; ++q) {
    jj[q] = q / CPL;
    cc[q] = lc + (q % CPL) * L;
    al[q] = (cc[q] < t) ? sa[jj[q] * t + cc[q]] : 0.0;
  }
  double acc = 0.0;
  for (int64_t r0 = lo + (int64_t)warp * RPW * U; r0 < hi; r0 += (int64_t)nw * RPW * U) {
    double wv[U][M], av[U][M];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = r0 + u * RPW + sub;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        const bool ok = i < hi && cc[q] < t;
        wv[u][q] = ok ? P.in[jj[q]][i * t + cc[q]] : 0.0;
        av[u][q] = ok ? P.out[jj[q]][i * t + cc[q]] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double dx = 0.0, dr = 0.0;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        dx = __fma_rn(wv[u][q], al[q], dx);
        dr = __fma_rn(av[u][q], al[q], dr);
      }
      for (int o = L >> 1; o > 0; o >>= 1) {
        dx += __shfl_xor_sync(0xffffffffu, dx, o);
        dr += __shfl_xor_sync(0xffffffffu, dr, o);
      }
      const int64_t i = r0 + u * RPW + sub;
      if (i < hi && lc == 0) {
        double ri = r[i];
        if (!skip) {
          x[i] += dx;
          ri -= dr;
        }
        rnew[i] = ri;
        acc = __fma_rn(ri, ri, acc);
      }
    }
  }
  const double tot = block_sum(acc, sred);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

cudaError_t launch_ca_update(cudaStream_t st, int64_t n, int t, int s, const CaPtrs& P, const double* alpha,
                             double* x, const double* r, double* rnew, double* part, int nblk) {
  if (s * t > kCaMax || s > kCaMaxBlocks) return cudaErrorInvalidValue;
  int L = 1;
  while (2 * L <= t && 2 * L <= 32) L *= 2;
  const int M = s * ((t + L - 1) / L);
  switch (M) {
    case 1: return launch_k(k_ca_update_m<1>, nblk, 256, 0, st, n, t, s, P, alpha, x, r, rnew, part);
    case 2: return launch_k(k_ca_update_m<2>, nblk, 256, 0, st, n, t, s, P, alpha, x, r, rnew, part);
    case 3: return launch_k(k_ca_update_m<3>, nblk, 256, 0, st, n, t, s, P, alpha, x, r, rnew, part);
    case 4: return launch_k(k_ca_update_m<4>, nblk, 256, 0, st, n, t, s, P, alpha, x, r, rnew, part);
    default: return launch_k(k_ca_update, nblk, 256, 0, st, n, t, s, P, alpha, x, r, rnew, part);
  }
}

// ============================================================================
// Vector kernels
// ============================================================================
__global__ void k_residual(int64_t n, const double* __restrict__ b, const double* __restrict__ y,
                           double* __restrict__ r, double* __restrict__ part) {
  __shared__ double sred[32];
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = b[i] - y[i];
    if (r) r[i] = v;
    acc = __fma_rn(v, v, acc);
  }
  const double s = block_sum(acc, sred);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

cudaError_t launch_residual(cudaStream_t st, int64_t n, const double* b, const double* y, double* r,
                            double* part, int nblk) {
  k_residual<<<nblk, kThreads, 0, st>>>(n, b, y, r, part);
  return cudaGetLastError();
}

__global__ void k_sumsq(int64_t n, const double* __restrict__ v, double* __restrict__ part) {
  __shared__ double sred[32];
  const int64_t lo = chunk_lo(n, blockIdx.x, gridDim.x), hi = chunk_lo(n, blockIdx.x + 1, gridDim.x);
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc = __fma_rn(v[i], v[i], acc);
  const double s = block_sum(acc, sred);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

cudaError_t launch_sumsq(cudaStream_t st, int64_t n, const double* v, double* part, int nblk) {
  k_sumsq<<<nblk, kThreads, 0, st>>>(n, v, part);
  return cudaGetLastError();
}

// (a6) one thread: the loop test of Alg 3/4/6 on the device, in the host
// loop's order — breakdown flag first (x stays the last completed iterate), then ρ = √(ρ²)
// (IEEE-rounded, the host's std::sqrt), hist[k] = ρ, k += 1, non-finite ρ stops (EKS_ERR_NONFINITE).
__global__ void k_loop_check(cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs, LoopState* st,
                             const double* __restrict__ scal, const int* __restrict__ flag, double* hist) {
  LoopState s = *st;
  s.iters += 1;
  const int fl = flag[0];
  unsigned int cont = 0;
  if (fl != 0x7fffffff) {
    s.stop = 2;
    s.fl = fl;
  } else {
    const double rho = sqrt(scal[1]);
    hist[s.k] = rho;
    s.k += 1;
    if (!isfinite(rho)) s.stop = 3;
    else if (rho > s.thr && s.k < s.kmax) cont = 1;
    else s.stop = 1;
  }
  s.phase = (s.phase + 1) % s.nphase;
  *st = s;
  cudaGraphSetConditional(hs, (unsigned int)s.phase);
  cudaGraphSetConditional(hw, cont);
}

cudaError_t launch_loop_check(cudaStream_t st, unsigned long long hwhile, unsigned long long hswitch,
                              LoopState* state, const double* scal, const int* flag, double* hist) {
  k_loop_check<<<1, 1, 0, st>>>((cudaGraphConditionalHandle)hwhile, (cudaGraphConditionalHandle)hswitch, state,
                                scal, flag, hist);
  return cudaGetLastError();
}

}  // namespace eks
