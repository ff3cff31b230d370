// eks_device.cuh — device helpers shared by the sweep kernels:
//   * tail_reduce: the fixed-order reduction of per-CTA partial sums done by the
//     last CTAs of the producing grid (no separate reduction launch);
//   * chol_warp<T>: the A-CholQR Cholesky B = RᵀR, R⁻¹ and α̃_b = R⁻ᵀ g in one warp,
//     every column of the factor held in the registers of one lane (T ≤ 32).
// Both reproduce, operation for operation, the separate kernels they replace
// (k_reduce32 and k_chol in eks_kernels.cu), so results are bitwise unchanged.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace eks {

// ---- Programmatic dependent launch (PDL): every hot kernel is launched with programmatic
// stream serialization; at its top it waits for the previous kernel's completion and memory
// (griddepcontrol.wait) and immediately allows the next kernel to be launched, so launch
// processing and CTA rasterisation overlap the tail of the running kernel.  Without the
// launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();  // EKS_PDL=0 disables (A/B measurements)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Where a producer kernel's per-CTA partials go when it reduces them itself.
// cnt == nullptr: no tail reduction (the host launches launch_reduce instead).
// Entries e < split land in out[e], entries e >= split in out2[e - split].
struct Tail {
  unsigned* cnt = nullptr;  // zero-initialised arrival counter, reset to 0 by the kernel
  double* out = nullptr;
  double* out2 = nullptr;
  int count = 0;            // reduced entries per partial
  int split = INT_MAX;
};

// Arguments of the Cholesky fused into the last CTA of the SpMM+Gram kernel (T ≤ 32, one rank).
struct CholArgs {
  int on = 0;                  // 1: run chol_warp on out = [B | g] after the reduction
  double* R = nullptr;         // R (t×t, may be null)
  double* Rinv = nullptr;      // R⁻¹ (t×t)
  double* alpha = nullptr;     // α̃_b = R⁻ᵀ g (null: no projection)
  int* flag = nullptr;         // breakdown: atomicMin(flag, gblock)
  int gblock = 0;
};

// ---- shared-memory addressing, fp64 DMMA, mbarriers and bulk (TMA) copies
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// D(8×8) += A(8×4, row) · B(4×8, col): lane (g = lane>>2, q = lane&3) holds
// a = A[g][q], b = B[q][g], d = {D[g][2q], D[g][2q+1]}.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(b))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}


__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Called by every thread of every CTA (≥ 256 threads) after the CTA has written its
// partial part[blockIdx.x * stride + e], e < tl.count.  The last NT = min(P, ⌈count/32⌉)
// CTAs to arrive wait until all P partials exist (the grid is a single wave, so every
// CTA is resident or has exited — no deadlock) and each reduces 32-entry slices in the
// order of k_reduce32: warp w sums b ≡ w (mod 8) ascending in batches of 8, then the
// 8 warps in order.  Returns true in exactly one CTA, the last one to finish: there
// all of out/out2 is written and visible.
__device__ __forceinline__ bool tail_reduce(const double* part, size_t stride, const Tail& tl) {
  __shared__ unsigned s_tk;
  __shared__ double s_red[8][33];
  const unsigned P = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_tk = atomicAdd(tl.cnt, 1u);
  __syncthreads();
  const unsigned tk = s_tk;
  const unsigned nsl = (unsigned)(tl.count + 31) / 32u;
  const unsigned NT = nsl < P ? nsl : P;
  if (tk < P - NT) return false;
  if (tid == 0)
    while (ld_acquire_u32(tl.cnt) < P) __nanosleep(32);
  __syncthreads();
  __threadfence();
  for (unsigned sl = tk - (P - NT); sl < nsl; sl += NT) {
    const size_t e = (size_t)sl * 32 + lane;
    double acc = 0.0;
    if (w < 8 && e < (size_t)tl.count) {  // warps 0..7 reduce (larger CTAs: the rest only synchronise)
      for (unsigned b0 = w; b0 < P; b0 += 64) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const unsigned b = b0 + 8 * k;
          v[k] = b < P ? __ldcg(part + (size_t)b * stride + e) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
      }
    }
    if (w < 8) s_red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && e < (size_t)tl.count) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += s_red[k][lane];
      if ((int)e < tl.split) tl.out[e] = t;
      else tl.out2[e - tl.split] = t;
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_tk = atomicAdd(tl.cnt, 1u);
  __syncthreads();
  const bool last = s_tk == P + NT - 1;
  if (last) {
    if (tid == 0) atomicExch(tl.cnt, 0u);  // ready for the next launch on the stream
    __threadfence();
  }
  return last;
}

// Cholesky of the t×t Gram B (upper triangle read), R⁻¹ and α̃ = R⁻ᵀ g, by one warp:
// lane j holds column j of the trailing matrix / of R (a[]) and of R⁻¹ (y[]).
// Right-looking elimination: at step k every trailing entry B_ij (k < i ≤ j) gets
// B_ij − R_ki·R_kj (product rounded, then subtracted, no fma) — exactly the
// subtractions of the oracle's left-looking loop in the same order, so R is bitwise
// equal to or_chol for equal B (reading R20).  Breakdown: pivot ≤ t·2⁻⁵²·max|B| (R6).
// R⁻¹ by the backward substitution of k_chol (same operations, same order).
// Core of chol_warp: leaves column j (= lane) of R in a[] and of R⁻¹ in y[]; returns the
// breakdown verdict (uniform over the warp).
template <int T>
__device__ __forceinline__ bool chol_warp_core(const double* B, double (&a)[T], double (&y)[T]) {
  static_assert(T <= 32, "one column per lane");
  const unsigned FULL = 0xffffffffu;
  const int j = threadIdx.x & 31;
  const bool act = j < T;
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    a[i] = act ? __ldcg(B + i * T + j) : 0.0;
    if (act && i <= j) m = fmax(m, fabs(a[i]));
    y[i] = (i == j) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  const double thr = __dmul_rn((double)T * 0x1p-52, m);
  bool fail = false;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const double d = __shfl_sync(FULL, a[k], k);
    if (!(d > thr)) fail = true;
    const double rkk = __dsqrt_rn(d);
    if (j > k) a[k] = __ddiv_rn(a[k], rkk);
    else if (j == k) a[k] = rkk;
#pragma unroll
    for (int i = k + 1; i < T; ++i) {
      const double rki = __shfl_sync(FULL, a[k], i);
      if (i <= j) a[i] = __dsub_rn(a[i], __dmul_rn(rki, a[k]));
    }
  }
  // R Y = I, Y upper triangular, k descending: Y_kj /= R_kk; Y_ij −= R_ik·Y_kj (i < k)
#pragma unroll
  for (int k = T - 1; k >= 0; --k) {
    const double rkk = __shfl_sync(FULL, a[k], k);
    if (j >= k) y[k] = __ddiv_rn(y[k], rkk);
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const double rik = __shfl_sync(FULL, a[i], k);
      if (j >= k) y[i] = __fma_rn(-rik, y[k], y[i]);
    }
  }
  return __any_sync(FULL, fail);
}

// Latency-lean variant for the solve path (the R⁻¹ kernel's prologue): the pivot's reciprocal
// square root (MUFU seed + two Newton steps + one correction, ≈ correctly rounded) replaces
// the sqrt and the T divisions of each step, and R⁻¹ multiplies by it too.  R agrees with
// chol_warp_core to a few ulps (not bitwise); the breakdown rule is the same (R6).
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y = rsqrt(d);                        // ~full precision already (CUDA's rsqrt)
  const double h = __dmul_rn(0.5, d);
  y = __fma_rn(y, __fma_rn(-h * y, y, 0.5), y);  // one Newton step: y(1.5 − ½ d y²)
  return y;
}
template <int T>
__device__ __forceinline__ bool chol_warp_fast(const double* B, double (&a)[T], double (&y)[T]) {
  static_assert(T <= 32, "one column per lane");
  const unsigned FULL = 0xffffffffu;
  const int j = threadIdx.x & 31;
  const bool act = j < T;
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    a[i] = act ? __ldcg(B + i * T + j) : 0.0;
    if (act && i <= j) m = fmax(m, fabs(a[i]));
    y[i] = (i == j) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  const double thr = __dmul_rn((double)T * 0x1p-52, m);
  bool fail = false;
  double rinv[T];  // 1/R_kk
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const double d = __shfl_sync(FULL, a[k], k);
    if (!(d > thr)) fail = true;
    const double ri = rsqrt_nr(d);
    rinv[k] = ri;
    if (j > k) a[k] = a[k] * ri;
    else if (j == k) a[k] = d * ri;
#pragma unroll
    for (int i = k + 1; i < T; ++i) {
      const double rki = __shfl_sync(FULL, a[k], i);
      if (i <= j) a[i] = __fma_rn(-rki, a[k], a[i]);
    }
  }
#pragma unroll
  for (int k = T - 1; k >= 0; --k) {
    if (j >= k) y[k] = y[k] * rinv[k];
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const double rik = __shfl_sync(FULL, a[i], k);
      if (j >= k) y[i] = __fma_rn(-rik, y[k], y[i]);
    }
  }
  return fail;
}

// chol_warp_fast with the outputs of launch_chol_fast (R, R⁻¹, α̃ = R⁻ᵀg, breakdown flag).
template <int T>
__device__ __forceinline__ void chol_warp_fast_out(const double* B, const double* g, double* Rout, double* Rinv,
                                                   double* alpha, int* flag, int gblock) {
  const int j = threadIdx.x & 31;
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

template <int T>
__device__ __forceinline__ void chol_warp(const double* B, const double* g, double* Rout, double* Rinv,
                                          double* alpha, int* flag, int gblock) {
  const int j = threadIdx.x & 31;
  const bool act = j < T;
  double a[T], y[T];
  const bool fail = chol_warp_core<T>(B, a, y);
  if (act) {
#pragma unroll
    for (int i = 0; i < T; ++i) {
      if (Rout) Rout[i * T + j] = (i <= j) ? a[i] : 0.0;
      Rinv[i * T + j] = y[i];
    }
    if (g != nullptr && alpha != nullptr) {
      double s = 0.0;  // α̃_j = Σ_{i ≤ j} (R⁻¹)_ij g_i, ascending i
#pragma unroll
      for (int i = 0; i < T; ++i)
        if (i <= j) s = __fma_rn(y[i], __ldcg(g + i), s);
      alpha[j] = s;
    }
  }
  if (fail && j == 0 && flag) atomicMin(flag, gblock);
}

// The same factorization for any T ≤ 64 with the columns in shared memory (sm: 2·T·(T+1)
// doubles) instead of registers — used inside kernels whose register budget is already
// spent (the last CTA of the fused SpMM+Gram).  Lane j owns columns j and j+32; the
// entries of row k of R travel by shuffle.  Same operations in the same order as
// chol_warp / k_chol.
template <int T>
__device__ __forceinline__ void chol_warp_smem(const double* B, const double* g, double* Rout, double* Rinv,
                                               double* alpha, int* flag, int gblock, double* sm) {
  static_assert(T <= 64, "two columns per lane at most");
  constexpr int CPL = (T + 31) / 32, SA = T + 1;
  const unsigned FULL = 0xffffffffu;
  double* sA = sm;
  double* sY = sm + T * SA;
  const int lane = threadIdx.x & 31;
  double m = 0.0;
  for (int e = lane; e < T * T; e += 32) {
    const int i = e / T, j = e % T;
    const double b = __ldcg(B + e);
    sA[i * SA + j] = b;
    sY[i * SA + j] = (i == j) ? 1.0 : 0.0;
    if (j >= i) m = fmax(m, fabs(b));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  const double thr = __dmul_rn((double)T * 0x1p-52, m);
  __syncwarp();
  bool fail = false;
  for (int k = 0; k < T; ++k) {
    const double d = sA[k * SA + k];
    if (!(d > thr)) fail = true;
    const double rkk = __dsqrt_rn(d);
    double rk[CPL];  // R_kj of the lane's columns (0 for j < k)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = lane + 32 * c;
      rk[c] = 0.0;
      if (j < T && j > k) rk[c] = __ddiv_rn(sA[k * SA + j], rkk);
      else if (j == k) rk[c] = rkk;
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = lane + 32 * c;
      if (j < T && j >= k) sA[k * SA + j] = rk[c];
    }
#pragma unroll 4
    for (int i = k + 1; i < T; ++i) {
      const double rki = __shfl_sync(FULL, (CPL == 1 || i < 32) ? rk[0] : rk[CPL - 1], i & 31);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int j = lane + 32 * c;
        if (j < T && i <= j) sA[i * SA + j] = __dsub_rn(sA[i * SA + j], __dmul_rn(rki, rk[c]));
      }
    }
    __syncwarp();
  }
  // R Y = I (each lane its own columns of Y; R is final)
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = lane + 32 * c;
    if (j < T)
      for (int k = j; k >= 0; --k) {
        const double ykj = __ddiv_rn(sY[k * SA + j], sA[k * SA + k]);
        sY[k * SA + j] = ykj;
#pragma unroll 4
        for (int i = 0; i < k; ++i) sY[i * SA + j] = __fma_rn(-sA[i * SA + k], ykj, sY[i * SA + j]);
      }
  }
  __syncwarp();
  for (int e = lane; e < T * T; e += 32) {
    const int i = e / T, j = e % T;
    if (Rout) Rout[e] = (i <= j) ? sA[i * SA + j] : 0.0;
    Rinv[e] = sY[i * SA + j];
  }
  if (g != nullptr && alpha != nullptr) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = lane + 32 * c;
      if (j < T) {
        double s = 0.0;
        for (int i = 0; i <= j; ++i) s = __fma_rn(sY[i * SA + j], __ldcg(g + i), s);
        alpha[j] = s;
      }
    }
  }
  if (__any_sync(FULL, fail) && lane == 0 && flag) atomicMin(flag, gblock);
}

}  // namespace eks
