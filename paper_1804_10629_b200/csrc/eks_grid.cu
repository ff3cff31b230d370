// eks_grid.cu — plane-marching fused SpMM + Gram for stencil-structured matrices.
//
// When eks_setup_csr finds that A is a 5-point (2D) or 7-point (3D) stencil on an
// nx × ny × nz lexicographic grid (every entry at an offset 0, ±1, ±nx, ±nx·ny that
// stays inside the grid), A·X is computed by 2.5D blocking: a CTA owns an (x, y)
// block of bx × by grid points and marches along z.  For every plane the producer
// warp streams the block's X rows with a one-point halo (by+2 contiguous runs) and
// the rows' 7 (5) stencil values into a stage of a shared-memory ring with
// cp.async.bulk (TMA) on full/empty mbarriers; the 8 consumer warps form each Y row
// from the three resident planes z−1, z, z+1 at fixed shared-memory offsets.  Every
// X row therefore crosses L2 → SM about (1 + 2/by + 2/bx)(1 + 2/zc) times instead of
// once per stencil entry, and the ±N² plane reuse never depends on L2 retention —
// the limit of the gather kernels.
//
// Accumulation order per Y entry: the stencil slots in ascending column order with
// value 0 in absent (boundary) slots — fma(0, x, y) = y exactly for finite x — i.e.
// the oracle's p-ascending CSR order (reading R20): Y is bitwise equal to k_spmm.
// The Gram / α̃ epilogue is the one of k_spmm_seg (per-warp DMMA over the warp's own
// rows, fixed warp order, tail reduction, optional Cholesky).
#include "eks_device.cuh"
#include "eks_sweep.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace eks {

namespace {

template <int T>
struct GrCfg {
  static constexpr int NWC = 8, NTH = 32 * (NWC + 1);  // 8 consumer warps + 1 producer warp
  static constexpr int R = 2048 / T;                   // output rows per plane-block (bx·by)
  static constexpr int RW = T == 8 ? 8 : 4;            // rows per warp unit (DMMA k = 4 rows)
  static constexpr int G = 32 / RW;                    // threads per row
  static constexpr int C = T / G;                      // columns per thread: pairs 2(gl + G·c2), c2 < C/2
                                                       // (the G lanes of a row read 16·G contiguous bytes
                                                       // per instruction: conflict-free shared loads)
  static constexpr int U = R / RW;                     // units per plane-block
  static constexpr int UPW = U / NWC;                  // units per consumer warp per plane
  static constexpr int S = T + 4;                      // Y scratch row stride
  static constexpr int MT = T / 8;
  static constexpr int NUT = MT * (MT + 1) / 2;        // upper 8×8 output tiles
  // t = 64: the 36 upper tiles (+ 8 Xᵀr tiles) are dealt to the warps and accumulated over the
  // whole plane-block from a CTA-level Y tile (double-buffered, one consumer barrier per plane)
  static constexpr bool CG = T >= 64;
  static constexpr int JOBS = NUT + MT;                // Gram tiles + r tiles
  static constexpr int JPW = CG ? (JOBS + NWC - 1) / NWC : 1;
  static_assert(U % NWC == 0, "units");
  static_assert(!CG || UPW == 1, "CTA-level Gram: one unit per warp, the warps' scratches form the Y tile");
  // PATCH mode (T = 16, 32): GP lanes per row, NG lane groups per warp, patches of up to 2 × 2 rows
  static constexpr int GP = T / 2, NG = 32 / GP;
  // rows of a warp's Y scratch: the patch consumer's NG·4 rows, else the unit's RW rows (a larger
  // scratch costs the t = 8 ring its fifth stage: 0.63 vs 0.74 of HBM at 384³)
  __host__ __device__ static constexpr int yr(bool patch) { return (patch && NG * 4 > RW) ? NG * 4 : RW; }
};

}  // namespace

// Stage bytes: X plane-block (bx+2)·(by+2·hy) rows, then R rows of VS stencil values, then R
// entries of r.
// SWZ (the t = 16 patch kernel): the X plane-block arrives by 2D tensor-map TMA with the 128-byte
// swizzle — every X row is one 128-byte line whose 16-byte chunks are permuted by (point & 7) —
// each y-line padded to a multiple of 8 points (PWP) so that every line starts on a 1024-byte
// swizzle atom; stages are 1024-byte aligned.
__host__ __device__ inline int grid_pwp(int bx, bool swz) { return swz ? ((bx + 2 + 7) & ~7) : bx + 2; }
template <int T>
__host__ __device__ inline size_t grid_xbytes(int bx, int by, int hy, bool swz) {
  return (size_t)grid_pwp(bx, swz) * (by + 2 * hy) * T * 8;
}
template <int T>
__host__ __device__ inline size_t grid_stage_bytes(int bx, int by, int hy, int vs, bool swz = false) {
  using K = GrCfg<T>;
  const size_t a = swz ? 1023 : 127;
  return ((grid_xbytes<T>(bx, by, hy, swz) + (size_t)K::R * vs * 8 + (size_t)K::R * 8) + a) & ~a;
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          saddr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(saddr(bar))
      : "memory");
}

// PATCH (3D, t = 16, 32): every group of T/2 lanes (one double2 column pair per lane) forms a 1 × 4
// patch of output rows (4 consecutive y-lines at one x) from one set of loads: the centre-plane
// rows with their ±1 x-neighbours, the ±y lines outside the patch and the ±z planes are each read
// once — 5.5 shared-memory row loads per output row instead of 7.
// PV (t = 16 patch variants, EKS_GRID_PV): 0 = Gram fragments from a per-warp Y scratch (default,
// measured best), 1 = X by swizzled tensor-map TMA, 2 = Gram fragments gathered by shuffles
template <int T, int W, bool PATCH = false, int PV = 0>
__global__ void __launch_bounds__(GrCfg<T>::NTH, 1)
    k_spmm_grid(const GridPlan gp, int bx, int by, int zc, const double* __restrict__ X, double* __restrict__ Y,
                const double* __restrict__ r, double* __restrict__ part, const Tail tl, const CholArgs ch, int NS,
                const bool gram, const __grid_constant__ CUtensorMap tmX) {
  using K = GrCfg<T>;
  pdl_enter();
  constexpr int S = K::S, G = K::G, C = K::C, RW = K::RW, NWC = K::NWC, MT = K::MT, H = T / 2;
  constexpr int VS = (W + 1) & ~1;
  static_assert(W == 5 || W == 7, "2D 5-point or 3D 7-point stencil");
  extern __shared__ __align__(128) unsigned char smraw_[];
  // SWZ (EKS_GRID_PV=1): the t = 16 patch kernel streams X by swizzled tensor-map TMA.  Measured slower
  // than the linear 1D bulk copies (0.57 vs 0.67 of HBM at 384³, profiles/spmm_micro_r02.txt): off by default
  constexpr bool SWZ = PATCH && T == 16 && PV == 1;
  unsigned char* smraw =
      SWZ ? reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw_) + 1023) & ~(uintptr_t)1023) : smraw_;
  const int nx = gp.nx, ny = gp.ny, nz = gp.nz;
  const int hy = ny > 1 ? 1 : 0;               // y halo (3D only)
  const int PW = bx + 2, PH = by + 2 * hy;     // plane-block extent
  const int PWP = grid_pwp(bx, SWZ);           // points per y-line in shared memory
  const int64_t plane = (int64_t)nx * ny;
  const size_t SB = grid_stage_bytes<T>(bx, by, hy, VS, SWZ);
  const size_t XB = grid_xbytes<T>(bx, by, hy, SWZ);  // X plane-block bytes of a stage
  double* sYw = reinterpret_cast<double*>(smraw + (size_t)NS * SB);  // [2 (CG)][NWC][YR][S]
  constexpr int YR = K::yr(PATCH);
  // XSCR (t = 16 patch consumer): the Gram's X fragments from a padded per-warp copy of the centre rows
  // (written with the Y rows) instead of the plane-block, whose 4 rows of a k-step are whole 128-byte
  // lines apart — the same banks: ncu showed 8 wavefronts per fragment load instead of 2
  // (t = 8: rows 64 B apart, 2-way only, and the scratch would cost the ring its fifth stage)
  constexpr bool XSCR = !K::CG && T >= 16 && (PATCH ? (T == 16 && PV == 0) : true);
  uint64_t* full = reinterpret_cast<uint64_t*>(sYw + ((K::CG ? 2 : 1) + (XSCR ? 1 : 0)) * NWC * YR * S);
  uint64_t* empty = full + 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q4 = lane & 3;
  const int nbx = (nx + bx - 1) / bx, nby = (ny + by - 1) / by, nzc = (nz + zc - 1) / zc;
  const bool rbulk = (nx % 2) == 0;  // r lines start 16-byte aligned (x0, bx even)
  const int64_t nunits = (int64_t)nbx * nby * nzc;
  // unit → block origin and z range
  auto unit_geom = [&](int64_t u, int& x0, int& y0, int& z0, int& z1) {
    const int zi = (int)(u % nzc);
    const int64_t b = u / nzc;
    x0 = (int)(b % nbx) * bx;
    y0 = (int)(b / nbx) * by;
    z0 = zi * zc;
    z1 = z0 + zc < nz ? z0 + zc : nz;
  };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // zero the X ring once: halo cells outside the grid are never written and must be finite
  for (size_t e = tid; e < (size_t)NS * SB / 16; e += K::NTH) reinterpret_cast<double2*>(smraw)[e] = make_double2(0, 0);
  __syncthreads();

  if (warp == NWC) {
    // ================= producer: one load step = one X plane-block (+ the values of the plane below it)
    int cur = 0;             // ring stage of this load step
    uint32_t eph = 0;        // empty-barrier phase parity of the stage's previous use
    int64_t gstep = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      int x0, y0, z0, z1;
      unit_geom(u, x0, y0, z0, z1);
      const int xa = x0 - 1 > 0 ? x0 - 1 : 0, xb = x0 + bx + 1 < nx ? x0 + bx + 1 : nx;  // X run [xa, xb)
      const int ob = x0 + bx < nx ? x0 + bx : nx;                                        // output x range [x0, ob)
      for (int p = z0 - 1; p <= z1; ++p, ++gstep) {
        const int s = cur;
        if (gstep >= NS) mbar_wait(empty + s, eph);
        if (++cur == NS) {
          cur = 0;
          if (gstep >= NS) eph ^= 1u;  // lap L ≥ 1 waits for release phase (L − 1) & 1
        }
        unsigned char* st = smraw + (size_t)s * SB;
        // lane l < PH: X line y0 − hy + l of plane p;  lane PH + l < PH + by: values of output line y0 + l, plane p − 1
        uint32_t bytes = 0;
        const int yy = y0 - hy + lane;
        const bool xline = lane < PH && p >= -gp.gb && p < nz + gp.ga && yy >= 0 && yy < ny;
        const int vl = lane - PH, vy = y0 + vl;
        const bool vline = vl >= 0 && vl < by && p - 1 >= z0 && p - 1 < z1 && vy < ny;
        const int rl = lane - PH - by, ry = y0 + rl;  // lanes for the lines of r (16-byte rows: nx even)
        const bool rline = gram && r != nullptr && rbulk && rl >= 0 && rl < by && p - 1 >= z0 && p - 1 < z1 && ry < ny;
        // SWZ: every line of a plane in [−gb, nz + ga) as a full (bx+2)-point box; rows outside the
        // tensor are zero-filled, rows of a neighbouring line / plane are finite and meet stencil
        // slots of value 0 (fma(0, x, y) = y)
        const bool pin = p >= -gp.gb && p < nz + gp.ga;
        if (SWZ ? (lane < PH && pin) : xline) bytes += SWZ ? (uint32_t)PW * T * 8 : (uint32_t)(xb - xa) * T * 8;
        if (vline) bytes += (uint32_t)(ob - x0) * VS * 8;
        if (rline) bytes += (uint32_t)(ob - x0) * 8;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(full + s, bytes);  // 0 bytes (plane outside the grid): the phase completes at once
        }
        __syncwarp();
        if constexpr (SWZ) {
          if (lane < PH && pin) {  // tensor rows from the first ghost plane: (p + gb)·plane + yy·nx + x0 − 1
            const int row = (int)((int64_t)(p + gp.gb) * plane + (int64_t)yy * nx + x0 - 1);
            tma_2d(st + (size_t)lane * PWP * T * 8, &tmX, 0, row, full + s);
          }
        } else if (xline) {
          const int64_t row = (int64_t)p * plane + (int64_t)yy * nx + xa;
          double* dst = reinterpret_cast<double*>(st) + ((size_t)lane * PW + (xa - x0 + 1)) * T;
          bulk_g2s(dst, X + row * T, (uint32_t)(xb - xa) * T * 8, full + s);
        }
        if (vline) {
          const int64_t row = (int64_t)(p - 1) * plane + (int64_t)vy * nx + x0;
          double* dst = reinterpret_cast<double*>(st + XB) + (size_t)vl * bx * VS;
          bulk_g2s(dst, gp.sv + row * VS, (uint32_t)(ob - x0) * VS * 8, full + s);
        }
        if (rline) {
          const int64_t row = (int64_t)(p - 1) * plane + (int64_t)ry * nx + x0;
          double* dst = reinterpret_cast<double*>(st + XB + (size_t)K::R * VS * 8) + (size_t)rl * bx;
          bulk_g2s(dst, r + row, (uint32_t)(ob - x0) * 8, full + s);
        }
      }
    }
  }

  constexpr int NACC = K::CG ? 1 : K::NUT, NACR = K::CG ? 1 : MT;
  double acc[NACC][2], accr[NACR][2];  // XᵀY (upper tiles) and Xᵀr (column 0 of an r-tile)
  double accj[K::JPW][2];               // CG: this warp's Gram / r tiles over the whole block
#pragma unroll
  for (int uu = 0; uu < NACC; ++uu) acc[uu][0] = acc[uu][1] = 0.0;
#pragma unroll
  for (int mi = 0; mi < NACR; ++mi) accr[mi][0] = accr[mi][1] = 0.0;
#pragma unroll
  for (int jj = 0; jj < K::JPW; ++jj) accj[jj][0] = accj[jj][1] = 0.0;
  int ybuf = 0;  // CG: Y tile buffer of this plane
  // CG: this warp's jobs, decoded once — job < NUT: upper tile (mi, ni); else the r tile of row block mi
  int jmi[K::JPW], jni[K::JPW];
#pragma unroll
  for (int jj = 0; jj < K::JPW; ++jj) {
    const int job = warp + jj * NWC;
    jmi[jj] = -1;
    jni[jj] = -1;
    if (job < K::NUT) {
      int mi = 0, rem = job;
      while (rem >= MT - mi) { rem -= MT - mi; ++mi; }
      jmi[jj] = mi;
      jni[jj] = mi + rem;
    } else if (job < K::JOBS) {
      jmi[jj] = job - K::NUT;
    }
  }
  if (warp < NWC) {
    // ================= consumers
    const int rw = lane / G, gl = lane % G;
    const int bxs = 31 - __clz(bx);  // bx is a power of two
    double* yw0 = sYw + (size_t)warp * YR * S;
    double* xw0 = sYw + (size_t)(NWC + warp) * YR * S;  // XSCR only
    int cur = 0;        // stage of the current load step
    uint32_t ph = 0;    // its full-barrier phase parity
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      int x0, y0, z0, z1;
      unit_geom(u, x0, y0, z0, z1);
      for (int p = z0 - 1; p <= z1; ++p) {
        mbar_wait(full + cur, ph);
        const int sm1 = cur == 0 ? NS - 1 : cur - 1, sm2 = sm1 == 0 ? NS - 1 : sm1 - 1;
        const int q = p - 1;  // output plane of this step
        if (q >= z0) {
          const double* Pm = reinterpret_cast<const double*>(smraw + (size_t)sm2 * SB);
          const double* P0 = reinterpret_cast<const double*>(smraw + (size_t)sm1 * SB);
          const double* Pp = reinterpret_cast<const double*>(smraw + (size_t)cur * SB);
          const double* Vs = reinterpret_cast<const double*>(smraw + (size_t)cur * SB + XB);
          const double* Rs = Vs + K::R * VS;
          const int64_t qrow = (int64_t)q * plane + (int64_t)y0 * nx + x0;  // global row of block point (0,0)
          double* yw = yw0 + (K::CG ? ybuf * NWC * YR * S : 0);
          if constexpr (PATCH) {
            constexpr int GP = K::GP, NG = K::NG;
            // 1 × 4 patches (a column of 4 y-lines): the 4 lane groups of a warp take x-adjacent
            // columns, so their rows' stencil values (64 B per row) fall in both bank halves
            // (2 × 2 patches put them 128 B apart: 4-way conflicts that cancelled the gain)
            constexpr int PX = 1, PY = 4, LPX = 0, PR = PX * PY, RPW = NG * PR;
            // the Gram from registers: t = 16 (4 lane groups = the 4 rows of a k-step), linear layout
            constexpr bool RGRAM = T == 16 && PV == 2;  // measured slower than the scratch (0.61 vs 0.67)
            const int gi = lane / GP, gl = lane % GP;
            const int ppx = bx / PX;                 // patches per block line (a power of 2)
            const int nsteps = K::R / (PR * NG * NWC);  // patch steps per warp and plane
            {
            for (int ps = 0; ps < nsteps; ++ps) {
              const int pp = (ps * NWC + warp) * NG + gi;  // patch of this lane group
              const int px0 = (pp & (ppx - 1)) * PX, py0 = (pp >> (bxs - LPX)) * PY;
              // ---- the patch's 4 rows, sliding up the y-lines: the centre of line dy+1 is loaded once
              // (as the +y neighbour of line dy and the centre of the next row); ±x and ±z per row.
              // Stencil slots in ascending column order (reading R20).
              // swizzled 128-byte X rows: column pair gl of point P sits at chunk gl ^ (P & 7)
              const int Pc = px0 + 1;  // the patch's point in its line
              const int sc = SWZ ? 2 * (gl ^ (Pc & 7)) : 2 * gl;
              const int sm_ = SWZ ? 2 * (gl ^ ((Pc - 1) & 7)) : 2 * gl, sp_ = SWZ ? 2 * (gl ^ ((Pc + 1) & 7)) : 2 * gl;
              const double* c0p = P0 + ((size_t)(py0 + hy) * PWP + Pc) * T;  // centre row, line 0 (unswizzled base)
              double2 cm = *reinterpret_cast<const double2*>(c0p - (size_t)PWP * T + sc);  // line −1 (−y of row 0)
              double2 c0 = *reinterpret_cast<const double2*>(c0p + sc);
#pragma unroll
              for (int dy = 0; dy < PY; ++dy) {
                const double* cp = c0p + (size_t)dy * PWP * T;
                const double2 cn = *reinterpret_cast<const double2*>(cp + (size_t)PWP * T + sc);  // +y (line dy+1)
                const double2 xm = *reinterpret_cast<const double2*>(cp - T + sm_);
                const double2 xp = *reinterpret_cast<const double2*>(cp + T + sp_);
                const size_t zo = (size_t)(cp - P0) + sc;
                const double2 zm = *reinterpret_cast<const double2*>(Pm + zo);
                const double2 zp = *reinterpret_cast<const double2*>(Pp + zo);
                const int ir = (py0 + dy) * bx + px0;
                const bool ok = x0 + px0 < nx && y0 + py0 + dy < ny;
                const int64_t grow = qrow + (int64_t)(py0 + dy) * nx + px0;
                const double2 nb[7] = {zm, cm, xm, c0, xp, cn, zp};
                double2 y = make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 0; k < VS; k += 2) {
                  const double2 av = ok ? *reinterpret_cast<const double2*>(Vs + ir * VS + k) : make_double2(0, 0);
                  y.x = __fma_rn(av.x, nb[k].x, y.x);
                  y.y = __fma_rn(av.x, nb[k].y, y.y);
                  if (k + 1 < 7) {
                    y.x = __fma_rn(av.y, nb[k + 1].x, y.x);
                    y.y = __fma_rn(av.y, nb[k + 1].y, y.y);
                  }
                }
                if (!ok) y = make_double2(0.0, 0.0);
                else reinterpret_cast<double2*>(Y)[grow * H + gl] = y;
                if constexpr (RGRAM) {
                  // Gram k-step over the 4 lane groups' rows of line dy (row q4 = group q4's row), its
                  // fragments gathered from the groups' registers by shuffles (no Y scratch round trip):
                  // lane (g, q4) takes column 8i + g of group q4's row from lane q4·GP + 4i + g/2
                  if (gram) {
                    const int ppq = (ps * NWC + warp) * NG + q4;
                    const int pxq = ppq & (ppx - 1), pyq = (ppq >> bxs) * PY + dy;
                    const bool okq = x0 + pxq < nx && y0 + pyq < ny;
                    double xa[MT], ybv[MT];
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                      const int src = q4 * GP + 4 * i + (g >> 1);
                      const double cx = __shfl_sync(0xffffffffu, c0.x, src), cy = __shfl_sync(0xffffffffu, c0.y, src);
                      const double yx = __shfl_sync(0xffffffffu, y.x, src), yy2 = __shfl_sync(0xffffffffu, y.y, src);
                      xa[i] = okq ? ((g & 1) ? cy : cx) : 0.0;
                      ybv[i] = (g & 1) ? yy2 : yx;
                    }
                    int ut = 0;
#pragma unroll
                    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
                      for (int ni = mi; ni < MT; ++ni, ++ut) dmma(acc[ut][0], acc[ut][1], xa[mi], ybv[ni]);
                    if (r != nullptr) {
                      const double br = okq ? (rbulk ? Rs[pyq * bx + pxq] : __ldg(r + qrow + (int64_t)pyq * nx + pxq))
                                            : 0.0;
#pragma unroll
                      for (int mi = 0; mi < MT; ++mi) accr[mi][0] = fma(xa[mi], br, accr[mi][0]);
                    }
                  }
                } else {
                  if (gram) {
                    *reinterpret_cast<double2*>(yw + (gi * PR + dy) * S + 2 * gl) = y;
                    if constexpr (XSCR)
                      *reinterpret_cast<double2*>(xw0 + (gi * PR + dy) * S + 2 * gl) = ok ? c0 : make_double2(0.0, 0.0);
                  }
                }
                cm = c0;
                c0 = cn;
              }
              if (!gram || RGRAM) continue;
              __syncwarp();
              // ---- Gram over the warp's RPW rows on DMMA (k-steps of 4 rows); t = 64 runs Gram-free only
              if constexpr (!K::CG) {
#pragma unroll
              for (int ks = 0; ks < RPW / 4; ++ks) {
                const int rq = ks * 4 + q4, gq = rq / PR, wq = rq % PR;
                const int ppq = (ps * NWC + warp) * NG + gq;
                const int pxq = (ppq & (ppx - 1)) * PX + wq % PX, pyq = (ppq >> (bxs - LPX)) * PY + wq / PX;
                const bool okq = x0 + pxq < nx && y0 + pyq < ny;
                const int Pq = pxq + 1;
                const double* xo = P0 + ((size_t)(pyq + hy) * PWP + Pq) * T;
                double xa[MT], ybv[MT];
#pragma unroll
                for (int i = 0; i < MT; ++i) {  // column 8i + g: chunk (4i + g/2) ^ (Pq & 7), half g & 1
                  xa[i] = XSCR ? xw0[rq * S + i * 8 + g]
                               : (okq ? xo[SWZ ? 2 * ((4 * i + (g >> 1)) ^ (Pq & 7)) + (g & 1) : i * 8 + g] : 0.0);
                  ybv[i] = yw[rq * S + i * 8 + g];
                }
                int ut = 0;
#pragma unroll
                for (int mi = 0; mi < MT; ++mi)
#pragma unroll
                  for (int ni = mi; ni < MT; ++ni, ++ut) dmma(acc[ut][0], acc[ut][1], xa[mi], ybv[ni]);
                if (r != nullptr) {
                  const int irq = pyq * bx + pxq;
                  // Xᵀr on the FMA pipe: the lane's X fragment (row q4 of the k-step, column 8·mi + g) times
                  // that row's r; the 4 lanes of a group are summed once at the end (a DMMA with r as
                  // column 0 of a tile costs the fp64 pipe ≈ 7 DFMA issue slots)
                  const double br = okq ? (rbulk ? Rs[irq] : __ldg(r + qrow + (int64_t)pyq * nx + pxq)) : 0.0;
#pragma unroll
                  for (int mi = 0; mi < MT; ++mi) accr[mi][0] = fma(xa[mi], br, accr[mi][0]);
                }
              }
              }  // !CG
              __syncwarp();
            }
            }
          } else {
#pragma unroll
          for (int uu = 0; uu < K::UPW; ++uu) {
            const int r0u = (warp + uu * NWC) * RW;  // first row of the unit in the plane-block
            const int ir = r0u + rw;
            const int ix = ir & (bx - 1), iy = ir >> bxs;
            const bool ok = x0 + ix < nx && y0 + iy < ny;
            const int64_t grow = qrow + (int64_t)iy * nx + ix;
            const int cen = (iy + hy) * PW + ix + 1;
            double vr = 0.0;
            if (gram && r != nullptr && ok) vr = rbulk ? Rs[ir] : __ldg(r + grow);
            double a[VS];
#pragma unroll
            for (int k = 0; k < VS; k += 2) {
              const double2 av = ok ? *reinterpret_cast<const double2*>(Vs + ir * VS + k) : make_double2(0, 0);
              a[k] = av.x;
              a[k + 1] = av.y;
            }
            // stencil slots in ascending column order
            const double* src[W];
            if constexpr (W == 7) {
              src[0] = Pm + cen * T;
              src[1] = P0 + (cen - PW) * T;
              src[2] = P0 + (cen - 1) * T;
              src[3] = P0 + cen * T;
              src[4] = P0 + (cen + 1) * T;
              src[5] = P0 + (cen + PW) * T;
              src[6] = Pp + cen * T;
            } else {
              src[0] = Pm + cen * T;
              src[1] = P0 + (cen - 1) * T;
              src[2] = P0 + cen * T;
              src[3] = P0 + (cen + 1) * T;
              src[4] = Pp + cen * T;
            }
#pragma unroll
            for (int c2 = 0; c2 < C / 2; ++c2) {
              double2 xv[W];
#pragma unroll
              for (int k = 0; k < W; ++k) xv[k] = *reinterpret_cast<const double2*>(src[k] + 2 * (gl + G * c2));
              double2 y = make_double2(0.0, 0.0);
#pragma unroll
              for (int k = 0; k < W; ++k) {
                y.x = __fma_rn(a[k], xv[k].x, y.x);
                y.y = __fma_rn(a[k], xv[k].y, y.y);
              }
              if (!ok) y = make_double2(0.0, 0.0);
              else reinterpret_cast<double2*>(Y)[grow * H + gl + G * c2] = y;
              if (gram) {
                *reinterpret_cast<double2*>(yw + rw * S + 2 * (gl + G * c2)) = y;
                if constexpr (XSCR)
                  *reinterpret_cast<double2*>(xw0 + rw * S + 2 * (gl + G * c2)) = ok ? xv[W / 2] : make_double2(0.0, 0.0);
              }
            }
            if (!gram) continue;
            __syncwarp();
            // ---- Gram over the unit's RW rows on DMMA: A = own X rows (plane q), B = [Y rows | r]
            // (t = 64: over the whole block below instead)
#pragma unroll
            for (int ks = 0; ks < (K::CG ? 0 : RW / 4); ++ks) {
              const int rq = ks * 4 + q4, irq = r0u + rq, ixq = irq & (bx - 1), iyq = irq >> bxs;
              const bool okq = x0 + ixq < nx && y0 + iyq < ny;
              const double* xo = P0 + ((iyq + hy) * PW + ixq + 1) * T;
              double xa[MT], yb[MT];
#pragma unroll
              for (int i = 0; i < MT; ++i) {
                xa[i] = XSCR ? xw0[rq * S + i * 8 + g] : (okq ? xo[i * 8 + g] : 0.0);
                yb[i] = yw[rq * S + i * 8 + g];
              }
              if constexpr (!K::CG) {
                int ut = 0;
#pragma unroll
                for (int mi = 0; mi < MT; ++mi)
#pragma unroll
                  for (int ni = mi; ni < MT; ++ni, ++ut) dmma(acc[ut][0], acc[ut][1], xa[mi], yb[ni]);
                if (r != nullptr) {
                  const double br = __shfl_sync(0xffffffffu, vr, rq * G);  // lane rq·G holds row rq's r
#pragma unroll
                  for (int mi = 0; mi < MT; ++mi) accr[mi][0] = fma(xa[mi], br, accr[mi][0]);  // FMA pipe (see above)
                }
              }
            }
            __syncwarp();
          }
          }  // PATCH / unit consumers
          if (K::CG && gram) {
            // ---- CTA-level Gram: all consumer warps' Y rows are in the Y tile; each warp
            // accumulates its tiles over the block's R rows (k-steps of 4 rows)
            asm volatile("bar.sync 1, %0;" ::"n"(32 * NWC) : "memory");
            const double* Yt = sYw + ybuf * NWC * YR * S;
#pragma unroll 2
            for (int kk = 0; kk < K::R; kk += 4) {  // the warp's jobs interleaved: independent DMMA chains
              const int irq = kk + q4, ixq = irq & (bx - 1), iyq = irq >> bxs;
              const bool okq = x0 + ixq < nx && y0 + iyq < ny;
              const double* xo = P0 + ((iyq + hy) * PW + ixq + 1) * T;
              const double rr = (g == 0 && okq && r != nullptr)
                                    ? (rbulk ? Rs[irq] : __ldg(r + qrow + (int64_t)iyq * nx + ixq)) : 0.0;
#pragma unroll
              for (int jj = 0; jj < K::JPW; ++jj)
                if (jmi[jj] >= 0) {
                  const double xa = okq ? xo[jmi[jj] * 8 + g] : 0.0;
                  const double bb = jni[jj] >= 0 ? Yt[irq * S + jni[jj] * 8 + g] : rr;
                  dmma(accj[jj][0], accj[jj][1], xa, bb);
                }
            }
            ybuf ^= 1;
          }
          if (lane == 0) mbar_arrive(empty + sm2);  // plane q−1 is no longer needed
        }
        if (p == z1 && lane == 0) {  // end of the unit: release the last two planes
          mbar_arrive(empty + sm1);
          mbar_arrive(empty + cur);
        }
        if (++cur == NS) {
          cur = 0;
          ph ^= 1u;
        }
      }
    }
  }
  // ================= epilogue (as k_spmm_seg): consumer warps' partials in warp order, lower half mirrored
  if (!gram) return;
  __syncthreads();
  double* red = reinterpret_cast<double*>(smraw);
  constexpr int PER = T * T + T;
  if constexpr (K::CG) {
    if (warp < NWC) {
#pragma unroll
      for (int jj = 0; jj < K::JPW; ++jj) {
        const int job = warp + jj * NWC;
        if (job < K::JOBS) {
          if (job < K::NUT) {
            int mi = 0, rem = job;
            while (rem >= MT - mi) { rem -= MT - mi; ++mi; }
            const int ni = mi + rem;
            double* d = red + (mi * 8 + g) * T + ni * 8 + 2 * q4;
            d[0] = accj[jj][0];
            d[1] = accj[jj][1];
          } else if (q4 == 0) {
            red[T * T + (job - K::NUT) * 8 + g] = accj[jj][0];
          }
        }
      }
    }
    __syncthreads();
  }
  if constexpr (!K::CG) {  // Xᵀr: rows q4 = 0..3 of every k-step sit in the 4 lanes of a group
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      accr[mi][0] += __shfl_xor_sync(0xffffffffu, accr[mi][0], 1);
      accr[mi][0] += __shfl_xor_sync(0xffffffffu, accr[mi][0], 2);
    }
  }
  for (int w = 0; w < (K::CG ? 0 : NWC); ++w) {
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
      if (q4 == 0)
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
          double* d = red + T * T + mi * 8 + g;
          *d = w == 0 ? accr[mi][0] : *d + accr[mi][0];
        }
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
    if constexpr (T <= 16) {  // the block's Cholesky by the last CTA (solve path: rsqrt pivots)
      if (last && ch.on && warp == 0)
        chol_warp_fast_out<T>(tl.out, r != nullptr ? tl.out + T * T : nullptr, ch.R, ch.Rinv, ch.alpha, ch.flag,
                              ch.gblock);
    }
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

template <int T>
static void grid_shape(const GridPlan& gp, int& bx, int& by, int& zc, int sms) {
  using K = GrCfg<T>;
  static const int by_env = [] {  // EKS_GRID_BY: plane-block height override for A/B measurements
    const char* e = getenv("EKS_GRID_BY");
    return e ? atoi(e) : 0;
  }();
  by = gp.ny > 1 ? (by_env > 0 ? by_env : 4) : 1;
  if (by > K::R / 4) by = K::R / 4;
  bx = K::R / by;
  const int64_t blocks = (int64_t)((gp.nx + bx - 1) / bx) * ((gp.ny + by - 1) / by);
  // z chunks so that every SM gets ≥ ~4 units (each chunk re-reads 2 halo planes)
  int64_t want = 4 * (int64_t)sms;
  int64_t nzc = (want + blocks - 1) / blocks;
  if (nzc < 1) nzc = 1;
  zc = (int)((gp.nz + nzc - 1) / nzc);
  if (zc < 8) zc = gp.nz < 8 ? gp.nz : 8;
  static const int zc_env = [] {  // EKS_GRID_ZC: z-chunk override for A/B measurements
    const char* e = getenv("EKS_GRID_ZC");
    return e ? atoi(e) : 0;
  }();
  if (zc_env > 0) zc = zc_env < gp.nz ? zc_env : gp.nz;
}

template <int T, int W>
static cudaError_t grid_t(cudaStream_t st, const GridPlan& gp, const double* X, double* Y, const double* r,
                          double* part, int nblk, const Tail& tl, const CholArgs& ch, bool gram) {
  using K = GrCfg<T>;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int bx, by, zc;
  grid_shape<T>(gp, bx, by, zc, sms);
  const int hy = gp.ny > 1 ? 1 : 0, vs = (W + 1) & ~1;
  static const bool patch_env = [] {  // EKS_GRID_PATCH=0: the per-row consumer (A/B measurements)
    const char* e = getenv("EKS_GRID_PATCH");
    return !(e && atoi(e) == 0);
  }();
  // t = 16 (swizzled TMA) and the Gram-free t = 64 launches; t = 32: measured slower (0.57 vs 0.63,
  // profiles/spmm_micro_r02.txt)
  constexpr bool PATCH_T = (T == 16 || T == 64) && W == 7;
  CUtensorMap tm;
  memset(&tm, 0, sizeof tm);
  static const int pv_env = [] {
    const char* e = getenv("EKS_GRID_PV");
    return e ? atoi(e) : 0;
  }();
  const bool swz_env = pv_env == 1;
  bool patch = PATCH_T && patch_env && by % 4 == 0 && bx + 2 <= 256 && (T == 16 || !gram);
  if (patch && T == 16 && swz_env) {  // the X tensor from the first ghost plane: T columns × (gb + nz + ga)·plane rows, 128B swizzle
    const PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    const int64_t plane = (int64_t)gp.nx * gp.ny, rows = (int64_t)(gp.gb + gp.nz + gp.ga) * plane;
    const cuuint64_t gdim[2] = {(cuuint64_t)T, (cuuint64_t)rows};
    const cuuint64_t gstride[1] = {(cuuint64_t)T * 8};
    const cuuint32_t box[2] = {(cuuint32_t)T, (cuuint32_t)(bx + 2)};
    const cuuint32_t es[2] = {1, 1};
    patch = enc != nullptr && rows < INT32_MAX &&
            enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X - (int64_t)gp.gb * plane * T), gdim,
                gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const bool swz = patch && T == 16 && swz_env;
  const size_t SB = grid_stage_bytes<T>(bx, by, hy, vs, swz);
  const bool xscr = !K::CG && T >= 16 && (patch ? (T == 16 && !swz && pv_env != 2) : true);  // the kernel's XSCR
  const size_t fixed = (size_t)((K::CG ? 2 : 1) + (xscr ? 1 : 0)) * K::NWC * K::yr(patch) * K::S * 8 + 16 * 8 + 128 +
                       (swz ? 1024 : 0);
  int ns = (int)((220 * 1024 - fixed) / SB);
  if (ns > 8) ns = 8;
  if (ns < 4) return cudaErrorInvalidConfiguration;
  size_t sm = (size_t)ns * SB + fixed;
  if (sm < (size_t)(T * T + T) * 8) sm = (size_t)(T * T + T) * 8;
  nblk = nblk < sms ? nblk : sms;  // one persistent CTA per SM
  if constexpr (PATCH_T) {
    if (patch && swz) {
      cudaFuncSetAttribute(k_spmm_grid<T, W, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      return launch_k(k_spmm_grid<T, W, true, 1>, nblk, K::NTH, sm, st, gp, bx, by, zc, X, Y, r, part, tl, ch,
                      ns, gram, tm);
    }
    if (patch && pv_env == 2 && T == 16) {
      cudaFuncSetAttribute(k_spmm_grid<T, W, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      return launch_k(k_spmm_grid<T, W, true, 2>, nblk, K::NTH, sm, st, gp, bx, by, zc, X, Y, r, part, tl, ch,
                      ns, gram, tm);
    }
    if (patch) {
      cudaFuncSetAttribute(k_spmm_grid<T, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      return launch_k(k_spmm_grid<T, W, true>, nblk, K::NTH, sm, st, gp, bx, by, zc, X, Y, r, part, tl, ch, ns,
                      gram, tm);
    }
  }
  cudaFuncSetAttribute(k_spmm_grid<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  return launch_k(k_spmm_grid<T, W>, nblk, K::NTH, sm, st, gp, bx, by, zc, X, Y, r, part, tl, ch, ns, gram, tm);
}

// Setup: the stencil values per row from the uploaded CSR (columns in the extended layout, so the offset
// of entry p of local row i is col[p] − halo_before − i in both the one-rank and the ghost-plane case):
// sv[i][k] = val[p] for the slot k of that offset (ascending: −c, −b, −1, 0, 1, b, c; 2D without ±c),
// 0 in absent slots; an entry at no slot or crossing an x-line (y-plane) boundary sets *bad.
__global__ void __launch_bounds__(256) k_grid_sv(int64_t n, const int* __restrict__ rp, const int* __restrict__ col,
                                                 const double* __restrict__ val, int64_t row_begin, int64_t halo_before,
                                                 int64_t nx, int64_t ny, int64_t b, int64_t c, int w,
                                                 double* __restrict__ sv, int* __restrict__ bad) {
  const int VS = (w + 1) & ~1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = row_begin + i, x = gi % nx, y = (gi / nx) % ny;
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool ok = true;
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t o = (int64_t)col[p] - halo_before - i;
      int k;
      if (w == 7) k = o == -c ? 0 : o == -b ? 1 : o == -1 ? 2 : o == 0 ? 3 : o == 1 ? 4 : o == b ? 5 : o == c ? 6 : -1;
      else k = o == -b ? 0 : o == -1 ? 1 : o == 0 ? 2 : o == 1 ? 3 : o == b ? 4 : -1;
      if (k < 0 || (o == 1 && x + 1 >= nx) || (o == -1 && x == 0) ||
          (w == 7 && ((o == b && y + 1 >= ny) || (o == -b && y == 0))))
        ok = false;
      else
        v[k] = val[p];
    }
    if (!ok) atomicExch(bad, 1);
#pragma unroll
    for (int k = 0; k < 8; k += 2)
      if (k < VS) *reinterpret_cast<double2*>(sv + i * VS + k) = make_double2(v[k], v[k + 1]);
  }
}

cudaError_t launch_grid_sv(cudaStream_t st, int64_t n, const int* rp, const int* col, const double* val,
                           int64_t row_begin, int64_t halo_before, int64_t nx, int64_t ny, int64_t b, int64_t c, int w,
                           double* sv, int* bad, int sms) {
  if (w != 5 && w != 7) return cudaErrorInvalidValue;
  k_grid_sv<<<sms * 8, 256, 0, st>>>(n, rp, col, val, row_begin, halo_before, nx, ny, b, c, w, sv, bad);
  return cudaGetLastError();
}

bool spmm_grid_fused_chol(int t) { return t == 8 || t == 16; }

bool spmm_grid_fits(int t, const GridPlan& gp) {
  if (gp.sv == nullptr || (gp.w != 5 && gp.w != 7)) return false;
  int bx = 0, by = 0, zc = 0;
  switch (t) {
    case 8: grid_shape<8>(gp, bx, by, zc, 148); break;
    case 16: grid_shape<16>(gp, bx, by, zc, 148); break;
    case 32: grid_shape<32>(gp, bx, by, zc, 148); break;
    case 64: grid_shape<64>(gp, bx, by, zc, 148); break;
    default: return false;
  }
  const int hy = gp.ny > 1 ? 1 : 0;
  const size_t SB = (size_t)(bx + 2) * (by + 2 * hy) * t * 8 + (size_t)(2048 / t) * ((gp.w + 1) & ~1) * 8 + 128;
  return 4 * SB + 16 * 1024 < 220 * 1024;
}

cudaError_t launch_spmm_grid(cudaStream_t st, int t, const GridPlan& gp, const double* X, double* Y, const double* r,
                             double* part, int nblk, const Tail& tl, const CholArgs& ch, bool gram) {
  if (ch.on && (!spmm_grid_fused_chol(t) || !gram)) return cudaErrorInvalidValue;
#define EKS_GRID_W(TT)                                                                  \
  return gp.w == 7 ? grid_t<TT, 7>(st, gp, X, Y, r, part, nblk, tl, ch, gram)           \
                   : grid_t<TT, 5>(st, gp, X, Y, r, part, nblk, tl, ch, gram);
  switch (t) {
    case 8: EKS_GRID_W(8)
    case 16: EKS_GRID_W(16)
    case 32: EKS_GRID_W(32)
    case 64: EKS_GRID_W(64)
    default: return cudaErrorInvalidValue;
  }
#undef EKS_GRID_W
}

}  // namespace eks
