// eks.cu — host driver and C ABI of libeks.so (include/eks.h, include/eks_kernels.h).
//
// One process per GPU.  Rank r owns a contiguous row slab; its n×t blocks are
// stored row-major with ghost rows ("halo") from the other ranks in an
// extended layout [ghosts of lower ranks | local rows | ghosts of higher ranks],
// so the SpMM indexes one array with remapped column indices.  Communication is
// NCCL: one halo exchange (ncclSend/ncclRecv on a comm stream, overlapped with
// the interior rows) per SpMM and one ncclAllReduce per reduced small
// matrix (CGS2 coefficients, Gram + Z2ᵀr, ρ²).  No CPU fallback: without a CUDA
// device every call fails with EKS_ERR_CUDA.
#include "../../include/eks.h"
#include "../../include/eks_kernels.h"
#include "eks_kernels.cuh"
#include "eks_sweep.cuh"

#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

using eks::kThreads;

namespace {

struct Recv { int peer; int64_t lo, hi, ext_off; };  // ghost rows [lo,hi) of peer → ext rows ext_off..
struct Send { int peer; int64_t lo, hi; };           // my global rows [lo,hi) → peer

struct Block {
  double* base = nullptr;  // ext allocation (ghost rows included) or local allocation
  double* loc = nullptr;   // first local row
  bool owned = true;       // false: aliases another Block's storage (store-Q-only AW ring)
  double* alloc = nullptr; // deep-ghost blocks of the matrix-powers kernel: the allocation (base = loc − halo rows)
};

struct ProfRec { int cls; cudaEvent_t a, b; };

}  // namespace

struct eks_ctx {
  int device = 0, rank = 0, nranks = 1;
  cudaStream_t stream = nullptr, own = nullptr, comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  ncclComm_t comm = nullptr;
  int sms = 148, nblk = 296, rho_nblk = 296;  // rho_nblk: CTAs that wrote the last scalar partials
  std::string err;
  // matrix (local slab)
  bool have_matrix = false;
  int64_t n_global = 0, row_begin = 0, row_end = 0, n = 0, nnz = 0;
  int* d_rp = nullptr;
  int* d_col = nullptr;
  double* d_val = nullptr;
  int64_t halo_before = 0, halo_after = 0;
  std::vector<Recv> recvs;
  std::vector<Send> sends;
  int64_t int_lo = 0, int_hi = 0;  // interior local rows (all columns local)
  int64_t maxrow = 0;              // longest local CSR row
  int ell_w = 0;                   // ELL copy of A (rows ≤ 8 entries): slots per row, 0 = none
  int* d_ecol = nullptr;
  double* d_eval = nullptr;
  int* d_tmax = nullptr;           // per ELL tile: largest ext column (L2 prefetch of the far slab)
  // segment plan of the TMA-staged SpMM (eks_sweep.cuh SegPlan); device arrays owned here
  bool seg_ok = false;
  eks::SegPlan seg{};
  int* d_seg = nullptr;
  int* d_segrows = nullptr;
  int* d_segown = nullptr;
  unsigned short* d_lidx = nullptr;
  double* d_sval = nullptr;
  int spmm_path = 0;               // 0 auto, 1 ell, 2 csr, 3 seg, 4 grid (EKS_SPMM_PATH, for A/B measurements)
  // stencil structure (eks_grid.cu GridPlan): plane-marching SpMM
  bool grid_ok = false;
  eks::GridPlan gplan{};
  double* d_sv = nullptr;
  // matrix-powers kernel of the CA variants at N > 1: stencil values of the
  // slab plus mpk_d ghost planes of each neighbour (exchanged once), slab table of all ranks
  std::vector<int64_t> ranges;
  double* mpk_sv = nullptr;
  int mpk_d = 0;           // ghost depth mpk_sv holds (0: not built)
  int mpk_ok_t = 0, mpk_ok_d = 0, mpk_ok = -1;  // cached all-ranks decision for (t, d): −1 unknown
  int ca_deep = 0;         // ghost depth (planes) the Vca blocks were allocated with
  // communication-avoiding outer iteration: the s monomial blocks, their A-products, the st×st
  // Gram / factor / inverse, g = Vᵀr and α̃
  std::vector<Block> Vca, AVca;
  double *Bca = nullptr, *gca = nullptr, *Rca = nullptr, *Rinvca = nullptr, *alphaca = nullptr, *Btmp = nullptr;
  double* cawork = nullptr;  // global workspace of the st×st Cholesky when st > kCaSmem
  int ca_cap = 0;  // st the buffers were sized for
  int chol_mode = 0;               // 0 one-warp Cholesky launch (default), 1 in the SpMM kernel's tail (EKS_CHOL)
  int ortho = 0;                   // 0 A-CholQR, 1 Pre-CholQR (eks_options.ortho, reading R30)
  // block-Jacobi IC(0) preconditioner (eks_setup_precond, reading R32): sweep [0] = forward with
  // the strict lower L, [1] = backward with the strict upper Lᵗ; per-domain level schedules
  int prec_nd = 0, prec_ndl = 0;   // preconditioner domains (global), of this slab
  int* pr_rp[2] = {nullptr, nullptr};
  int* pr_col[2] = {nullptr, nullptr};
  double* pr_val[2] = {nullptr, nullptr};
  double* pr_diag = nullptr;
  int* pr_domlev[2] = {nullptr, nullptr};
  int* pr_levptr[2] = {nullptr, nullptr};
  int* pr_rows[2] = {nullptr, nullptr};
  int pr_levels[2] = {0, 0};       // longest level chain of a domain (forward, backward)
  int pr_ring[2] = {0, 0};         // shared-memory ring rows of k_trsv_ring (0: not applicable)
  int pr_E[2] = {0, 0};            // entries per position of the flattened schedule
  int* pr_prow[2] = {nullptr, nullptr};
  int* pr_pout[2] = {nullptr, nullptr};
  int pr_maxlev[2] = {0, 0};       // most levels of one domain
  int pr_maxrows[2] = {0, 0};      // most rows of one level
  int pr_maxe[2] = {0, 0};         // most off-diagonal entries of one row
  Block Zq1, Zq2;                  // the block in forward / backward schedule order
  int* pr_pne[2] = {nullptr, nullptr};
  double* pr_pdiag[2] = {nullptr, nullptr};
  int* pr_pcol[2] = {nullptr, nullptr};
  double* pr_pval[2] = {nullptr, nullptr};
  bool use_prec = false;           // this solve applies M⁻¹ (eks_options.precond)
  Block Zp;                        // M⁻¹·Z of the next block
  double* pre = nullptr;           // Pre-CholQR / restructured scratch: [G | R1⁻¹ | −R1⁻¹ | g] (3t²+t)
  // workspace, keyed by t
  int ws_t = 0;
  std::vector<Block> Wpool, AWpool;  // Wpool ext layout, AWpool local
  // store-Q-only mode of the full-basis methods (eks_options.aq_cache, reading R24): A·Q is not kept;
  // AWpool entries alias a ring of two local blocks (A·W of the last two blocks), CGS2 takes
  // C = Qᵀ(A·Z) with explicit SpMMs of Z and Z1 (scratch: Ze ext, Ysc local)
  bool aq_off = false, last_aq_off = false;
  // lazy basis (s-step SRE-CG and the basis sweep, t ≥ 8): a ring slot keeps Z2 (not W = Z2 R⁻¹), its
  // A·W and R⁻¹ (Rslot, t×t per slot); Q·C products use R⁻¹C (folded by the sweeps)
  bool lazy = false, last_lazy = false;
  double* Rslot = nullptr;
  int rslot_cap = 0;
  Block AWring[2], Ze, Ysc;
  Block Zs, Z1, xv, tmpv;            // xv: ext vector
  double *b = nullptr, *r = nullptr, *rnew = nullptr, *dx = nullptr;
  double* part = nullptr;
  size_t part_cap = 0;  // doubles
  double *C1 = nullptr, *C2 = nullptr;
  size_t C_cap = 0;
  double* part2 = nullptr;  // per-CTA partials of the fused next-block C1
  size_t part2_cap = 0;
  bool c1_ready = false;    // C1 of the next CGS pass already reduced into C1
  // one-synch CGS2 (eks_options.onesynch, reading R36): [C2 | B1 | g1] of a block in one buffer, one
  // stacked reduction per block (2 per block with C1, 2s+1 per outer iteration with ρ²)
  bool onesynch = false;
  double* os = nullptr;
  size_t os_cap = 0;
  double *Bg = nullptr, *Rm = nullptr, *Rinv = nullptr, *alpha = nullptr, *scal = nullptr;
  int alpha_cap = 0;
  int* flag = nullptr;
  unsigned* cnt = nullptr;   // arrival counters of the tail reductions (one per call site, self-resetting)
  bool rho_fused = false;    // ‖r_k‖² already reduced into scal[1] by the last block's R⁻¹ kernel
  bool chol_fused = false;   // R, R⁻¹, α̃ of the block already produced by the SpMM+Gram kernel
  double* h_scal = nullptr;  // pinned: [0..3] doubles, [4] flag as double
  int* h_flag = nullptr;     // pinned INT_MAX source
  std::vector<double> hist;
  // device-resident loop control (eks_options.use_graph = 2): loop state and ρ history on the device
  eks::LoopState* d_loop = nullptr;
  double* d_hist = nullptr;
  size_t hist_cap = 0;
  // profiling
  bool prof_on = false;
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> ev_pool;
  eks_profile prof{};
  long long launches = 0;
  double model_bytes = 0.0, model_flops = 0.0;
  // basis bookkeeping of the last solve / sweep (eks_k_last_basis)
  int last_t = 0, last_nblocks = 0, last_ring = 0;
};

namespace {

eks_status fail(eks_ctx* c, eks_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return st;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(ctx, EKS_ERR_CUDA, "%s: %s (%s:%d)", #call,               \
                                       cudaGetErrorString(e_), __FILE__, __LINE__);              \
  } while (0)
#define NK(call)                                                                                  \
  do {                                                                                            \
    ncclResult_t r_ = (call);                                                                     \
    if (r_ != ncclSuccess) return fail(ctx, EKS_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)
#define ST(call)                     \
  do {                               \
    eks_status s_ = (call);          \
    if (s_ != EKS_OK) return s_;     \
  } while (0)

bool valid_t(int t) { return t == 1 || t == 2 || t == 4 || t == 8 || t == 16 || t == 32 || t == 64; }

// ---------------------------------------------------------------- profiling
cudaEvent_t pev(eks_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct KScope {
  eks_ctx* c;
  int cls;
  cudaEvent_t a = nullptr;
  KScope(eks_ctx* c_, int cls_) : c(c_), cls(cls_) {
    if (cls != EKS_K_COMM) c->launches++;  // count only this library's kernels
    c->prof.launches[cls]++;
    if (c->prof_on) {
      a = pev(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~KScope() {
    if (c->prof_on) {
      cudaEvent_t b = pev(c);
      cudaEventRecord(b, c->stream);
      c->prof_pending.push_back({cls, a, b});
    }
  }
};
void prof_harvest(eks_ctx* c) {  // call after a stream sync
  for (auto& p : c->prof_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->prof.ms[p.cls] += ms;
    c->ev_pool.push_back(p.a);
    c->ev_pool.push_back(p.b);
  }
  c->prof_pending.clear();
}

void account(eks_ctx* c, int cls, double bytes, double flops) {
  c->prof.bytes[cls] += bytes;
  c->prof.flops[cls] += flops;
  c->model_bytes += bytes;
  c->model_flops += flops;
}

// ---------------------------------------------------------------- memory
eks_status dalloc(eks_ctx* ctx, double** p, size_t count) {
  if (*p) return EKS_OK;
  cudaError_t e = cudaMalloc((void**)p, sizeof(double) * (count ? count : 1));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(ctx, EKS_ERR_OOM, "cudaMalloc(%zu doubles): %s", count, cudaGetErrorString(e));
  }
  return EKS_OK;
}
void dfree(void* p) {
  if (p) cudaFree(p);
}

int64_t n_ext(const eks_ctx* c) { return c->halo_before + c->n + c->halo_after; }

eks_status alloc_block(eks_ctx* ctx, Block* B, int t, bool ext) {
  if (B->base) return EKS_OK;
  int64_t rows = ext ? n_ext(ctx) : ctx->n;
  ST(dalloc(ctx, &B->base, (size_t)rows * t));
  B->loc = B->base + (ext ? ctx->halo_before * t : 0);
  return EKS_OK;
}

void free_workspace(eks_ctx* c) {
  for (auto& b : c->Vca) dfree(b.alloc ? b.alloc : b.base);
  for (auto& b : c->AVca) dfree(b.base);
  c->Vca.clear();
  c->AVca.clear();
  for (double** p : {&c->Bca, &c->gca, &c->Rca, &c->Rinvca, &c->alphaca, &c->Btmp, &c->pre, &c->cawork}) {
    dfree(*p);
    *p = nullptr;
  }
  c->ca_cap = 0;
  for (auto& b : c->Wpool) if (b.owned) dfree(b.base);
  for (auto& b : c->AWpool) if (b.owned) dfree(b.base);
  c->Wpool.clear();
  c->AWpool.clear();
  for (Block* b : {&c->Zs, &c->Z1, &c->xv, &c->tmpv, &c->Zp, &c->Zq1, &c->Zq2, &c->AWring[0], &c->AWring[1], &c->Ze,
                   &c->Ysc}) {
    dfree(b->base);
    *b = Block{};
  }
  for (double** p : {&c->b, &c->r, &c->rnew, &c->dx, &c->part, &c->C1, &c->C2, &c->Bg, &c->Rm, &c->Rinv,
                     &c->alpha, &c->scal, &c->Rslot, &c->os}) { dfree(*p); *p = nullptr; }
  c->rslot_cap = 0;
  c->os_cap = 0;
  dfree(c->flag);
  c->flag = nullptr;
  dfree(c->cnt);
  c->cnt = nullptr;
  c->part_cap = c->C_cap = 0;
  dfree(c->part2);
  c->part2 = nullptr;
  c->part2_cap = 0;
  c->c1_ready = false;
  c->alpha_cap = 0;
  c->ws_t = 0;
}

eks_status ensure_workspace(eks_ctx* ctx, int t, int s) {
  if (ctx->ws_t != t) {
    free_workspace(ctx);
    ctx->ws_t = t;
  }
  ST(alloc_block(ctx, &ctx->Zs, t, false));
  ST(alloc_block(ctx, &ctx->Z1, t, false));
  ST(alloc_block(ctx, &ctx->xv, 1, true));
  ST(alloc_block(ctx, &ctx->tmpv, 1, false));
  for (double** p : {&ctx->b, &ctx->r, &ctx->rnew, &ctx->dx}) ST(dalloc(ctx, p, (size_t)ctx->n));
  ST(dalloc(ctx, &ctx->Bg, (size_t)t * t + t));
  ST(dalloc(ctx, &ctx->Rm, (size_t)t * t));
  ST(dalloc(ctx, &ctx->Rinv, (size_t)t * t));
  if (ctx->rslot_cap < 3) {  // R⁻¹ of the 3 ring slots of the lazy basis
    dfree(ctx->Rslot);
    ctx->Rslot = nullptr;
    ST(dalloc(ctx, &ctx->Rslot, (size_t)3 * t * t));
    ctx->rslot_cap = 3;
  }
  ST(dalloc(ctx, &ctx->pre, (size_t)3 * t * t + t));
  ST(dalloc(ctx, &ctx->scal, 16));
  if (!ctx->flag) {  // flag[0]: breakdown block (atomicMin); flag[3]: INT_MAX, the device-side reset source
    CK(cudaMalloc((void**)&ctx->flag, sizeof(int) * 4));
    CK(cudaMemcpy(ctx->flag + 3, ctx->h_flag, sizeof(int), cudaMemcpyHostToDevice));
  }
  if (!ctx->cnt) {
    CK(cudaMalloc((void**)&ctx->cnt, sizeof(unsigned) * 16));
    CK(cudaMemset(ctx->cnt, 0, sizeof(unsigned) * 16));
  }
  if (ctx->alpha_cap < s * t) {
    dfree(ctx->alpha);
    ctx->alpha = nullptr;
    ST(dalloc(ctx, &ctx->alpha, (size_t)s * t));
    ctx->alpha_cap = s * t;
  }
  size_t need_part = (size_t)ctx->nblk * ((size_t)t * t + t + 8);
  if (ctx->part_cap < need_part) {
    dfree(ctx->part);
    ctx->part = nullptr;
    ST(dalloc(ctx, &ctx->part, need_part));
    ctx->part_cap = need_part;
  }
  return EKS_OK;
}

eks_status ensure_part(eks_ctx* ctx, size_t doubles) {
  if (ctx->part_cap >= doubles) return EKS_OK;
  dfree(ctx->part);
  ctx->part = nullptr;
  ST(dalloc(ctx, &ctx->part, doubles));
  ctx->part_cap = doubles;
  return EKS_OK;
}

eks_status ensure_C(eks_ctx* ctx, size_t doubles) {
  if (ctx->C_cap >= doubles) return EKS_OK;
  dfree(ctx->C1);
  dfree(ctx->C2);
  ctx->C1 = ctx->C2 = nullptr;
  ST(dalloc(ctx, &ctx->C1, doubles));
  ST(dalloc(ctx, &ctx->C2, doubles));
  ctx->C_cap = doubles;
  return EKS_OK;
}

// Tail reduction of a producer kernel's per-CTA partials into out[0..count) (eks_device.cuh).
eks_status ensure_os(eks_ctx* ctx, size_t doubles) {
  if (ctx->os_cap >= doubles) return EKS_OK;
  dfree(ctx->os);
  ctx->os = nullptr;
  ST(dalloc(ctx, &ctx->os, doubles));
  ctx->os_cap = doubles;
  return EKS_OK;
}

eks::Tail tail(eks_ctx* ctx, int slot, double* out, size_t count, double* out2 = nullptr, int split = INT_MAX) {
  eks::Tail tl;
  tl.cnt = ctx->cnt + slot;
  tl.out = out;
  tl.out2 = out2;
  tl.count = (int)count;
  tl.split = split;
  return tl;
}

// ---------------------------------------------------------------- communication
eks_status allreduce(eks_ctx* ctx, double* buf, size_t count) {
  if (ctx->nranks == 1 || count == 0) return EKS_OK;
  KScope k(ctx, EKS_K_COMM);
  NK(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  return EKS_OK;
}

eks_status halo_start(eks_ctx* ctx, const Block& X, int t) {
  if (ctx->nranks == 1) return EKS_OK;
  CK(cudaEventRecord(ctx->ev_ready, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_ready, 0));
  NK(ncclGroupStart());
  for (const Send& s : ctx->sends)
    NK(ncclSend(X.loc + (s.lo - ctx->row_begin) * t, (size_t)(s.hi - s.lo) * t, ncclDouble, s.peer, ctx->comm,
                ctx->comm_stream));
  for (const Recv& r : ctx->recvs)
    NK(ncclRecv(X.base + r.ext_off * t, (size_t)(r.hi - r.lo) * t, ncclDouble, r.peer, ctx->comm,
                ctx->comm_stream));
  NK(ncclGroupEnd());
  CK(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
  return EKS_OK;
}

int spmm_path_for(const eks_ctx* ctx, int t);

bool gram_split_env() {
  static const bool on = [] {  // EKS_GRAM64=fused: the in-kernel CTA-level Gram at t = 64 (A/B measurements)
    const char* e = getenv("EKS_GRAM64");
    return !(e && !strcmp(e, "fused"));
  }();
  return on;
}

// Y = A X.  Stencil operators (t ≥ 8): the plane-marching kernel without its Gram epilogue, after the
// ghost-plane exchange.  Otherwise CSR with the halo exchange overlapped with the interior rows.
eks_status spmm(eks_ctx* ctx, const Block& X, double* Y, int t) {
  if (eks::sweep_supported(t) && spmm_path_for(ctx, t) == 4) {
    ST(halo_start(ctx, X, t));
    if (ctx->nranks > 1) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    account(ctx, EKS_K_SPMM, 8.0 * ctx->gplan.w * ctx->n + 16.0 * ctx->n * t, 2.0 * ctx->nnz * t);
    KScope k(ctx, EKS_K_SPMM);
    CK(eks::launch_spmm_grid(ctx->stream, t, ctx->gplan, X.loc, Y, nullptr, nullptr, ctx->nblk, eks::Tail{},
                             eks::CholArgs{}, false));
    return EKS_OK;
  }
  ST(halo_start(ctx, X, t));
  account(ctx, EKS_K_SPMM, 12.0 * ctx->nnz + 4.0 * (ctx->n + 1) + 16.0 * ctx->n * t, 2.0 * ctx->nnz * t);
  if (ctx->nranks == 1) {
    KScope k(ctx, EKS_K_SPMM);
    CK(eks::launch_spmm(ctx->stream, t, 0, (int)ctx->n, ctx->d_rp, ctx->d_col, ctx->d_val, X.base, Y, ctx->sms));
    return EKS_OK;
  }
  {
    KScope k(ctx, EKS_K_SPMM);
    CK(eks::launch_spmm(ctx->stream, t, (int)ctx->int_lo, (int)ctx->int_hi, ctx->d_rp, ctx->d_col, ctx->d_val,
                        X.base, Y, ctx->sms));
  }
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
  {
    KScope k(ctx, EKS_K_SPMM);
    CK(eks::launch_spmm(ctx->stream, t, 0, (int)ctx->int_lo, ctx->d_rp, ctx->d_col, ctx->d_val, X.base, Y,
                        ctx->sms));
    CK(eks::launch_spmm(ctx->stream, t, (int)ctx->int_hi, (int)ctx->n, ctx->d_rp, ctx->d_col, ctx->d_val, X.base,
                        Y, ctx->sms));
  }
  return EKS_OK;
}

// out (nl·t·t [+t]) = Σ over all rows of Lᵀ R [and L_0ᵀ v], allreduced over ranks unless `ar` is
// false (the caller then stacks several outputs into one allreduce).
eks_status tn_reduce(eks_ctx* ctx, int t, int nl, const double* const* L, const double* R, const double* v,
                     double* out, bool ar = true) {
  if (v && nl != 1) return fail(ctx, EKS_ERR_INVALID_ARG, "internal: v needs one left block");
  const size_t total = (size_t)nl * t * t + (v ? t : 0);
  if (eks::sweep_supported(t)) {
    const int maxb = eks::sweep_max_blocks(t);
    for (int j0 = 0; j0 < nl;) {
      int k = 1;
      while (2 * k <= maxb && 2 * k <= nl - j0) k *= 2;  // power-of-two chunks of left blocks
      eks::SweepPtrs P{};
      for (int j = 0; j < k; ++j) P.l[j] = L[j0 + j];
      const size_t stride = eks::sweep_part_stride(t, k, v != nullptr);
      ST(ensure_part(ctx, stride * ctx->nblk));
      account(ctx, EKS_K_COEF, 8.0 * ctx->n * ((double)(k + 1) * t + (v ? 1 : 0)),
              2.0 * ctx->n * t * (t * k + (v ? 1 : 0)));
      {
        KScope ks(ctx, EKS_K_COEF);  // partials reduced by the sweep's last CTAs into out
        CK(eks::launch_sweep(ctx->stream, t, 0, k, v != nullptr, ctx->n, R, nullptr, P, nullptr, v, ctx->part,
                             ctx->nblk, tail(ctx, 1, out + (size_t)j0 * t * t, stride)));
      }
      j0 += k;
    }
    return ar ? allreduce(ctx, out, total) : EKS_OK;
  }
  const size_t stride = eks::tn_partials_stride(t, nl, v != nullptr);
  ST(ensure_part(ctx, stride * ctx->nblk));
  account(ctx, EKS_K_COEF, 8.0 * ctx->n * ((double)(nl + 1) * t + (v ? 1 : 0)), 2.0 * ctx->n * t * (t * nl + (v ? 1 : 0)));
  {
    KScope k(ctx, EKS_K_COEF);
    CK(eks::launch_tn_partials(ctx->stream, t, ctx->n, nl, L, R, v, ctx->part, ctx->nblk));
  }
  {
    KScope k(ctx, EKS_K_REDUCE);
    CK(eks::launch_reduce(ctx->stream, ctx->part, ctx->nblk, stride, stride, out));
  }
  return ar ? allreduce(ctx, out, stride) : EKS_OK;
}

// Zout = Zin − Σ_j Q_j C_j  (CGS update)
eks_status ts_update(eks_ctx* ctx, int t, int nq, const double* const* Q, const double* C, const double* Zin,
                     double* Zout, const double* const* RQ = nullptr) {
  if (eks::sweep_supported(t)) {
    const int maxb = eks::sweep_max_blocks(t);
    for (int j0 = 0; j0 < nq;) {
      const int k = std::min(maxb, nq - j0);
      eks::SweepPtrs P{};
      for (int j = 0; j < k; ++j) {
        P.q[j] = Q[j0 + j];
        P.rq[j] = RQ ? RQ[j0 + j] : nullptr;  // lazy blocks: Q_j = Z2_j R_j⁻¹
      }
      account(ctx, EKS_K_UPDATE, 8.0 * ctx->n * ((double)k * t + 2.0 * t), 2.0 * ctx->n * t * t * k);
      KScope ks(ctx, EKS_K_UPDATE);
      CK(eks::launch_sweep(ctx->stream, t, k, 0, false, ctx->n, j0 == 0 ? Zin : Zout, Zout, P,
                           C + (size_t)j0 * t * t, nullptr, nullptr, ctx->nblk));
      j0 += k;
    }
    return EKS_OK;
  }
  account(ctx, EKS_K_UPDATE, 8.0 * ctx->n * ((double)nq * t + 2.0 * t), 2.0 * ctx->n * t * t * nq);
  KScope k(ctx, EKS_K_UPDATE);
  CK(eks::launch_ts_update(ctx->stream, t, ctx->n, nq, Q, C, Zin, Zout, ctx->nblk));
  return EKS_OK;
}

// Fused CGS pass: Z1 = Z − Q C1 and C2 = (AQ)ᵀ Z1 in one sweep (nq ≤ 2 window of SRE-CG).
eks_status update_coef(eks_ctx* ctx, int t, int nq, const double* const* Q, const double* const* AQ,
                       const double* C1, const double* Z, double* Z1, double* C2, bool ar = true,
                       const double* const* RQ = nullptr) {
  eks::SweepPtrs P{};
  for (int j = 0; j < nq; ++j) {
    P.q[j] = Q[j];
    P.l[j] = AQ[j];
    P.rq[j] = RQ ? RQ[j] : nullptr;
  }
  const size_t stride = eks::sweep_part_stride(t, nq, false);
  ST(ensure_part(ctx, stride * ctx->nblk));
  // algorithmic bytes: read Z, Q_j, AQ_j (once each — for SRE-CG Z is AQ_last itself), write Z1
  const bool alias = nq > 0 && AQ[nq - 1] == Z;
  account(ctx, EKS_K_UPCOEF, 8.0 * ctx->n * ((double)2 * nq * t + 2.0 * t - (alias ? t : 0)),
          4.0 * ctx->n * t * t * nq);
  {
    KScope ks(ctx, EKS_K_UPCOEF);  // C2 partials reduced by the sweep's last CTAs
    CK(eks::launch_sweep(ctx->stream, t, nq, nq, false, ctx->n, Z, Z1, P, C1, nullptr, ctx->part, ctx->nblk,
                         tail(ctx, 0, C2, stride)));
  }
  return ar ? allreduce(ctx, C2, stride) : EKS_OK;
}

// Which fused SpMM+Gram kernel runs for this t: 4 plane-marching (stencil-structured A), 0 TMA-
// staged segments, 1 ELL gathers, 2 CSR.  Measured (tools/spmm_micro.py): plane-marching is
// fastest for t ≤ 32, then ELL; the segment kernel for t = 64.  EKS_SPMM_PATH=grid|seg|ell|csr
// forces one for A/B measurements.
int spmm_path_for(const eks_ctx* ctx, int t) {
  const bool grid = ctx->grid_ok && eks::spmm_grid_fits(t, ctx->gplan);
  if (grid && (ctx->spmm_path == 4 || ctx->spmm_path == 0)) return 4;
  const bool seg = ctx->seg_ok && eks::spmm_seg_fits(t, ctx->ell_w, ctx->seg.cap);
  if (seg && (ctx->spmm_path == 3 || (ctx->spmm_path == 0 && t == 64))) return 0;
  if (ctx->ell_w && ctx->spmm_path <= 1) return 1;
  return 2;
}

// Y = A·X and out = [XᵀY | Xᵀr] (t·t + t, allreduced): the A-CholQR Gram with the α̃ projection.
// One rank: the fused SpMM+Gram kernel, whose last CTA also factors B when `ch` is given
// (t ≤ 32; ctx->chol_fused tells the caller).  Several ranks: SpMM with halo overlap, then
// the Gram sweep and an allreduce.
eks_status spmm_gram(eks_ctx* ctx, const Block& X, double* Y, int t, const double* r, double* out,
                     const eks::CholArgs* ch = nullptr, bool ar = true) {
  ctx->chol_fused = false;
  const bool grid_multi = ctx->nranks != 1 && eks::sweep_supported(t) && spmm_path_for(ctx, t) == 4;
  if ((ctx->nranks != 1 && !grid_multi) || !eks::sweep_supported(t)) {
    ST(spmm(ctx, X, Y, t));
    const double* L[1] = {X.loc};
    return tn_reduce(ctx, t, 1, L, Y, r, out, ar);
  }
  if (t == 64 && spmm_path_for(ctx, t) == 4 && gram_split_env()) {
    // t = 64: the plane-marching SpMM without its Gram, then the Gram [Z2ᵀ(AZ2) (upper tiles) | Z2ᵀr]
    // as its own DMMA sweep over Z2 and AZ2 — the in-kernel CTA-level Gram was LSU/latency-bound
    // (0.20 of HBM); measured faster together (profiles/spmm_micro_r02.txt)
    ST(spmm(ctx, X, Y, t));
    const size_t stride = eks::sweep_part_stride(t, 1, r != nullptr);
    ST(ensure_part(ctx, stride * ctx->nblk));
    account(ctx, EKS_K_COEF, 8.0 * ctx->n * (2.0 * t + (r ? 1.0 : 0.0)), ctx->n * t * (t + 8.0) + 2.0 * ctx->n * t);
    {
      KScope k(ctx, EKS_K_COEF);
      CK(eks::launch_gram_upper(ctx->stream, t, ctx->n, X.loc, Y, r, ctx->part, ctx->nblk, tail(ctx, 2, out, stride)));
    }
    return (ar && ctx->nranks > 1) ? allreduce(ctx, out, stride) : EKS_OK;
  }
  if (grid_multi) {  // ghost planes first (the persistent kernel occupies every SM: no overlap)
    ST(halo_start(ctx, X, t));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
  }
  const size_t stride = eks::sweep_part_stride(t, 1, true);
  ST(ensure_part(ctx, stride * ctx->nblk));
  eks::CholArgs c{};
  const int path = spmm_path_for(ctx, t);
  // algorithmic bytes of the representation of A the kernel streams: CSR 12·nnz + 4(n+1); the
  // plane-marching kernel's stencil values 8·w per row (no indices); + X read, Y written, r read
  const double abytes = path == 4 ? 8.0 * ctx->gplan.w * ctx->n : 12.0 * ctx->nnz + 4.0 * (ctx->n + 1);
  account(ctx, EKS_K_SPMM, abytes + 16.0 * ctx->n * t + (r ? 8.0 * ctx->n : 0.0), 2.0 * ctx->nnz * t);
  account(ctx, EKS_K_COEF, 0.0, 2.0 * ctx->n * t * (t + 1));  // the Gram epilogue: flops only
  // EKS_CHOL=1: the SpMM kernel's last CTA factors B (measured slower than the separate one-warp
  // launch the solve uses by default: 1894 vs 2085 outer it/s on cfg2)
  if (ch && ctx->chol_mode == 1 && ctx->nranks == 1 &&
      ((path == 4 && eks::spmm_grid_fused_chol(t)) || (path != 4 && eks::spmm_gram_fused_chol(t)))) {
    c = *ch;
    c.on = 1;
  }
  {
    KScope k(ctx, EKS_K_SPMM);
    if (path == 4)
      CK(eks::launch_spmm_grid(ctx->stream, t, ctx->gplan, X.loc, Y, r, ctx->part, ctx->nblk,
                               tail(ctx, 2, out, stride), c));
    else if (path == 0)
      CK(eks::launch_spmm_seg(ctx->stream, t, ctx->n, ctx->seg, ctx->ell_w, X.base, Y, r, ctx->part, ctx->nblk,
                              tail(ctx, 2, out, stride), c));
    else if (path == 1)
      CK(eks::launch_spmm_gram_ell(ctx->stream, t, ctx->n, ctx->d_ecol, ctx->d_eval, ctx->ell_w, ctx->d_tmax, n_ext(ctx),
                                   X.base,
                                   (int64_t)(X.loc - X.base) / t, Y, r, ctx->part, ctx->nblk, tail(ctx, 2, out, stride),
                                   c));
    else
      CK(eks::launch_spmm_gram(ctx->stream, t, ctx->n, ctx->d_rp, ctx->d_col, ctx->d_val, (int)ctx->maxrow, X.base,
                               (int64_t)(X.loc - X.base) / t, Y, r, ctx->part, ctx->nblk, tail(ctx, 2, out, stride),
                               c));
  }
  ctx->chol_fused = c.on != 0;
  return (ar && ctx->nranks > 1) ? allreduce(ctx, out, stride) : EKS_OK;
}

// CGS2 of Z against the window (Q, AQ): two passes of C = (AQ)ᵀZ, Z -= Q C (reading R3/R24).
eks_status cgs2(eks_ctx* ctx, int t, const std::vector<const double*>& Q, const std::vector<const double*>& AQ,
                const double* Z, double* Zout, const std::vector<const double*>* RQv = nullptr) {
  const int nq = (int)Q.size();
  const double* const* RQ = (RQv && !RQv->empty()) ? RQv->data() : nullptr;
  if (AQ.empty() && nq > 0) {
    // store-Q-only (reading R24): twice { C = Qᵀ(A·Z) ; Z = Z − Q·C } with explicit SpMMs — the
    // oracle's definition-mode algebra; Z and Z1 pass through the ext-layout scratch Ze (ghost rows)
    ST(alloc_block(ctx, &ctx->Ze, t, true));
    ST(alloc_block(ctx, &ctx->Ysc, t, false));
    ST(ensure_C(ctx, (size_t)nq * t * t));
    ctx->c1_ready = false;
    if (Z != ctx->Ze.loc)
      CK(cudaMemcpyAsync(ctx->Ze.loc, Z, sizeof(double) * ctx->n * t, cudaMemcpyDeviceToDevice, ctx->stream));
    ST(spmm(ctx, ctx->Ze, ctx->Ysc.loc, t));
    ST(tn_reduce(ctx, t, nq, Q.data(), ctx->Ysc.loc, nullptr, ctx->C1));  // C1 = Qᵀ(A·Z)
    ST(ts_update(ctx, t, nq, Q.data(), ctx->C1, ctx->Ze.loc, ctx->Ze.loc));  // Z1 = Z − Q C1 (in place)
    ST(spmm(ctx, ctx->Ze, ctx->Ysc.loc, t));
    ST(tn_reduce(ctx, t, nq, Q.data(), ctx->Ysc.loc, nullptr, ctx->C2));  // C2 = Qᵀ(A·Z1)
    return ts_update(ctx, t, nq, Q.data(), ctx->C2, ctx->Ze.loc, Zout);      // Z2 = Z1 − Q C2
  }
  if (!ctx->c1_ready) {
    ST(ensure_C(ctx, (size_t)nq * t * t));
    ST(tn_reduce(ctx, t, nq, AQ.data(), Z, nullptr, ctx->C1));  // C1 = (AQ)ᵀ Z
  }
  ctx->c1_ready = false;  // (else C1 came fused from the previous block's R⁻¹ kernel)
  if (eks::sweep_supported(t) && eks::sweep_fused_supported(t, nq)) {
    ST(update_coef(ctx, t, nq, Q.data(), AQ.data(), ctx->C1, Z, ctx->Z1.loc, ctx->C2, true, RQ));  // Z1, C2 = (AQ)ᵀ Z1
  } else {
    ST(ts_update(ctx, t, nq, Q.data(), ctx->C1, Z, ctx->Z1.loc, RQ));
    ST(tn_reduce(ctx, t, nq, AQ.data(), ctx->Z1.loc, nullptr, ctx->C2));
  }
  ST(ts_update(ctx, t, nq, Q.data(), ctx->C2, ctx->Z1.loc, Zout, RQ));  // Z2 = Z1 − Q C2
  return EKS_OK;
}

// CGS2 of the s blocks V_i against the window with the reductions stacked: C1 of every block in
// one allreduce, C2 of every block in a second one (same kernels and arithmetic order as cgs2()).
eks_status cgs2_stacked(eks_ctx* ctx, int t, const std::vector<const double*>& Q,
                        const std::vector<const double*>& AQ, std::vector<Block>& V, std::vector<Block>& V1) {
  const int nq = (int)Q.size(), s = (int)V.size();
  const size_t cb = (size_t)nq * t * t;
  ST(ensure_C(ctx, cb * s));
  for (int i = 0; i < s; ++i) ST(tn_reduce(ctx, t, nq, AQ.data(), V[i].loc, nullptr, ctx->C1 + cb * i, false));
  ST(allreduce(ctx, ctx->C1, cb * s));
  const bool fused = eks::sweep_supported(t) && eks::sweep_fused_supported(t, nq);
  for (int i = 0; i < s; ++i) {
    if (fused) {
      ST(update_coef(ctx, t, nq, Q.data(), AQ.data(), ctx->C1 + cb * i, V[i].loc, V1[i].loc, ctx->C2 + cb * i, false));
    } else {
      ST(ts_update(ctx, t, nq, Q.data(), ctx->C1 + cb * i, V[i].loc, V1[i].loc));
      ST(tn_reduce(ctx, t, nq, AQ.data(), V1[i].loc, nullptr, ctx->C2 + cb * i, false));
    }
  }
  ST(allreduce(ctx, ctx->C2, cb * s));
  for (int i = 0; i < s; ++i) ST(ts_update(ctx, t, nq, Q.data(), ctx->C2 + cb * i, V1[i].loc, V[i].loc));
  return EKS_OK;
}

eks_status chol(eks_ctx* ctx, int t, const double* B, const double* g, double* R, double* Rinv, double* alpha,
                int gblock) {
  KScope k(ctx, EKS_K_CHOL);
  CK(eks::launch_chol(ctx->stream, t, B, g, R, Rinv, alpha, ctx->flag, gblock));
  return EKS_OK;
}

eks_status reset_flag(eks_ctx* ctx) {  // device to device (capturable into a conditional graph body)
  CK(cudaMemcpyAsync(ctx->flag, ctx->flag + 3, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
  return EKS_OK;
}

// ρ² partials → scal[slot] (allreduced)
eks_status reduce_scalar(eks_ctx* ctx, double* slot) {
  {
    KScope k(ctx, EKS_K_REDUCE);
    CK(eks::launch_reduce(ctx->stream, ctx->part, ctx->rho_nblk, 1, 1, slot));
  }
  return allreduce(ctx, slot, 1);
}

// Wait for the stream.  With NCCL (several ranks) the wait polls ncclCommGetAsyncError: a failed or
// vanished peer makes the collective on this rank fail with EKS_ERR_NCCL (the communicator is aborted,
// so the pending kernels return) instead of hanging the solve.
eks_status stream_wait(eks_ctx* ctx) {
  if (ctx->nranks == 1 || !ctx->comm) {
    CK(cudaStreamSynchronize(ctx->stream));
    return EKS_OK;
  }
  for (;;) {
    const cudaError_t q = cudaStreamQuery(ctx->stream);
    if (q == cudaSuccess) return EKS_OK;
    if (q != cudaErrorNotReady) CK(q);
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(ctx->comm, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
      ncclCommAbort(ctx->comm);
      ctx->comm = nullptr;
      return fail(ctx, EKS_ERR_NCCL, "NCCL asynchronous error: %s (communicator aborted)", ncclGetErrorString(ae));
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

eks_status sync_scalars(eks_ctx* ctx, int count) {
  CK(cudaMemcpyAsync(ctx->h_scal, ctx->scal, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_flag + 1, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ST(stream_wait(ctx));
  if (ctx->prof_on) prof_harvest(ctx);
  return EKS_OK;
}

eks_status check_ready(eks_ctx* ctx) {
  if (!ctx) return EKS_ERR_INVALID_ARG;
  if (!ctx->have_matrix) return fail(ctx, EKS_ERR_STATE, "eks_setup_csr has not been called");
  if (ctx->nranks > 1 && !ctx->comm) return fail(ctx, EKS_ERR_NCCL, "the NCCL communicator was aborted");
  CK(cudaSetDevice(ctx->device));
  return EKS_OK;
}

eks_status copy_in(eks_ctx* ctx, double* dst, const double* src, int64_t count, eks_mem where) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * count,
                     where == EKS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream));
  return EKS_OK;
}
eks_status copy_out(eks_ctx* ctx, double* dst, const double* src, int64_t count, eks_mem where) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * count,
                     where == EKS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
  return EKS_OK;
}

// block slot for global block index gb: SRE-CG ring of 3, full-Q methods one per block
eks_status slot(eks_ctx* ctx, int t, int idx, Block** W, Block** AW) {
  while ((int)ctx->Wpool.size() <= idx) {
    Block w, aw;
    ctx->Wpool.push_back(w);
    ctx->AWpool.push_back(aw);
  }
  eks_status s1 = alloc_block(ctx, &ctx->Wpool[idx], t, true);
  if (s1 != EKS_OK) return s1;
  if (ctx->aq_off) {  // store-Q-only: A·W lives in a ring of two (the next block's Z and the update)
    Block& rg = ctx->AWring[idx & 1];
    s1 = alloc_block(ctx, &rg, t, false);
    if (s1 != EKS_OK) return s1;
    Block& aw = ctx->AWpool[idx];
    if (aw.owned) dfree(aw.base);
    aw.base = rg.base;
    aw.loc = rg.loc;
    aw.owned = false;
  } else {
    if (!ctx->AWpool[idx].owned) ctx->AWpool[idx] = Block{};  // was a ring alias of a store-Q-only solve
    s1 = alloc_block(ctx, &ctx->AWpool[idx], t, false);
    if (s1 != EKS_OK) return s1;
  }
  *W = &ctx->Wpool[idx];
  *AW = &ctx->AWpool[idx];
  return EKS_OK;
}

struct Window {
  std::vector<const double*> Q, AQ, RQ;  // RQ: R⁻¹ of lazy blocks (Q holds Z2), empty otherwise
};

// Window of the next block: SRE-CG → last min(2,#) blocks (Alg 4, reading R11);
// SRE-CG2 / MSDO-CG → all blocks (Alg 3 P:151/Alg 6).
Window window_for(eks_ctx* ctx, int t, int method, int nblocks, int ring) {
  Window w;
  int first = (method == EKS_SRE_CG) ? std::max(0, nblocks - 2) : 0;
  for (int j = first; j < nblocks; ++j) {
    int idx = ring ? j % ring : j;
    w.Q.push_back(ctx->Wpool[idx].loc);
    if (!ctx->aq_off) w.AQ.push_back(ctx->AWpool[idx].loc);  // store-Q-only: AQ empty
    if (ctx->lazy) w.RQ.push_back(ctx->Rslot + (size_t)idx * t * t);
  }
  return w;
}

// Y = M⁻¹Z = L⁻ᵗL⁻¹Z for an n×t block (Y may alias Z): the two level-scheduled sweeps.
eks_status prec_apply(eks_ctx* ctx, int t, const double* Z, double* Y) {
  KScope k(ctx, EKS_K_OTHER);
  account(ctx, EKS_K_OTHER, 2.0 * (12.0 * ctx->nnz / 2 + 16.0 * ctx->n * t), 2.0 * ctx->nnz * t);
  bool ring = true;
  for (int w = 0; w < 2; ++w)
    ring = ring && ctx->pr_ring[w] && eks::trsv_ring_smem(ctx->pr_ring[w], t, ctx->pr_maxlev[w]) <= 220 * 1024;
  if (ring) {  // gather into the forward order, forward → backward order, backward → natural order
    ST(alloc_block(ctx, &ctx->Zq1, t, false));
    ST(alloc_block(ctx, &ctx->Zq2, t, false));
    CK(eks::launch_perm_gather(ctx->stream, ctx->n, t, ctx->pr_prow[0], Z, ctx->Zq1.loc, ctx->sms));
    for (int w = 0; w < 2; ++w)
      CK(eks::launch_trsv_ring(ctx->stream, ctx->prec_ndl, t, ctx->pr_ring[w], ctx->pr_maxlev[w], ctx->pr_maxrows[w],
                               ctx->pr_prow[w],
                               ctx->pr_pout[w], ctx->pr_pne[w], ctx->pr_pdiag[w], ctx->pr_pcol[w], ctx->pr_pval[w],
                               ctx->pr_E[w], ctx->pr_domlev[w], ctx->pr_levptr[w], w ? ctx->Zq2.loc : ctx->Zq1.loc,
                               w ? Y : ctx->Zq2.loc));
    return EKS_OK;
  }
  for (int w = 0; w < 2; ++w)
    if (ctx->pr_maxe[w] > 32)  // long rows: a warp per (row, column)
      CK(eks::launch_trsv_lev_long(ctx->stream, ctx->prec_ndl, t, ctx->pr_rp[w], ctx->pr_col[w], ctx->pr_val[w],
                                   ctx->pr_diag, ctx->pr_domlev[w], ctx->pr_levptr[w], ctx->pr_rows[w], w ? Y : Z, Y));
    else
      CK(eks::launch_trsv_lev(ctx->stream, ctx->prec_ndl, t, ctx->pr_rp[w], ctx->pr_col[w], ctx->pr_val[w],
                              ctx->pr_diag, ctx->pr_domlev[w], ctx->pr_levptr[w], ctx->pr_rows[w], w ? Y : Z, Y));
  return EKS_OK;
}

// Pre-CholQR's Euclidean stage on Z (in place): G = ZᵀZ = R1ᵀR1, Z ← Z R1⁻¹ (reading R30).
// AZ is scratch (overwritten later by A·Z) for the t the update sweep does not cover.
eks_status pre_euclid(eks_ctx* ctx, int t, const Block& Z, double* AZ, int gb) {
  double* G = ctx->pre;
  double* R1inv = G + (size_t)t * t;
  double* pack = R1inv + (size_t)t * t;
  const double* L[1] = {Z.loc};
  ST(tn_reduce(ctx, t, 1, L, Z.loc, nullptr, G));
  {
    KScope k(ctx, EKS_K_CHOL);
    CK(eks::launch_chol_fast(ctx->stream, t, G, nullptr, ctx->Rm, R1inv, nullptr, ctx->flag, gb));
  }
  KScope k(ctx, EKS_K_APPLY);
  account(ctx, EKS_K_APPLY, 16.0 * ctx->n * t, 2.0 * ctx->n * t * t);
  if (eks::sweep_supported(t)) {  // Z = 0 − Z·(−R1⁻¹) on the DMMA update sweep
    CK(eks::launch_ca_pack(ctx->stream, t, 1, R1inv, pack));
    eks::SweepPtrs P{};
    P.q[0] = Z.loc;
    CK(eks::launch_sweep(ctx->stream, t, 1, 0, false, ctx->n, nullptr, Z.loc, P, pack, nullptr, nullptr, ctx->nblk));
  } else {
    CK(eks::launch_apply(ctx->stream, t, ctx->n, Z.loc, AZ, R1inv, nullptr, nullptr, nullptr, nullptr, nullptr,
                         nullptr, nullptr, 4, ctx->nblk));
  }
  return EKS_OK;
}

// Restructured update of one block (Alg 1/2 lines 14-17, reading R31): g = W_iᵀ r_{i−1},
// x += W_i g, r_i = r_{i−1} − AW_i g (and the per-CTA partials of ‖r_i‖²).
eks_status restructured_update(eks_ctx* ctx, int t, const double* W, const double* AW, const double* rin,
                               double* rout) {
  double* g = ctx->pre + (size_t)3 * t * t;
  {
    KScope k(ctx, EKS_K_COEF);
    account(ctx, EKS_K_COEF, 8.0 * ctx->n * (t + 1), 2.0 * ctx->n * t);
    CK(eks::launch_wtv(ctx->stream, ctx->n, t, W, rin, ctx->part, ctx->nblk));
  }
  {
    KScope k(ctx, EKS_K_REDUCE);
    CK(eks::launch_reduce(ctx->stream, ctx->part, ctx->nblk, t, t, g));
  }
  ST(allreduce(ctx, g, t));
  eks::CaPtrs P{};
  P.in[0] = W;
  P.out[0] = const_cast<double*>(AW);
  P.flag = ctx->flag;
  KScope k(ctx, EKS_K_APPLY);
  account(ctx, EKS_K_APPLY, 8.0 * ctx->n * (2.0 * t + 4.0), 4.0 * ctx->n * t);
  CK(eks::launch_ca_update(ctx->stream, ctx->n, t, 1, P, g, ctx->xv.loc, rin, rout, ctx->part, ctx->nblk));
  ctx->rho_nblk = ctx->nblk;
  return EKS_OK;
}

// One-synch CGS2 of Z against the window (DESIGN reading R36; the oracle's
// MODE_ONESYNCH): pass 1 as in cgs2() (C1 = (AQ)ᵀZ, fused from the previous block's R⁻¹ kernel for
// SRE-CG), Z1 = Z − Q C1 with C2 = (AQ)ᵀZ1 (NOT reduced yet); the SpMM runs on Z1: A·Z1, B1 = Z1ᵀAZ1,
// g1 = Z1ᵀr; ONE stacked allreduce of [C2 | B1 | g1]; then, since QᵀAQ = I and QᵀAZ1 = C2,
//   Z2ᵀAZ2 = B1 − C2ᵀC2,  Z2ᵀr = g1 − C2ᵀ(Qᵀr)  (k_onesynch_fix, into Bg),
//   Z2 = Z1 − Q C2,  A·Z2 = A·Z1 − (AQ) C2     (two update sweeps, in place).
// Leaves Z2 in Z (the block's slot), A·Z2 in AZ and [B | g] in Bg for the Cholesky and R⁻¹ kernels.
eks_status onesynch_block(eks_ctx* ctx, int t, const Window& w, const double* Zsrc, Block& Z, double* AZ,
                          bool with_update, int i) {
  const int nq = (int)w.Q.size();
  const size_t cb = (size_t)nq * t * t;
  const double* const* RQ = w.RQ.empty() ? nullptr : w.RQ.data();
  ST(ensure_C(ctx, cb));
  ST(ensure_os(ctx, cb + (size_t)t * t + t));
  if (!ctx->c1_ready) ST(tn_reduce(ctx, t, nq, w.AQ.data(), Zsrc, nullptr, ctx->C1));  // C1 = (AQ)ᵀZ (synch 1)
  ctx->c1_ready = false;
  double* C2 = ctx->os;
  double* Bg1 = ctx->os + cb;
  if (eks::sweep_supported(t) && eks::sweep_fused_supported(t, nq)) {
    ST(update_coef(ctx, t, nq, w.Q.data(), w.AQ.data(), ctx->C1, Zsrc, Z.loc, C2, false, RQ));
  } else {
    ST(ts_update(ctx, t, nq, w.Q.data(), ctx->C1, Zsrc, Z.loc, RQ));
    ST(tn_reduce(ctx, t, nq, w.AQ.data(), Z.loc, nullptr, C2, false));
  }
  ST(spmm_gram(ctx, Z, AZ, t, with_update ? ctx->r : nullptr, Bg1, nullptr, false));
  ST(allreduce(ctx, ctx->os, cb + (size_t)t * t + t));  // synch 2: [C2 | B1 | g1]
  // window blocks of this outer iteration (block i of it): the last i' = min(i, nq); their
  // α̃ = Wᵀr_{k−1} start at alpha + (i − i')·t
  const int ic = std::min(i, nq);
  {
    KScope k(ctx, EKS_K_CHOL);
    account(ctx, EKS_K_CHOL, 0.0, (double)nq * t * t * (t + 1) + 2.0 * ic * t * t);
    CK(eks::launch_onesynch_fix(ctx->stream, t, nq, nq - ic, C2, Bg1,
                                (with_update && ic > 0) ? ctx->alpha + (size_t)(i - ic) * t : nullptr,
                                ctx->Bg));
  }
  ST(ts_update(ctx, t, nq, w.Q.data(), C2, Z.loc, Z.loc, RQ));  // Z2 = Z1 − Q C2
  ST(ts_update(ctx, t, nq, w.AQ.data(), C2, AZ, AZ));           // A·Z2 = A·Z1 − (AQ) C2
  return EKS_OK;
}

// One A-orthonormalized block: Zsrc (or the split of r) → W_new, AW_new, R⁻¹, alpha_b.
eks_status make_block(eks_ctx* ctx, int t, int method, int ring, int nblocks, bool seed_from_r, const double* Zsrc,
                      Block* Wn, Block* AWn, int alpha_off, int gb, int mode) {
  Window w = window_for(ctx, t, method, nblocks, ring);
  if (seed_from_r) {
    double* dst = (w.Q.empty() && !ctx->use_prec) ? Wn->loc : ctx->Zs.loc;
    {
      KScope k(ctx, EKS_K_SPLIT);
      CK(eks::launch_split(ctx->stream, t, ctx->n, ctx->row_begin, ctx->n_global, ctx->r, dst));
    }
    account(ctx, EKS_K_SPLIT, 8.0 * ctx->n * (t + 1), 0.0);
    Zsrc = dst;
  }
  if (ctx->use_prec) {  // Alg 8-10: seed M⁻¹[T(r)] = L⁻ᵗ[T(L⁻¹r)], powers M⁻¹A·W
    ST(alloc_block(ctx, &ctx->Zp, t, false));
    ST(prec_apply(ctx, t, Zsrc, ctx->Zp.loc));
    Zsrc = ctx->Zp.loc;
  }
  const bool with_update = !(mode & 4);
  // lazy basis: this block's R⁻¹ lives in its ring slot (the later windows fold it into their
  // coefficients) and the R⁻¹ kernel leaves Z2 in the slot instead of W
  double* Rinv = ctx->lazy ? ctx->Rslot + (size_t)(nblocks % ring) * t * t : ctx->Rinv;
  const bool os = ctx->onesynch && !w.Q.empty() && !w.AQ.empty();
  if (os) {
    ST(onesynch_block(ctx, t, w, Zsrc, *Wn, AWn->loc, with_update, alpha_off / t));
  } else if (!w.Q.empty()) {
    ST(cgs2(ctx, t, w.Q, w.AQ, Zsrc, Wn->loc, &w.RQ));  // "A-orthonormalize W against Q"
  } else if (Zsrc != Wn->loc) {
    CK(cudaMemcpyAsync(Wn->loc, Zsrc, sizeof(double) * ctx->n * t, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (ctx->ortho == 1) ST(pre_euclid(ctx, t, *Wn, AWn->loc, gb));  // Pre-CholQR (reading R30)
  // "A-orthonormalize W": A-CholQR with one SpMM of Z2 (AW = (A Z2) R⁻¹)
  eks::CholArgs ch{};
  ch.R = ctx->Rm;
  ch.Rinv = Rinv;
  ch.alpha = with_update ? ctx->alpha + alpha_off : nullptr;
  ch.flag = ctx->flag;
  ch.gblock = gb;
  // t ≤ 32: the R⁻¹ kernel factors the Gram itself (every CTA, identical inputs on every rank);
  // otherwise the last CTA of the SpMM+Gram kernel or a separate Cholesky launch does it.
  if (!os) ST(spmm_gram(ctx, *Wn, AWn->loc, t, with_update ? ctx->r : nullptr, ctx->Bg, &ch));
  else ctx->chol_fused = false;  // B, g corrected by onesynch_block
  if (!ctx->chol_fused) {  // default: one-warp Cholesky launch (rsqrt pivots for t ≤ 32)
    KScope k(ctx, EKS_K_CHOL);
    CK(eks::launch_chol_fast(ctx->stream, t, ctx->Bg, with_update ? ctx->Bg + t * t : nullptr, ctx->Rm, Rinv,
                             with_update ? ctx->alpha + alpha_off : nullptr, ctx->flag, gb));
  }
  // SRE-CG: the next block's window is {W_prev, W_new} and its Z is AW_new, so the R⁻¹ kernel
  // that produces AW_new also accumulates the next CGS pass-1 coefficients C1 = [AW_prev, AW_new]ᵀAW_new.
  const int c1n = (ring && !ctx->use_prec && eks::apply_c1_supported(t, 2)) ? (nblocks == 0 ? 1 : 2) : 0;
  if (c1n) ST(ensure_C(ctx, (size_t)2 * t * t));
  if (ctx->part2_cap < (size_t)ctx->nblk * (2 * t * t + 2)) {
    dfree(ctx->part2);
    ctx->part2 = nullptr;
    ST(dalloc(ctx, &ctx->part2, (size_t)ctx->nblk * (2 * t * t + 2)));
    ctx->part2_cap = (size_t)ctx->nblk * (2 * t * t + 2);
  }
  const bool last = (mode & 2) && with_update;
  ctx->rho_fused = false;
  {
    KScope k(ctx, EKS_K_APPLY);
    // bytes: AZ2 read + AW written, Z2 read (eager or x update) + W written (eager), AW_prev (fused
    // next-C1), the x/r vectors; flops: the triangular products (1 lazy, 2 eager), next-C1, x/r
    const double nblk_io = (ctx->lazy ? 2.0 + (with_update ? 1.0 : 0.0) : 4.0) * t + (c1n == 2 ? t : 0) +
                           (with_update ? 4.0 : 0.0);
    account(ctx, EKS_K_APPLY, 8.0 * ctx->n * nblk_io,
            (ctx->lazy ? 1.0 : 2.0) * ctx->n * t * (t + 8.0) + 2.0 * c1n * ctx->n * t * t + 4.0 * ctx->n * t);
    if (eks::sweep_supported(t)) {
      // partials [C1 | ‖rnew‖²] reduced by the kernel's last CTAs into C1 and scal[1]
      const size_t cnt1 = (size_t)c1n * t * t;
      const eks::Tail tl = (cnt1 + (last ? 1 : 0)) ? tail(ctx, 3, ctx->C1, cnt1 + (last ? 1 : 0), ctx->scal + 1,
                                                           (int)cnt1)
                                                    : eks::Tail{};
      CK(eks::launch_apply_tc(ctx->stream, t, ctx->n, Wn->loc, AWn->loc, Rinv,
                              with_update ? ctx->alpha + alpha_off : nullptr, ctx->xv.loc, ctx->dx, ctx->r, ctx->rnew,
                              ctx->flag, mode | (ctx->lazy ? 8 : 0), ctx->nblk, c1n,
                              c1n == 2 ? ctx->AWpool[(nblocks - 1) % ring].loc : nullptr, ctx->part2, tl));
      ctx->rho_fused = last;
    } else {
      CK(eks::launch_apply(ctx->stream, t, ctx->n, Wn->loc, AWn->loc, ctx->Rinv,
                           with_update ? ctx->alpha + alpha_off : nullptr, ctx->xv.loc, ctx->dx, ctx->r, ctx->rnew,
                           ctx->part, ctx->flag, mode, ctx->nblk));
      ctx->rho_nblk = ctx->nblk;
    }
  }
  if (c1n) {
    ST(allreduce(ctx, ctx->C1, (size_t)c1n * t * t));
    ctx->c1_ready = true;
  }
  return EKS_OK;
}

// lazy basis: W = Z2·R⁻¹ of ring slot idx into out (device, n×t): 0 − Z2·(−R⁻¹) on the update sweep.
eks_status materialize_w(eks_ctx* ctx, int t, int idx, double* out) {
  double* pack = ctx->pre + (size_t)2 * t * t;  // [G | R1⁻¹ | pack | g] scratch of Pre-CholQR
  CK(eks::launch_ca_pack(ctx->stream, t, 1, ctx->Rslot + (size_t)idx * t * t, pack));
  eks::SweepPtrs P{};
  P.q[0] = ctx->Wpool[idx].loc;
  CK(eks::launch_sweep(ctx->stream, t, 1, 0, false, ctx->n, nullptr, out, P, pack, nullptr, nullptr, ctx->nblk));
  return EKS_OK;
}

bool lazy_env() {
  static const bool on = [] {  // EKS_LAZY_W=0: materialize W in every block (A/B measurements)
    const char* e = getenv("EKS_LAZY_W");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// A-CholQR of one block in place (the Alg 7 seed): B = Zᵀ(AZ), R, W = Z R⁻¹, AW = (AZ) R⁻¹.
eks_status acholqr_block(eks_ctx* ctx, int t, Block& Z, double* AZ, int gb) {
  ST(spmm_gram(ctx, Z, AZ, t, nullptr, ctx->Bg));
  {
    KScope k(ctx, EKS_K_CHOL);
    CK(eks::launch_chol_fast(ctx->stream, t, ctx->Bg, nullptr, ctx->Rm, ctx->Rinv, nullptr, ctx->flag, gb));
  }
  KScope k(ctx, EKS_K_APPLY);
  if (eks::sweep_supported(t))
    CK(eks::launch_apply_tc(ctx->stream, t, ctx->n, Z.loc, AZ, ctx->Rinv, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, 4, ctx->nblk, 0, nullptr, ctx->part2, eks::Tail{}));
  else
    CK(eks::launch_apply(ctx->stream, t, ctx->n, Z.loc, AZ, ctx->Rinv, nullptr, nullptr, nullptr, nullptr, nullptr,
                         nullptr, nullptr, 4, ctx->nblk));
  return EKS_OK;
}

// ---- Matrix-powers kernel with depth-d ghost zones (reading R37) ----
// The CA variants need V_i = A^i V_0, i = 1..d (d = s − 1), of a block whose rows are spread over the
// ranks.  Instead of one ghost-plane exchange per product, V_0's d boundary planes are exchanged ONCE
// and power i is computed on the slab plus (d − i) ghost planes of each neighbour (redundant work on
// the ghost planes), so that power i + 1 finds its ghost plane already there.  The ghost
// rows of A (their stencil values) are exchanged once per operator.  Every product is a launch of the
// plane-marching SpMM on a sub-range of planes, so each row is the same fma chain as in the global
// product (bitwise equal powers).
//
// Host plan: the slab has nz planes; db / da ghost planes exist below / above (d next to another rank,
// 0 at the boundary of the grid; in between only for a virtual slab whose distance to the boundary is
// < d).  Power i computes planes [zlo, zhi) (slab-relative, zlo ≤ 0) and reads one plane further
// where gb / ga = 1.
struct MpkStep { int zlo, zhi, gb, ga; };

void mpk_plan(int nz, int d, int db, int da, MpkStep* st) {
  for (int i = 1; i <= d; ++i) {
    const int below = std::min(db, d - i), above = std::min(da, d - i);
    st[i - 1] = MpkStep{-below, nz + above, db > below ? 1 : 0, da > above ? 1 : 0};
  }
}

// V[i] = A·V[i−1], i = 1..d, on the shrinking plane ranges of mpk_plan.  V[i] points at slab plane 0
// of a buffer holding planes [−db, nz + da); sv_ext = stencil values from plane −db on.
eks_status mpk_local(eks_ctx* ctx, int t, int d, int nz, int db, int da, const double* sv_ext, double* const* V) {
  std::vector<MpkStep> st(d);
  mpk_plan(nz, d, db, da, st.data());
  const int64_t plane = (int64_t)ctx->gplan.nx * ctx->gplan.ny;
  const int VS = (ctx->gplan.w + 1) & ~1;
  for (int i = 1; i <= d; ++i) {
    const MpkStep& m = st[i - 1];
    eks::GridPlan gp = ctx->gplan;
    gp.nz = m.zhi - m.zlo;
    gp.gb = m.gb;
    gp.ga = m.ga;
    gp.sv = sv_ext + (size_t)(m.zlo + db) * plane * VS;
    if (!eks::spmm_grid_fits(t, gp)) return fail(ctx, EKS_ERR_INVALID_ARG, "matrix powers: plane range does not fit");
    const int64_t rows = (int64_t)gp.nz * plane;
    account(ctx, EKS_K_SPMM, 8.0 * gp.w * rows + 16.0 * rows * t, 2.0 * gp.w * rows * t);
    KScope k(ctx, EKS_K_SPMM);
    CK(eks::launch_spmm_grid(ctx->stream, t, gp, V[i - 1] + m.zlo * plane * t, V[i] + m.zlo * plane * t, nullptr,
                             nullptr, ctx->nblk, eks::Tail{}, eks::CholArgs{}, false));
  }
  return EKS_OK;
}

// Can the CA powers of this solve run as the matrix-powers kernel?  Several ranks, the plane-marching
// SpMM on every rank, no preconditioner (M⁻¹ couples rows of a domain: no ghost rows for it), every
// slab at least d planes thick (the ghost planes then come from the two neighbour ranks only).  The
// answer must be the same on all ranks (the exchanges pair up): one MIN allreduce per (t, d), cached.
// EKS_MPK=0 keeps the one-exchange-per-product path; EKS_MPK=force also takes the matrix-powers code
// path on ONE rank (no neighbours: the same products through mpk_powers and the deep-ghost block
// layout — the integration test of the path on a one-GPU box).
eks_status mpk_usable(eks_ctx* ctx, int t, int d, bool& on) {
  on = false;
  static const int env_mode = [] {
    const char* e = getenv("EKS_MPK");
    return e && !strcmp(e, "0") ? 0 : (e && !strcmp(e, "force") ? 2 : 1);
  }();
  const bool env_on = env_mode != 0;
  if (d < 1) return EKS_OK;
  if (ctx->nranks == 1) {
    on = env_mode == 2 && !ctx->use_prec && eks::sweep_supported(t) && spmm_path_for(ctx, t) == 4;
    if (env_mode == 2 && !on)  // the test switch must not pass silently on the default path
      return fail(ctx, EKS_ERR_INVALID_ARG, "EKS_MPK=force: the matrix-powers path does not apply (t=%d)", t);
    return EKS_OK;
  }
  if (ctx->mpk_ok >= 0 && ctx->mpk_ok_t == t && ctx->mpk_ok_d == d) {
    on = ctx->mpk_ok == 1;
    return EKS_OK;
  }
  bool mine = env_on && !ctx->use_prec && eks::sweep_supported(t) && spmm_path_for(ctx, t) == 4;
  if (mine) {
    const int64_t plane = (int64_t)ctx->gplan.nx * ctx->gplan.ny;
    for (int q = 0; q < ctx->nranks; ++q) mine = mine && ctx->ranges[2 * q + 1] - ctx->ranges[2 * q] >= d * plane;
  }
  double v = mine ? 1.0 : 0.0;  // MIN over ranks through the fp64 scratch of the Cholesky flag's neighbours
  double* dv = nullptr;
  ST(dalloc(ctx, &dv, 1));
  CK(cudaMemcpyAsync(dv, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  NK(ncclAllReduce(dv, dv, 1, ncclDouble, ncclMin, ctx->comm, ctx->stream));
  CK(cudaMemcpyAsync(&v, dv, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  dfree(dv);
  ctx->mpk_ok = v == 1.0 ? 1 : 0;
  ctx->mpk_ok_t = t;
  ctx->mpk_ok_d = d;
  on = ctx->mpk_ok == 1;
  return EKS_OK;
}

// Send my d lowest planes to rank − 1 and my d highest to rank + 1; receive theirs into the ghost
// zones right before / after the slab (row width `w` doubles: t for a block, VS for stencil values).
eks_status mpk_exchange(eks_ctx* ctx, double* loc, int w, int d) {
  const int64_t plane = (int64_t)ctx->gplan.nx * ctx->gplan.ny;
  const size_t cnt = (size_t)d * plane * w;
  if (ctx->nranks == 1) return EKS_OK;  // no neighbours (EKS_MPK=force)
  KScope k(ctx, EKS_K_COMM);
  CK(cudaEventRecord(ctx->ev_ready, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_ready, 0));
  NK(ncclGroupStart());
  if (ctx->rank > 0) {
    NK(ncclSend(loc, cnt, ncclDouble, ctx->rank - 1, ctx->comm, ctx->comm_stream));
    NK(ncclRecv(loc - cnt, cnt, ncclDouble, ctx->rank - 1, ctx->comm, ctx->comm_stream));
  }
  if (ctx->rank + 1 < ctx->nranks) {
    NK(ncclSend(loc + (size_t)ctx->n * w - cnt, cnt, ncclDouble, ctx->rank + 1, ctx->comm, ctx->comm_stream));
    NK(ncclRecv(loc + (size_t)ctx->n * w, cnt, ncclDouble, ctx->rank + 1, ctx->comm, ctx->comm_stream));
  }
  NK(ncclGroupEnd());
  CK(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
  return EKS_OK;
}

// The d monomial powers V[1..d] of V[0] (deep-ghost blocks) on several ranks: stencil values of the
// ghost planes once per operator and depth, ONE exchange of V[0]'s boundary planes, d local products.
eks_status mpk_powers(eks_ctx* ctx, int t, int d, std::vector<Block>& V) {
  const int64_t plane = (int64_t)ctx->gplan.nx * ctx->gplan.ny;
  const int VS = (ctx->gplan.w + 1) & ~1;
  const int db = ctx->rank > 0 ? d : 0, da = ctx->rank + 1 < ctx->nranks ? d : 0;
  if (ctx->mpk_d != d) {
    dfree(ctx->mpk_sv);
    ctx->mpk_sv = nullptr;
    ctx->mpk_d = 0;
    ST(dalloc(ctx, &ctx->mpk_sv, (size_t)(db + da) * plane * VS + (size_t)ctx->n * VS));
    double* mid = ctx->mpk_sv + (size_t)db * plane * VS;
    CK(cudaMemcpyAsync(mid, ctx->gplan.sv, sizeof(double) * ctx->n * VS, cudaMemcpyDeviceToDevice, ctx->stream));
    ST(mpk_exchange(ctx, mid, VS, d));
    ctx->mpk_d = d;
  }
  ST(mpk_exchange(ctx, V[0].loc, t, d));
  std::vector<double*> L(d + 1);
  for (int i = 0; i <= d; ++i) L[i] = V[i].loc;
  return mpk_local(ctx, t, d, (int)(ctx->n / plane), db, da, ctx->mpk_sv, L.data());
}

// One outer iteration of CA SRE-CG / CA SRE-CG2 / CA MSDO-CG (base = the s-step method):
//   W = T(r_{k−1}) (k = 1, or every k for MSDO) or A·W_last;  Alg 7: A-orthonormalize W
//   against the window and itself;  V = [W, AW, …, A^{s−1}W];  CGS2 of every V_i
//   against the window (column-wise identical to CGS2 of the n×st block);  ONE A-CholQR of the
//   st columns: AV_i = A·V_i, B_ij = V_iᵀ AV_j (i ≤ j) and g = Vᵀr_{k−1}, R = chol(B), W = V R⁻¹,
//   AW = AV R⁻¹, α̃ = R⁻ᵀ g;  x += W α̃, r_k = r_{k−1} − AW α̃  (reading R28).
// Window: the last (s+1) blocks (CA SRE-CG, Alg 5 input m = (s+1)t) or all blocks.
eks_status ca_outer(eks_ctx* ctx, int t, int s, int base, int arnoldi, int k, int& nblocks, int ring) {
  const int st = s * t;
  ctx->rho_fused = false;  // ‖r_k‖² comes from k_ca_update's per-CTA partials
  ctx->c1_ready = false;
  bool mpk = false;
  ST(mpk_usable(ctx, t, s - 1, mpk));
  const int deep = mpk ? s - 1 : 0;
  if (ctx->ca_cap != st || (int)ctx->Vca.size() != s || ctx->ca_deep != deep) {
    for (auto& b : ctx->Vca) dfree(b.alloc ? b.alloc : b.base);
    for (auto& b : ctx->AVca) dfree(b.base);
    for (double** p : {&ctx->Bca, &ctx->gca, &ctx->Rca, &ctx->Rinvca, &ctx->alphaca, &ctx->Btmp, &ctx->cawork}) {
      dfree(*p);
      *p = nullptr;
    }
    ctx->Vca.assign(s, Block{});
    ctx->AVca.assign(s, Block{});
    for (int i = 0; i < s; ++i) {
      if (deep) {  // `deep` ghost planes next to each neighbour rank (≥ the one plane of the halo layout)
        Block& B = ctx->Vca[i];
        const int64_t plane = (int64_t)ctx->gplan.nx * ctx->gplan.ny;
        const int64_t rb = ctx->rank > 0 ? deep * plane : 0, ra = ctx->rank + 1 < ctx->nranks ? deep * plane : 0;
        ST(dalloc(ctx, &B.alloc, (size_t)(rb + ctx->n + ra) * t));
        B.loc = B.alloc + rb * t;
        B.base = B.loc - ctx->halo_before * t;
      } else {
        ST(alloc_block(ctx, &ctx->Vca[i], t, true));
      }
      ST(alloc_block(ctx, &ctx->AVca[i], t, false));
    }
    ctx->ca_deep = deep;
    ST(dalloc(ctx, &ctx->Bca, (size_t)st * st));
    ST(dalloc(ctx, &ctx->gca, (size_t)st));
    ST(dalloc(ctx, &ctx->Rca, (size_t)st * st));
    ST(dalloc(ctx, &ctx->Rinvca, (size_t)st * st));
    ST(dalloc(ctx, &ctx->alphaca, (size_t)st));
    ST(dalloc(ctx, &ctx->Btmp, (size_t)s * (s + 1) / 2 * t * t + (size_t)s * t));
    if (eks::chol_dyn_work(st)) ST(dalloc(ctx, &ctx->cawork, eks::chol_dyn_work(st)));
    ctx->ca_cap = st;
  }
  std::vector<const double*> Q, AQ;
  const int first = base == EKS_SRE_CG ? std::max(0, nblocks - (s + 1)) : 0;
  for (int j = first; j < nblocks; ++j) {
    const int idx = ring ? j % ring : j;
    Q.push_back(ctx->Wpool[idx].loc);
    AQ.push_back(ctx->AWpool[idx].loc);
  }
  std::vector<Block>& V = ctx->Vca;
  std::vector<Block>& AV = ctx->AVca;
  // seed
  if (base == EKS_MSDO_CG || k == 1) {
    {
      KScope kk(ctx, EKS_K_SPLIT);
      CK(eks::launch_split(ctx->stream, t, ctx->n, ctx->row_begin, ctx->n_global, ctx->r, V[0].loc));
    }
    if (ctx->use_prec) ST(prec_apply(ctx, t, V[0].loc, V[0].loc));  // L⁻ᵗ[T(L⁻¹r)] = M⁻¹[T(r)]
  } else {
    const int idx = ring ? (nblocks - 1) % ring : nblocks - 1;
    ST(spmm(ctx, ctx->Wpool[idx], V[0].loc, t));
    if (ctx->use_prec) ST(prec_apply(ctx, t, V[0].loc, V[0].loc));  // M⁻¹A W_{j−1}
  }
  if (arnoldi == 7) {  // Alg 7 lines 1-4
    if (!Q.empty()) ST(cgs2(ctx, t, Q, AQ, V[0].loc, V[0].loc));
    ST(acholqr_block(ctx, t, V[0], AV[0].loc, nblocks));
  }
  if (mpk) {  // matrix-powers kernel: one exchange of s − 1 ghost planes, then local products
    ST(mpk_powers(ctx, t, s - 1, V));
  } else {
    for (int i = 1; i < s; ++i) {  // monomial powers (M⁻¹A with the preconditioner)
      ST(spmm(ctx, V[i - 1], V[i].loc, t));
      if (ctx->use_prec) ST(prec_apply(ctx, t, V[i].loc, V[i].loc));
    }
  }
  if (!Q.empty()) ST(cgs2_stacked(ctx, t, Q, AQ, V, AV));  // AV serves as the pass-1 scratch
  // Gram B (st×st, upper blocks) and g = Vᵀ r_{k−1}: block column j = [V_0..V_{j−1}]ᵀAV_j, then
  // [V_jᵀAV_j | V_jᵀr] from the fused SpMM+Gram kernel that forms AV_j, into Btmp (column j at
  // offset (j(j+1)/2)·t·t + j·t); ONE allreduce for all of them.
  std::vector<const double*> L(s);
  for (int i = 0; i < s; ++i) L[i] = V[i].loc;
  auto off = [&](int j) { return (size_t)j * (j + 1) / 2 * t * t + (size_t)j * t; };
  for (int j = 0; j < s; ++j) {
    ST(spmm_gram(ctx, V[j], AV[j].loc, t, ctx->r, ctx->Btmp + off(j) + (size_t)j * t * t, nullptr, false));
    if (j > 0) ST(tn_reduce(ctx, t, j, L.data(), AV[j].loc, nullptr, ctx->Btmp + off(j), false));
  }
  ST(allreduce(ctx, ctx->Btmp, off(s)));
  for (int j = 0; j < s; ++j) {
    for (int i = 0; i <= j; ++i)
      CK(cudaMemcpy2DAsync(ctx->Bca + (size_t)i * t * st + (size_t)j * t, sizeof(double) * st,
                           ctx->Btmp + off(j) + (size_t)i * t * t, sizeof(double) * t, sizeof(double) * t, t,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->gca + (size_t)j * t, ctx->Btmp + off(j) + (size_t)(j + 1) * t * t, sizeof(double) * t,
                       cudaMemcpyDeviceToDevice, ctx->stream));
  }
  {
    KScope kk(ctx, EKS_K_CHOL);
    if (st <= 32 && (st & (st - 1)) == 0)  // one-warp register Cholesky (upper triangle only)
      CK(eks::launch_chol_fast(ctx->stream, st, ctx->Bca, ctx->gca, ctx->Rca, ctx->Rinvca, ctx->alphaca, ctx->flag,
                               nblocks));
    else
      CK(eks::launch_chol_dyn(ctx->stream, st, ctx->Bca, ctx->gca, ctx->Rca, ctx->Rinvca, ctx->alphaca, ctx->flag,
                              nblocks, ctx->cawork));
  }
  // W = V R⁻¹, AW = AV R⁻¹ into the new slots
  eks::CaPtrs Pw{}, Pa{}, Pu{};
  for (int j = 0; j < s; ++j) {
    Block *Wn = nullptr, *AWn = nullptr;
    ST(slot(ctx, t, ring ? (nblocks + j) % ring : nblocks + j, &Wn, &AWn));
    Pw.in[j] = V[j].loc;
    Pw.out[j] = Wn->loc;
    Pa.in[j] = AV[j].loc;
    Pa.out[j] = AWn->loc;
    Pu.in[j] = Wn->loc;
    Pu.out[j] = AWn->loc;
  }
  Pw.flag = Pa.flag = Pu.flag = ctx->flag;
  {
    KScope kk(ctx, EKS_K_APPLY);
    if (eks::sweep_supported(t)) {
      // W_j = 0 − Σ_{i≤j} V_i·(−R⁻¹_ij) on the DMMA update sweep (−R⁻¹ column blocks packed),
      // in chunks of at most sweep_max_blocks(t) input blocks accumulated into W_j
      CK(eks::launch_ca_pack(ctx->stream, t, s, ctx->Rinvca, ctx->Btmp));
      const int maxb = eks::sweep_max_blocks(t);
      for (int j = 0; j < s; ++j) {
        const double* C = ctx->Btmp + (size_t)j * (j + 1) / 2 * t * t;
        for (int c0 = 0; c0 <= j; c0 += maxb) {
          const int kb = std::min(maxb, j + 1 - c0);
          eks::SweepPtrs Sw{}, Sa{};
          for (int i = 0; i < kb; ++i) {
            Sw.q[i] = Pw.in[c0 + i];
            Sa.q[i] = Pa.in[c0 + i];
          }
          const double* Ck = C + (size_t)c0 * t * t;
          CK(eks::launch_sweep(ctx->stream, t, kb, 0, false, ctx->n, c0 ? Pw.out[j] : nullptr, Pw.out[j], Sw, Ck,
                               nullptr, nullptr, ctx->nblk));
          CK(eks::launch_sweep(ctx->stream, t, kb, 0, false, ctx->n, c0 ? Pa.out[j] : nullptr, Pa.out[j], Sa, Ck,
                               nullptr, nullptr, ctx->nblk));
        }
      }
    } else {
      CK(eks::launch_ca_combine(ctx->stream, ctx->n, t, s, Pw, ctx->Rinvca, ctx->sms, false));
      CK(eks::launch_ca_combine(ctx->stream, ctx->n, t, s, Pa, ctx->Rinvca, ctx->sms, false));
    }
    CK(eks::launch_ca_update(ctx->stream, ctx->n, t, s, Pu, ctx->alphaca, ctx->xv.loc, ctx->r, ctx->rnew, ctx->part,
                             ctx->nblk));
    ctx->rho_nblk = ctx->nblk;
  }
  account(ctx, EKS_K_APPLY, 8.0 * ctx->n * (4.0 * st + 3.0), 2.0 * ctx->n * st * (st + 2));
  nblocks += s;
  return EKS_OK;
}

// r = b − A x (x in ctx->xv), scal[slot] = ||r||² ; if r_out == nullptr only the norm
eks_status residual(eks_ctx* ctx, double* r_out, double* slotp) {
  ST(spmm(ctx, ctx->xv, ctx->tmpv.loc, 1));
  {
    KScope k(ctx, EKS_K_OTHER);
    CK(eks::launch_residual(ctx->stream, ctx->n, ctx->b, ctx->tmpv.loc, r_out, ctx->part, ctx->nblk));
    ctx->rho_nblk = ctx->nblk;
  }
  return reduce_scalar(ctx, slotp);
}

// ---------------------------------------------------------------- halo plan (host only)
// Rank `rank` owns rows [ranges[2r], ranges[2r+1]).  For every other rank q the
// ghost rows it needs are the contiguous range [lo_q, hi_q) spanning all its
// off-slab column indices owned by q (exact for banded/stencil matrices, a
// superset otherwise).  Extended layout: ghost ranges of lower ranks, local
// rows, ghost ranges of higher ranks — so the SpMM reads one array.  The
// interior run is the longest run of rows with only local columns: it is
// multiplied while the halo is in flight.
struct HaloPlan {
  int64_t halo_before = 0, halo_after = 0, int_lo = 0, int_hi = 0;
  std::vector<Recv> recvs;
  std::vector<int64_t> need;  // 2*nranks: [lo,hi) received from each rank (0,0 if none)
  std::vector<int32_t> ecol;  // columns remapped to the extended layout
};

void plan_halo(int rank, int nranks, const int64_t* ranges, int64_t n, const int64_t* rp, const int32_t* col,
               HaloPlan& P) {
  const int64_t row_begin = ranges[2 * rank], row_end = ranges[2 * rank + 1];
  const int64_t nnz = rp[n];
  if (nranks == 1) {  // no ghosts: the extended columns are the columns (P.ecol left empty), all rows interior
    P = HaloPlan{};
    P.need.assign(2, 0);
    P.int_hi = n;
    return;
  }
  auto owner = [&](int64_t c) {
    int q = 0;
    while (q < nranks && !(c >= ranges[2 * q] && c < ranges[2 * q + 1])) ++q;
    return q;
  };
  std::vector<int64_t> glo(nranks, INT64_MAX), ghi(nranks, INT64_MIN);
  for (int64_t p = 0; p < nnz; ++p) {
    const int64_t c = col[p];
    if (c < row_begin || c >= row_end) {
      const int q = owner(c);
      glo[q] = std::min(glo[q], c);
      ghi[q] = std::max(ghi[q], c + 1);
    }
  }
  P.recvs.clear();
  P.need.assign(2 * nranks, 0);
  std::vector<int64_t> off(nranks, 0);
  int64_t ext = 0;
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      off[q] = ext;
      ext += n;
      continue;
    }
    if (glo[q] < ghi[q]) {
      off[q] = ext;
      P.recvs.push_back({q, glo[q], ghi[q], ext});
      P.need[2 * q] = glo[q];
      P.need[2 * q + 1] = ghi[q];
      ext += ghi[q] - glo[q];
    }
  }
  P.halo_before = off[rank];
  P.halo_after = ext - off[rank] - n;
  P.ecol.assign(nnz, 0);
  std::vector<char> interior(n, 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = col[p];
      if (c >= row_begin && c < row_end) {
        P.ecol[p] = (int32_t)(P.halo_before + (c - row_begin));
      } else {
        const int q = owner(c);
        P.ecol[p] = (int32_t)(off[q] + (c - glo[q]));
        interior[i] = 0;
      }
    }
  int64_t best_lo = 0, best_len = 0, cur = 0;
  for (int64_t i = 0; i <= n; ++i) {
    if (i < n && interior[i]) {
      ++cur;
      continue;
    }
    if (cur > best_len) {
      best_len = cur;
      best_lo = i - cur;
    }
    cur = 0;
  }
  P.int_lo = best_lo;
  P.int_hi = best_lo + best_len;
}

// Segment plan for the TMA-staged SpMM (eks_sweep.cuh SegPlan): per plan tile of kSegPT rows,
// the sorted distinct X rows its entries use, merged into runs (gaps of ≤ 2 rows are copied
// too); every entry's column becomes a row of the concatenated runs.  Not built (the ELL
// gather kernel runs instead) when a tile needs more than kSegMax runs.
eks_status build_seg_plan(eks_ctx* ctx, int64_t n, const std::vector<int64_t>& rp, const std::vector<int32_t>& ecol,
                          const std::vector<double>& val, int64_t halo_before, int w) {
  constexpr int PT = eks::kSegPT, SM = eks::kSegMax, GAP = 2;
  const int64_t ntp = (n + PT - 1) / PT;
  std::vector<int32_t> seg((size_t)ntp * SM * 2, 0), rows((size_t)ntp, 0), own((size_t)ntp, 0);
  const int VS = (w + 1) & ~1;  // value slots per row (eks::seg_vs)
  std::vector<uint16_t> lidx((size_t)ntp * PT * 8, 0);
  std::vector<double> sv((size_t)ntp * PT * VS, 0.0);
  std::vector<int32_t> cols;
  int cap = 0;
  for (int64_t p = 0; p < ntp; ++p) {
    cols.clear();
    const int64_t i0 = p * PT, i1 = std::min(n, i0 + PT);
    for (int64_t i = i0; i < i1; ++i) {
      cols.push_back((int32_t)(halo_before + i));
      for (int64_t q = rp[i]; q < rp[i + 1]; ++q) cols.push_back(ecol[q]);
    }
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    int32_t rs[SM], rl[SM], ro[SM];
    int nr = 0, tot = 0;
    for (int32_t c : cols) {
      if (nr > 0 && c <= rs[nr - 1] + rl[nr - 1] + GAP) {
        rl[nr - 1] = c - rs[nr - 1] + 1;
        continue;
      }
      if (nr == SM) return EKS_OK;  // too irregular: keep the gather kernels
      rs[nr] = c;
      rl[nr] = 1;
      ++nr;
    }
    for (int q = 0; q < nr; ++q) {
      ro[q] = tot;
      tot += rl[q];
      seg[((size_t)p * SM + q) * 2] = rs[q];
      seg[((size_t)p * SM + q) * 2 + 1] = rl[q];
    }
    if (tot > 65535) return EKS_OK;
    cap = std::max(cap, tot);
    rows[p] = tot;
    auto bufrow = [&](int32_t c) {
      int q = 0;
      while (q + 1 < nr && c >= rs[q + 1]) ++q;
      return ro[q] + (c - rs[q]);
    };
    own[p] = bufrow((int32_t)(halo_before + i0));
    for (int rr = 0; rr < PT; ++rr)
      for (int k = 0; k < 8; ++k) {  // row-major: 8 local indices (16 bytes) and VS values per row
        const int64_t i = i0 + rr, e = ((size_t)p * PT + rr) * 8 + k, ev = ((size_t)p * PT + rr) * VS + k;
        if (i < n && k < rp[i + 1] - rp[i]) {
          lidx[e] = (uint16_t)bufrow(ecol[rp[i] + k]);
          sv[ev] = val[rp[i] + k];
        } else {
          lidx[e] = (uint16_t)(i < n ? bufrow((int32_t)(halo_before + i)) : 0);
        }
      }
  }
  auto up = [&](void** d, const void* h, size_t bytes) -> eks_status {
    CK(cudaMalloc(d, bytes + 16));
    CK(cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice));
    return EKS_OK;
  };
  ST(up((void**)&ctx->d_seg, seg.data(), sizeof(int32_t) * seg.size()));
  ST(up((void**)&ctx->d_segrows, rows.data(), sizeof(int32_t) * rows.size()));
  ST(up((void**)&ctx->d_segown, own.data(), sizeof(int32_t) * own.size()));
  ST(up((void**)&ctx->d_lidx, lidx.data(), sizeof(uint16_t) * lidx.size()));
  ST(up((void**)&ctx->d_sval, sv.data(), sizeof(double) * sv.size()));
  ctx->seg.seg = ctx->d_seg;
  ctx->seg.rows = ctx->d_segrows;
  ctx->seg.own = ctx->d_segown;
  ctx->seg.lidx = ctx->d_lidx;
  ctx->seg.val = ctx->d_sval;
  ctx->seg.cap = cap;
  ctx->seg_ok = true;
  return EKS_OK;
}

// Host loops over the rows of a (possibly 56M-row) slab on all host threads: f(lo, hi) per chunk.
template <typename F>
void parallel_rows(int64_t n, F&& f) {
  const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), (int)(n / 65536) + 1));
  if (nt == 1) {
    f((int64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int k = 0; k < nt; ++k) th.emplace_back([&, k] { f(n * k / nt, n * (k + 1) / nt); });
  for (auto& x : th) x.join();
}

// Stencil structure for the plane-marching SpMM (eks_grid.cu): the distinct positive column offsets
// must be {1, b} (2D: nx = b, planes are x-lines) or {1, b, c} with b | c (3D: nx = b, ny = c/b),
// mirrored by the negative ones, and no ±1 (±nx) entry may cross an x-line (y-plane) boundary.
// Several ranks: the slab [row_begin, row_begin + n) must be whole planes and the ghost rows of the
// extended layout exactly the neighbouring planes (halo_before/after ∈ {0, plane}); columns are GLOBAL.
// Values are stored per row in ascending offset order, 0 in absent slots (VS = (w+1)&~1 per row).
// geom = {nx, ny, nz, w, gb, ga}; false (nothing built, the ELL/CSR kernels run) otherwise.
// Detection only: geom = {nx, ny, nz, w, gb, ga} and the positive offsets b = nx, c = nx·ny (2D: c = 0)
// from the offsets of the first rows; the per-entry check comes with the fill (host or device).
bool grid_detect(int64_t n, const int64_t* rp, const int32_t* col, int64_t row_begin, int64_t halo_before,
                 int64_t halo_after, int64_t geom[6], int64_t& b, int64_t& c) {
  int64_t pos[3] = {0, 0, 0};
  int np = 0;
  // the offsets from the first rows (a stencil shows all of them within a few planes); an offset
  // first appearing later is caught by the full check below (not a stencil: nothing built)
  const int64_t scan = std::min<int64_t>(n, (int64_t)1 << 22);
  for (int64_t i = 0; i < scan && np <= 3; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t o = (int64_t)col[p] - (row_begin + i);
      if (o <= 0) continue;
      int k = 0;
      while (k < np && pos[k] != o) ++k;
      if (k == np) {
        if (np == 3) return false;
        pos[np++] = o;
      }
    }
  for (int a2 = 1; a2 < np; ++a2)  // np ≤ 3: insertion sort (std::sort trips -Warray-bounds here)
    for (int b2 = a2; b2 > 0 && pos[b2 - 1] > pos[b2]; --b2) std::swap(pos[b2 - 1], pos[b2]);
  if (np < 2 || pos[0] != 1) return false;
  b = pos[1];
  c = np == 3 ? pos[2] : 0;
  int64_t nx = b, ny = 1, plane = b;
  if (np == 3) {
    if (c % b) return false;
    ny = c / b;
    plane = c;
  }
  if (n % plane || row_begin % plane) return false;
  if ((halo_before != 0 && halo_before != plane) || (halo_after != 0 && halo_after != plane)) return false;
  const int64_t nz = n / plane;
  if (nx >= INT32_MAX || ny >= INT32_MAX || nz >= INT32_MAX) return false;
  geom[0] = nx;
  geom[1] = ny;
  geom[2] = nz;
  geom[3] = np == 3 ? 7 : 5;
  geom[4] = halo_before ? 1 : 0;
  geom[5] = halo_after ? 1 : 0;
  return true;
}

bool grid_plan_host(int64_t n, const int64_t* rp, const int32_t* col, const double* val, int64_t row_begin,
                    int64_t halo_before, int64_t halo_after, int64_t geom[6], std::vector<double>& sv) {
  int64_t b = 0, c = 0;
  if (!grid_detect(n, rp, col, row_begin, halo_before, halo_after, geom, b, c)) return false;
  const int64_t nx = geom[0], ny = geom[1];
  const int w = (int)geom[3], VS = (w + 1) & ~1;
  const int64_t offs7[7] = {-c, -b, -1, 0, 1, b, c};
  const int64_t offs5[5] = {-b, -1, 0, 1, b};
  const int64_t* offs = w == 7 ? offs7 : offs5;
  sv.assign((size_t)n * VS, 0.0);
  std::atomic<bool> ok{true};
  parallel_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi && ok.load(std::memory_order_relaxed); ++i) {
      const int64_t x = (row_begin + i) % nx, y = ((row_begin + i) / nx) % ny;
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int64_t o = (int64_t)col[p] - (row_begin + i);
        int k = -1;
        for (int q = 0; q < w; ++q)
          if (offs[q] == o) k = q;
        const bool bad = k < 0 || (o == 1 && x + 1 >= nx) || (o == -1 && x == 0) ||
                         (w == 7 && ((o == b && y + 1 >= ny) || (o == -b && y == 0)));
        if (bad) {
          ok = false;
          return;
        }
        sv[(size_t)i * VS + k] = val[p];
      }
    }
  });
  return ok.load();
}

eks_status build_grid_plan(eks_ctx* ctx, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                           int64_t row_begin, int64_t halo_before, int64_t halo_after) {
  (void)val;
  int64_t g[6], b = 0, c = 0;
  if (!grid_detect(n, rp, col, row_begin, halo_before, halo_after, g, b, c)) return EKS_OK;
  // the stencil values are scattered from the uploaded CSR by a device kernel (columns in the extended
  // layout: offset = ecol − halo_before − i); an entry outside the stencil leaves the plan unbuilt
  const int VS = ((int)g[3] + 1) & ~1;
  CK(cudaMalloc((void**)&ctx->d_sv, sizeof(double) * (size_t)n * VS));
  int* d_bad = nullptr;
  CK(cudaMalloc((void**)&d_bad, sizeof(int)));
  CK(cudaMemset(d_bad, 0, sizeof(int)));
  CK(eks::launch_grid_sv(ctx->stream, n, ctx->d_rp, ctx->d_col, ctx->d_val, row_begin, halo_before, g[0], g[1], b, c,
                         (int)g[3], ctx->d_sv, d_bad, ctx->sms));
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_bad);
  if (bad) {
    dfree(ctx->d_sv);
    ctx->d_sv = nullptr;
    return EKS_OK;
  }
  ctx->gplan.nx = (int)g[0];
  ctx->gplan.ny = (int)g[1];
  ctx->gplan.nz = (int)g[2];
  ctx->gplan.w = (int)g[3];
  ctx->gplan.gb = (int)g[4];
  ctx->gplan.ga = (int)g[5];
  ctx->gplan.sv = ctx->d_sv;
  ctx->grid_ok = true;
  return EKS_OK;
}

// Timing events of one solve, destroyed on every exit path.
struct EventPair {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t create() {
    cudaError_t e = cudaEventCreate(&e0);
    return e == cudaSuccess ? cudaEventCreate(&e1) : e;
  }
  ~EventPair() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

// A stream capture that is ended on every exit path: an error inside the captured region must not
// leave the (possibly caller-owned) stream in an invalidated capture state.
struct CaptureGuard {
  cudaStream_t st;
  bool open = false;
  explicit CaptureGuard(cudaStream_t s) : st(s) {}
  cudaError_t begin() {
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    open = e == cudaSuccess;
    return e;
  }
  cudaError_t end(cudaGraph_t* g) {
    open = false;
    return cudaStreamEndCapture(st, g);
  }
  ~CaptureGuard() {
    if (!open) return;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(st, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
};

// Everything a steady-state s-step SRE-CG outer iteration allocates lazily (ring slots, C1/C2 of the
// 2-block window, per-CTA partials of every sweep, the fused next-C1 partials), allocated up front
// so that a CUDA-graph capture never meets a cudaMalloc/cudaFree.
eks_status prealloc_steady(eks_ctx* ctx, int t, int ring) {
  for (int idx = 0; idx < ring; ++idx) {
    Block *W = nullptr, *AW = nullptr;
    ST(slot(ctx, t, idx, &W, &AW));
  }
  ST(ensure_C(ctx, (size_t)2 * t * t));
  if (ctx->onesynch) ST(ensure_os(ctx, (size_t)3 * t * t + t));
  size_t stride = std::max(eks::tn_partials_stride(t, 2, false), eks::tn_partials_stride(t, 1, true));
  if (eks::sweep_supported(t))
    stride = std::max({stride, eks::sweep_part_stride(t, 2, false), eks::sweep_part_stride(t, 1, true)});
  ST(ensure_part(ctx, stride * ctx->nblk));
  if (ctx->part2_cap < (size_t)ctx->nblk * (2 * t * t + 2)) {
    dfree(ctx->part2);
    ctx->part2 = nullptr;
    ST(dalloc(ctx, &ctx->part2, (size_t)ctx->nblk * (2 * t * t + 2)));
    ctx->part2_cap = (size_t)ctx->nblk * (2 * t * t + 2);
  }
  return EKS_OK;
}

void begin_run(eks_ctx* ctx, const eks_options* opt) {
  ctx->prof_on = opt && opt->profile;
  ctx->prof = eks_profile{};
  ctx->launches = 0;
  ctx->model_bytes = ctx->model_flops = 0.0;
  ctx->c1_ready = false;
  ctx->aq_off = false;  // set per solve (full-basis methods)
  ctx->lazy = false;    // set per solve / sweep (s-step SRE-CG, t ≥ 8)
  ctx->onesynch = opt && opt->onesynch;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

eks_status eks_get_unique_id(unsigned char id[128]) {
  if (!id) return EKS_ERR_INVALID_ARG;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return EKS_ERR_NCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return EKS_OK;
}

eks_status eks_create(eks_ctx** out, const eks_dist* dist) {
  if (!out) return EKS_ERR_INVALID_ARG;
  *out = nullptr;
  eks_ctx* ctx = new (std::nothrow) eks_ctx();
  if (!ctx) return EKS_ERR_OOM;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    delete ctx;
    return EKS_ERR_CUDA;  // no CPU fallback
  }
  if (dist) {
    if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks || dist->device < 0 || dist->device >= ndev) {
      delete ctx;
      return EKS_ERR_INVALID_ARG;
    }
    ctx->rank = dist->rank;
    ctx->nranks = dist->nranks;
    ctx->device = dist->device;
  } else {
    cudaGetDevice(&ctx->device);
  }
  eks_status st = EKS_OK;
  do {
    if (cudaSetDevice(ctx->device) != cudaSuccess) { st = EKS_ERR_CUDA; break; }
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
    ctx->nblk = eks::sweep_ctas(ctx->sms);
    if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess) { st = EKS_ERR_CUDA; break; }
    ctx->stream = ctx->own;
    if (cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking) != cudaSuccess) { st = EKS_ERR_CUDA; break; }
    cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming);
    if (cudaMallocHost((void**)&ctx->h_scal, 16 * sizeof(double)) != cudaSuccess) { st = EKS_ERR_CUDA; break; }
    if (cudaMallocHost((void**)&ctx->h_flag, 4 * sizeof(int)) != cudaSuccess) { st = EKS_ERR_CUDA; break; }
    ctx->h_flag[0] = INT_MAX;
    if (const char* e = getenv("EKS_CHOL")) ctx->chol_mode = atoi(e);
    if (const char* e = getenv("EKS_SPMM_PATH"))
      ctx->spmm_path = !strcmp(e, "ell") ? 1 : (!strcmp(e, "csr") ? 2 : (!strcmp(e, "seg") ? 3 : (!strcmp(e, "grid") ? 4 : 0)));
    if (ctx->nranks > 1) {
      ncclUniqueId u;
      memcpy(&u, dist->nccl_id, 128);
      if (ncclCommInitRank(&ctx->comm, ctx->nranks, u, ctx->rank) != ncclSuccess) { st = EKS_ERR_NCCL; break; }
    }
  } while (0);
  if (st != EKS_OK) {
    eks_destroy(ctx);
    return st;
  }
  *out = ctx;
  return EKS_OK;
}

eks_status eks_set_stream(eks_ctx* ctx, void* stream) {
  if (!ctx) return EKS_ERR_INVALID_ARG;
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own;
  return EKS_OK;
}

eks_status eks_setup_csr(eks_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t row_end, const int64_t* row_ptr,
                         const int32_t* col_idx, const double* vals, eks_mem where) {
  if (!ctx) return EKS_ERR_INVALID_ARG;
  if (!row_ptr || !col_idx || !vals) return fail(ctx, EKS_ERR_INVALID_ARG, "NULL matrix pointer");
  ctx->prec_nd = 0;  // a new matrix invalidates the preconditioner (its buffers go on the next setup/destroy)
  if (n_global <= 0 || row_begin < 0 || row_end <= row_begin || row_end > n_global)
    return fail(ctx, EKS_ERR_INVALID_ARG, "bad row range [%lld,%lld) of n=%lld", (long long)row_begin,
                (long long)row_end, (long long)n_global);
  if (n_global >= INT_MAX) return fail(ctx, EKS_ERR_INVALID_ARG, "n_global must be < 2^31 (int32 columns)");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = row_end - row_begin;
  // host views of the caller's arrays (EKS_MEM_HOST: used in place, no copy; device: copied down)
  std::vector<int64_t> rpv;
  std::vector<int32_t> colv;
  std::vector<double> valv;
  const int64_t* RP = row_ptr;
  if (where != EKS_MEM_HOST) {
    rpv.resize(n + 1);
    CK(cudaMemcpy(rpv.data(), row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    RP = rpv.data();
  }
  if (RP[0] != 0) return fail(ctx, EKS_ERR_BAD_MATRIX, "row_ptr[0] != 0");
  {
    std::atomic<int64_t> bad{INT64_MAX};
    parallel_rows(n, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i)
        if (RP[i + 1] < RP[i]) {
          int64_t cur = bad.load();
          while (i < cur && !bad.compare_exchange_weak(cur, i)) {
          }
          break;
        }
    });
    if (bad.load() != INT64_MAX)
      return fail(ctx, EKS_ERR_BAD_MATRIX, "row_ptr not monotone at row %lld", (long long)bad.load());
  }
  const int64_t nnz = RP[n];
  if (nnz >= INT_MAX) return fail(ctx, EKS_ERR_INVALID_ARG, "local nnz must be < 2^31");
  const int32_t* COL = col_idx;
  const double* VAL = vals;
  if (where != EKS_MEM_HOST) {
    colv.resize(nnz);
    valv.resize(nnz);
    CK(cudaMemcpy(colv.data(), col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(valv.data(), vals, sizeof(double) * nnz, cudaMemcpyDeviceToHost));
    COL = colv.data();
    VAL = valv.data();
  }
  // One rank, host arrays: the columns and values go to the device as they are, so their copies are
  // started now and run under the host-side validation (end-to-end setup time; on a validation error
  // the new buffers are dropped and the context keeps its previous matrix).
  int* early_col = nullptr;
  double* early_val = nullptr;
  struct EarlyGuard {  // any error return before the hand-over frees the early copies
    eks_ctx* c;
    int** col;
    double** val;
    ~EarlyGuard() {
      if (*col || *val) {
        cudaStreamSynchronize(c->stream);
        dfree(*col);
        dfree(*val);
      }
    }
  } early_guard{ctx, &early_col, &early_val};
  if (where == EKS_MEM_HOST && ctx->nranks == 1 && nnz > 0) {
    if (cudaMalloc((void**)&early_col, sizeof(int) * nnz + 16) != cudaSuccess ||
        cudaMalloc((void**)&early_val, sizeof(double) * nnz + 16) != cudaSuccess) {
      cudaGetLastError();
      dfree(early_col);
      dfree(early_val);
      early_col = nullptr;
      early_val = nullptr;  // not enough room next to the previous matrix: the plain order below
    } else {
      CK(cudaMemcpyAsync(early_col, COL, sizeof(int) * nnz, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(early_val, VAL, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  // validation (SPEC S:30-33 invariants): sorted unique columns in range, positive diagonal — on all
  // host threads; the first failing row (lowest index) is reported
  {
    std::mutex mu;
    int64_t bad_row = INT64_MAX;
    int bad_kind = 0;
    int64_t maxrow = 0;
    parallel_rows(n, [&](int64_t lo, int64_t hi) {
      int64_t mr = 0;
      for (int64_t i = lo; i < hi; ++i) {
        mr = std::max(mr, RP[i + 1] - RP[i]);
        int kind = 0;
        bool diag = false;
        for (int64_t p = RP[i]; p < RP[i + 1] && !kind; ++p) {
          const int64_t c = COL[p];
          if (c < 0 || c >= n_global) kind = 1;
          else if (p > RP[i] && COL[p - 1] >= c) kind = 2;
          else if (c == row_begin + i) {
            if (!(VAL[p] > 0.0)) kind = 3;
            diag = true;
          }
        }
        if (!kind && !diag) kind = 4;
        if (kind) {
          std::lock_guard<std::mutex> g(mu);
          if (i < bad_row) {
            bad_row = i;
            bad_kind = kind;
          }
          break;
        }
      }
      std::lock_guard<std::mutex> g(mu);
      maxrow = std::max(maxrow, mr);
    });
    if (bad_kind) {
      static const char* what[] = {"", "column out of range", "columns not strictly ascending",
                                   "non-positive diagonal", "missing diagonal"};
      return fail(ctx, EKS_ERR_BAD_MATRIX, "%s in row %lld", what[bad_kind], (long long)(row_begin + bad_row));
    }
    ctx->maxrow = maxrow;
  }
  // ---- slab table of all ranks
  std::vector<int64_t> ranges(2 * ctx->nranks);
  ranges[2 * ctx->rank] = row_begin;
  ranges[2 * ctx->rank + 1] = row_end;
  if (ctx->nranks > 1) {
    int64_t* d = nullptr;
    CK(cudaMalloc((void**)&d, sizeof(int64_t) * 2 * ctx->nranks));
    CK(cudaMemcpy(d + 2 * ctx->rank, ranges.data() + 2 * ctx->rank, 2 * sizeof(int64_t), cudaMemcpyHostToDevice));
    NK(ncclAllGather(d + 2 * ctx->rank, d, 2, ncclInt64, ctx->comm, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(ranges.data(), d, sizeof(int64_t) * 2 * ctx->nranks, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int q = 0; q + 1 < ctx->nranks; ++q)
      if (ranges[2 * q + 1] != ranges[2 * q + 2] || ranges[0] != 0 || ranges[2 * ctx->nranks - 1] != n_global)
        return fail(ctx, EKS_ERR_INVALID_ARG, "rank slabs must tile [0,n) in rank order");
  }
  // ---- halo plan (host-only, also exported as eks_plan_halo for the multi-rank CPU tests)
  HaloPlan plan;
  plan_halo(ctx->rank, ctx->nranks, ranges.data(), n, RP, COL, plan);
  ctx->ranges = ranges;
  dfree(ctx->mpk_sv);
  ctx->mpk_sv = nullptr;
  ctx->mpk_d = 0;
  ctx->mpk_ok = -1;
  const int64_t old_before = ctx->halo_before, old_after = ctx->halo_after;
  ctx->recvs = plan.recvs;
  ctx->sends.clear();
  ctx->halo_before = plan.halo_before;
  ctx->halo_after = plan.halo_after;
  if (ctx->nranks > 1) {
    // everyone learns who needs which of its rows
    std::vector<int64_t> req(2 * ctx->nranks * ctx->nranks, 0);
    for (int q = 0; q < 2 * ctx->nranks; ++q) req[2 * ctx->rank * ctx->nranks + q] = plan.need[q];
    int64_t* d = nullptr;
    const size_t per = 2 * ctx->nranks;
    CK(cudaMalloc((void**)&d, sizeof(int64_t) * per * ctx->nranks));
    CK(cudaMemcpy(d + per * ctx->rank, req.data() + per * ctx->rank, sizeof(int64_t) * per, cudaMemcpyHostToDevice));
    NK(ncclAllGather(d + per * ctx->rank, d, per, ncclInt64, ctx->comm, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(req.data(), d, sizeof(int64_t) * per * ctx->nranks, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int q = 0; q < ctx->nranks; ++q) {
      if (q == ctx->rank) continue;
      const int64_t lo = req[2 * (q * ctx->nranks + ctx->rank)], hi = req[2 * (q * ctx->nranks + ctx->rank) + 1];
      if (hi > lo) ctx->sends.push_back({q, lo, hi});
    }
  }
  const int32_t* ECOL = plan.ecol.empty() ? COL : plan.ecol.data();  // one rank: the columns themselves
  ctx->int_lo = plan.int_lo;
  ctx->int_hi = plan.int_hi;
  // ---- upload (the block workspace survives when the slab geometry is unchanged)
  if (!ctx->have_matrix || ctx->n != n || old_before != ctx->halo_before || old_after != ctx->halo_after)
    free_workspace(ctx);
  for (void* p : {(void*)ctx->d_rp, (void*)ctx->d_col, (void*)ctx->d_val, (void*)ctx->d_ecol, (void*)ctx->d_eval,
                  (void*)ctx->d_tmax, (void*)ctx->d_seg, (void*)ctx->d_segrows, (void*)ctx->d_segown,
                  (void*)ctx->d_lidx, (void*)ctx->d_sval})
    dfree(p);
  dfree(ctx->d_sv);
  ctx->d_sv = nullptr;
  ctx->grid_ok = false;
  ctx->d_tmax = ctx->d_seg = ctx->d_segrows = ctx->d_segown = nullptr;
  ctx->d_lidx = nullptr;
  ctx->d_sval = nullptr;
  ctx->seg_ok = false;
  ctx->d_rp = nullptr;
  ctx->d_col = nullptr;
  ctx->d_val = nullptr;
  ctx->d_ecol = nullptr;
  ctx->d_eval = nullptr;
  ctx->ell_w = 0;
  ctx->have_matrix = false;
  std::vector<int32_t> rp32(n + 1);
  parallel_rows(n + 1, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) rp32[i] = (int32_t)RP[i];
  });
  // +16 bytes of padding: the fused SpMM copies aligned 16-byte chunks that may run past the end
  CK(cudaMalloc((void**)&ctx->d_rp, sizeof(int) * (n + 1) + 16));
  CK(cudaMemcpy(ctx->d_rp, rp32.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
  if (early_col) {  // copied under the validation (one rank: ECOL = COL)
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->d_col = early_col;
    ctx->d_val = early_val;
    early_col = nullptr;
    early_val = nullptr;
  } else {
    CK(cudaMalloc((void**)&ctx->d_col, sizeof(int) * nnz + 16));
    CK(cudaMalloc((void**)&ctx->d_val, sizeof(double) * nnz + 16));
    CK(cudaMemcpy(ctx->d_col, ECOL, sizeof(int) * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_val, VAL, sizeof(double) * nnz, cudaMemcpyHostToDevice));
  }
  // ELL copy for the fused SpMM+Gram when every row has ≤ 8 entries (tiles of kEllTR rows,
  // slot-major inside a tile; padding: value 0 and the row's own column)
  // the plane-marching plan first: when it applies (one rank, stencil structure) and no path is
  // forced (EKS_SPMM_PATH), the ELL copy and the TMA segment plan are never used, so they are not
  // built (host setup time is part of the end-to-end number)
  ST(build_grid_plan(ctx, n, RP, COL, VAL, row_begin, plan.halo_before, plan.halo_after));
  const bool skip_alt = ctx->grid_ok && ctx->spmm_path == 0;
  const int w = skip_alt ? 0 : eks::ell_width((int)ctx->maxrow);
  if (w > 0) {
    const std::vector<int64_t> rp(RP, RP + n + 1);
    const std::vector<int32_t> ecol(ECOL, ECOL + nnz);
    const std::vector<double> val(VAL, VAL + nnz);
    const int64_t TR = eks::kEllTR, ntiles = (n + TR - 1) / TR;
    std::vector<int32_t> ec((size_t)ntiles * TR * w), tmax((size_t)ntiles, 0);
    std::vector<double> ev((size_t)ntiles * TR * w, 0.0);
    for (int64_t tile = 0; tile < ntiles; ++tile)
      for (int k = 0; k < w; ++k)
        for (int64_t rr = 0; rr < TR; ++rr) {
          const int64_t i = tile * TR + rr, e = (tile * w + k) * TR + rr;
          const int64_t len = i < n ? rp[i + 1] - rp[i] : 0;
          if (k < len) {
            ec[e] = ecol[rp[i] + k];
            ev[e] = val[rp[i] + k];
          } else {
            ec[e] = (int32_t)(plan.halo_before + (i < n ? i : 0));
          }
          tmax[tile] = std::max(tmax[tile], ec[e]);
        }
    CK(cudaMalloc((void**)&ctx->d_ecol, sizeof(int32_t) * ec.size()));
    CK(cudaMalloc((void**)&ctx->d_eval, sizeof(double) * ev.size()));
    CK(cudaMemcpy(ctx->d_ecol, ec.data(), sizeof(int32_t) * ec.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_eval, ev.data(), sizeof(double) * ev.size(), cudaMemcpyHostToDevice));
    CK(cudaMalloc((void**)&ctx->d_tmax, sizeof(int32_t) * tmax.size()));
    CK(cudaMemcpy(ctx->d_tmax, tmax.data(), sizeof(int32_t) * tmax.size(), cudaMemcpyHostToDevice));
    ST(build_seg_plan(ctx, n, rp, ecol, val, plan.halo_before, w));
    ctx->ell_w = w;
  }
  ctx->n_global = n_global;
  ctx->row_begin = row_begin;
  ctx->row_end = row_end;
  ctx->n = n;
  ctx->nnz = nnz;
  ctx->have_matrix = true;
  return EKS_OK;
}

extern "C++" {
namespace {
void free_precond(eks_ctx* ctx) {
  for (int w = 0; w < 2; ++w) {
    for (void* p : {(void*)ctx->pr_rp[w], (void*)ctx->pr_col[w], (void*)ctx->pr_val[w], (void*)ctx->pr_domlev[w],
                    (void*)ctx->pr_levptr[w], (void*)ctx->pr_rows[w], (void*)ctx->pr_prow[w], (void*)ctx->pr_pne[w],
                    (void*)ctx->pr_pdiag[w], (void*)ctx->pr_pcol[w], (void*)ctx->pr_pval[w], (void*)ctx->pr_pout[w]})
      dfree(p);
    ctx->pr_prow[w] = ctx->pr_pne[w] = ctx->pr_pcol[w] = ctx->pr_pout[w] = nullptr;
    ctx->pr_pdiag[w] = ctx->pr_pval[w] = nullptr;
    ctx->pr_rp[w] = ctx->pr_col[w] = ctx->pr_domlev[w] = ctx->pr_levptr[w] = ctx->pr_rows[w] = nullptr;
    ctx->pr_val[w] = nullptr;
  }
  dfree(ctx->pr_diag);
  ctx->pr_diag = nullptr;
  ctx->prec_nd = ctx->prec_ndl = 0;
  ctx->pr_ring[0] = ctx->pr_ring[1] = 0;
}

template <typename T>
eks_status upload(eks_ctx* ctx, T** dst, const std::vector<T>& v) {
  CK(cudaMalloc((void**)dst, sizeof(T) * std::max<size_t>(1, v.size())));
  if (!v.empty()) CK(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return EKS_OK;
}
}  // namespace
}  // extern "C++"

// Block-Jacobi IC(0) (reading R32), built on the host once per matrix: for each local row i, the
// entries of its domain's lower triangle are scattered into a dense row marker; each L_ik (k < i,
// ascending) subtracts Σ_j L_kj·L_ij over row k's strict-lower entries found in the marker.
eks_status eks_setup_precond(eks_ctx* ctx, eks_precond kind, int nd, const int64_t* row_ptr, const int32_t* col_idx,
                             const double* vals, eks_mem where) {
  if (!ctx) return EKS_ERR_INVALID_ARG;
  if (kind != EKS_PREC_IC0 && kind != EKS_PREC_CHOL) return fail(ctx, EKS_ERR_INVALID_ARG, "unknown preconditioner");
  if (!ctx->have_matrix) return fail(ctx, EKS_ERR_STATE, "eks_setup_csr has not been called");
  if (nd < 1 || !row_ptr || !col_idx || !vals) return fail(ctx, EKS_ERR_INVALID_ARG, "bad eks_setup_precond arguments");
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  free_precond(ctx);
  const int64_t N = ctx->n_global, n = ctx->n, r0 = ctx->row_begin;
  auto dlo = [&](int64_t d) { return d * N / nd; };
  int d0 = -1, d1 = -1;
  for (int d = 0; d <= nd; ++d) {
    if (dlo(d) == r0 && d0 < 0 && d < nd) d0 = d;
    if (dlo(d) == ctx->row_end) d1 = d;
  }
  if (d0 < 0 || d1 <= d0) return fail(ctx, EKS_ERR_INVALID_ARG, "slab is not a union of the %d preconditioner domains", nd);
  auto ndl_of = [](int a, int b) { return b - a; };
  std::vector<int64_t> rp(n + 1);
  if (where == EKS_MEM_HOST) memcpy(rp.data(), row_ptr, sizeof(int64_t) * (n + 1));
  else CK(cudaMemcpy(rp.data(), row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
  if (rp[0] != 0) return fail(ctx, EKS_ERR_BAD_MATRIX, "row_ptr[0] != 0");
  const int64_t nnz = rp[n];
  if (nnz != ctx->nnz) return fail(ctx, EKS_ERR_INVALID_ARG, "CSR differs from eks_setup_csr's");
  std::vector<int32_t> col(nnz);
  std::vector<double> val(nnz);
  if (where == EKS_MEM_HOST) {
    memcpy(col.data(), col_idx, sizeof(int32_t) * nnz);
    memcpy(val.data(), vals, sizeof(double) * nnz);
  } else {
    CK(cudaMemcpy(col.data(), col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(val.data(), vals, sizeof(double) * nnz, cudaMemcpyDeviceToHost));
  }
  // the same validation as eks_setup_csr: the IC(0) elimination below relies on
  // strictly ascending columns within a row (p < q stands in for col[p] < col[q])
  for (int64_t i = 0; i < n; ++i) {
    if (rp[i + 1] < rp[i]) return fail(ctx, EKS_ERR_BAD_MATRIX, "row_ptr not monotone at row %lld", (long long)i);
    bool diag = false;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = col[p];
      if (c < 0 || c >= N) return fail(ctx, EKS_ERR_BAD_MATRIX, "column %lld out of range", (long long)c);
      if (p > rp[i] && col[p - 1] >= c)
        return fail(ctx, EKS_ERR_BAD_MATRIX, "columns not strictly ascending in row %lld", (long long)(r0 + i));
      if (c == r0 + i) {
        if (!(val[p] > 0.0)) return fail(ctx, EKS_ERR_BAD_MATRIX, "non-positive diagonal in row %lld", (long long)(r0 + i));
        diag = true;
      }
    }
    if (!diag) return fail(ctx, EKS_ERR_BAD_MATRIX, "missing diagonal in row %lld", (long long)(r0 + i));
  }
  // strict-lower L (local columns) and its diagonal
  std::vector<int> dom(n);
  for (int d = d0; d < d1; ++d)
    for (int64_t g = dlo(d); g < dlo(d + 1); ++g) dom[g - r0] = d - d0;
  std::vector<int> Lrp(n + 1, 0), Lcol;
  std::vector<double> Lval, diag(n, 0.0);
  if (kind == EKS_PREC_IC0) {
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int64_t j = (int64_t)col[p] - r0;
        if (j < 0 || j > i || dom[j] != dom[i]) continue;
        if (j == i) diag[i] = val[p];
        else {
          Lcol.push_back((int)j);
          Lval.push_back(val[p]);
        }
      }
      Lrp[i + 1] = (int)Lcol.size();
    }
    std::vector<int64_t> mark(n, -1);  // mark[j] = position of L_ij in the current row i
    for (int64_t i = 0; i < n; ++i) {
      for (int p = Lrp[i]; p < Lrp[i + 1]; ++p) mark[Lcol[p]] = p;
      for (int p = Lrp[i]; p < Lrp[i + 1]; ++p) {
        const int k = Lcol[p];
        double v = Lval[p];
        for (int q = Lrp[k]; q < Lrp[k + 1]; ++q) {  // row k's columns j < k
          const int64_t pj = mark[Lcol[q]];
          if (pj >= 0 && pj < p) v -= Lval[q] * Lval[pj];
        }
        Lval[p] = v / diag[k];
      }
      double dd = diag[i];
      for (int p = Lrp[i]; p < Lrp[i + 1]; ++p) dd -= Lval[p] * Lval[p];
      for (int p = Lrp[i]; p < Lrp[i + 1]; ++p) mark[Lcol[p]] = -1;
      if (!(dd > 0.0)) return fail(ctx, EKS_ERR_BREAKDOWN, "IC(0) pivot %lld <= 0", (long long)(i + r0));
      diag[i] = std::sqrt(dd);
    }
  } else {
    // complete Cholesky of each diagonal block (Table 6): the fill of the natural-order factor stays in
    // the row envelope, so row i of the strict lower L holds columns first[i]..i−1; domains are
    // independent and factorized on all host threads
    std::vector<int> first(n);
    for (int64_t i = 0; i < n; ++i) {
      int64_t f = i;
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int64_t j = (int64_t)col[p] - r0;
        if (j >= 0 && j < i && dom[j] == dom[i]) f = std::min(f, j);
        if (j == i) diag[i] = val[p];
      }
      first[i] = (int)f;
      if ((int64_t)Lrp[i] + (i - f) >= INT_MAX) return fail(ctx, EKS_ERR_OOM, "Cholesky envelope exceeds 2^31 entries");
      Lrp[i + 1] = Lrp[i] + (int)(i - f);
    }
    Lcol.resize(Lrp[n]);
    Lval.assign(Lrp[n], 0.0);
    for (int64_t i = 0; i < n; ++i) {
      for (int p = Lrp[i]; p < Lrp[i + 1]; ++p) Lcol[p] = first[i] + (p - Lrp[i]);
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int64_t j = (int64_t)col[p] - r0;
        if (j >= first[i] && j < i) Lval[Lrp[i] + (j - first[i])] = val[p];
      }
    }
    std::atomic<int64_t> bad{-1};
    std::atomic<int> next{0};
    auto work = [&]() {
      for (int d; (d = next++) < ndl_of(d0, d1);) {
        const int64_t lo = dlo(d + d0) - r0, hi = dlo(d + d0 + 1) - r0;
        for (int64_t i = lo; i < hi; ++i) {
          const int fi = first[i];
          double* Li = Lval.data() + Lrp[i];  // Li[j − fi] = L_ij
          for (int j = fi; j < i; ++j) {
            const int fj = first[j];
            const double* Lj = Lval.data() + Lrp[j];
            double v = Li[j - fi];
            for (int k = std::max(fi, fj); k < j; ++k) v -= Li[k - fi] * Lj[k - fj];
            Li[j - fi] = v / diag[j];
          }
          double dd = diag[i];
          for (int k = fi; k < i; ++k) dd -= Li[k - fi] * Li[k - fi];
          if (!(dd > 0.0)) {
            bad = i + r0;
            return;
          }
          diag[i] = std::sqrt(dd);
        }
      }
    };
    const int nthr = std::max(1, std::min<int>(ndl_of(d0, d1), (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int k = 1; k < nthr; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    if (bad >= 0) return fail(ctx, EKS_ERR_BREAKDOWN, "Cholesky pivot %lld <= 0", (long long)bad.load());
  }
  // Lᵗ strict upper (row i: L_ki, k > i, ascending k)
  std::vector<int> Urp(n + 1, 0), Ucol(Lcol.size());
  std::vector<double> Uval(Lcol.size());
  for (int c : Lcol) ++Urp[c + 1];
  for (int64_t i = 0; i < n; ++i) Urp[i + 1] += Urp[i];
  {
    std::vector<int> fill(Urp.begin(), Urp.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int p = Lrp[i]; p < Lrp[i + 1]; ++p) {
        Ucol[fill[Lcol[p]]] = (int)i;
        Uval[fill[Lcol[p]]++] = Lval[p];
      }
  }
  // level schedules per domain: forward lev(i) = 1 + max lev(k), k < i in row i of L;
  // backward from the last row with Lᵗ
  const int ndl = d1 - d0;
  std::vector<int> sched[2], ringw(2, 0), maxe_w(2, 0);
  for (int w = 0; w < 2; ++w) {
    const std::vector<int>& R = w ? Urp : Lrp;
    const std::vector<int>& Cc = w ? Ucol : Lcol;
    std::vector<int> lev(n, 0);
    if (!w)
      for (int64_t i = 0; i < n; ++i)
        for (int p = R[i]; p < R[i + 1]; ++p) lev[i] = std::max(lev[i], lev[Cc[p]] + 1);
    else
      for (int64_t i = n - 1; i >= 0; --i)
        for (int p = R[i]; p < R[i + 1]; ++p) lev[i] = std::max(lev[i], lev[Cc[p]] + 1);
    std::vector<int> domlev(ndl + 1, 0), levptr, rows;
    int maxl = 0;
    for (int d = 0; d < ndl; ++d) {
      const int64_t lo = dlo(d + d0) - r0, hi = dlo(d + d0 + 1) - r0;
      int nl = 0;
      for (int64_t i = lo; i < hi; ++i) nl = std::max(nl, lev[i] + 1);
      maxl = std::max(maxl, nl);
      std::vector<std::vector<int>> by(nl);
      for (int64_t i = lo; i < hi; ++i) by[lev[i]].push_back((int)i);
      domlev[d] = (int)levptr.size();
      for (auto& v : by) {
        levptr.push_back((int)rows.size());
        rows.insert(rows.end(), v.begin(), v.end());
      }
    }
    domlev[ndl] = (int)levptr.size();
    levptr.push_back((int)rows.size());
    ctx->pr_levels[w] = maxl;
    // ring width: the smallest power of two W such that the row that next takes a row's slot
    // (r + W forward, r − W backward, same domain) is solved at a later level than every reader
    // of r; rows must have ≤ kTrsvMaxE entries.  0 = use the plain kernel.
    {
      std::vector<int> maxrd(n, -1);
      int maxe = 0;
      for (int64_t i = 0; i < n; ++i) {
        maxe = std::max(maxe, R[i + 1] - R[i]);
        for (int p = R[i]; p < R[i + 1]; ++p) maxrd[Cc[p]] = std::max(maxrd[Cc[p]], lev[i]);
      }
      int best = 0;
      if (maxe <= eks::kTrsvMaxE)
        for (int W = 2; W <= 4096 && !best; W *= 2) {
          bool ok = true;
          // every row r owns slot r & (W-1) from its own level until its last reader's level;
          // the next row of the slot chain (r + W forward, r − W backward, same domain) must
          // be solved strictly later, for EVERY r (rows without readers included: otherwise
          // the chain r, r+W, r+2W, … need not be level-monotone and two rows of one level
          // could share a slot)
          for (int64_t r = 0; r < n && ok; ++r) {
            const int need = std::max(lev[r], maxrd[r]);
            const int64_t j = w ? r - W : r + W;
            if (j < 0 || j >= n || dom[j] != dom[r]) continue;
            ok = lev[j] > need;
          }
          if (ok) best = W;
        }
      ringw[w] = best;
      maxe_w[w] = maxe;
      ctx->pr_maxe[w] = maxe;
    }
    sched[w] = rows;
    int maxdl = 0, maxr = 0;
    for (int d = 0; d < ndl; ++d) maxdl = std::max(maxdl, domlev[d + 1] - domlev[d]);
    for (size_t q = 0; q + 1 < levptr.size(); ++q) maxr = std::max(maxr, levptr[q + 1] - levptr[q]);
    ctx->pr_maxlev[w] = maxdl;
    ctx->pr_maxrows[w] = maxr;
    ST(upload(ctx, &ctx->pr_rp[w], R));
    ST(upload(ctx, &ctx->pr_col[w], Cc));
    ST(upload(ctx, &ctx->pr_val[w], w ? Uval : Lval));
    ST(upload(ctx, &ctx->pr_domlev[w], domlev));
    ST(upload(ctx, &ctx->pr_levptr[w], levptr));
    ST(upload(ctx, &ctx->pr_rows[w], rows));
  }
  // flattened level-order schedules for k_trsv_ring (both sweeps must qualify): position → row,
  // output index (forward: the row's position in the backward schedule; backward: the row)
  if (ringw[0] && ringw[1]) {
    std::vector<int> bpos(n);
    for (size_t q = 0; q < sched[1].size(); ++q) bpos[sched[1][q]] = (int)q;
    for (int w = 0; w < 2; ++w) {
      const std::vector<int>& R = w ? Urp : Lrp;
      const std::vector<int>& Cc = w ? Ucol : Lcol;
      const std::vector<double>& V = w ? Uval : Lval;
      const std::vector<int>& rows = sched[w];
      const int E = maxe_w[w] <= 4 ? std::max(1, maxe_w[w]) : 8;  // the kernel's instantiations
      std::vector<int> prow(rows.size()), pout(rows.size()), pne(rows.size()), pcol(rows.size() * E, 0);
      std::vector<double> pdiag(rows.size()), pval(rows.size() * E, 0.0);
      for (size_t q = 0; q < rows.size(); ++q) {
        const int i = rows[q];
        prow[q] = i;
        pout[q] = w ? i : bpos[i];
        pne[q] = R[i + 1] - R[i];
        pdiag[q] = 1.0 / diag[i];
        for (int p = R[i], e = 0; p < R[i + 1]; ++p, ++e) {
          pcol[q * E + e] = Cc[p];
          pval[q * E + e] = V[p];
        }
      }
      ctx->pr_E[w] = E;
      ctx->pr_ring[w] = ringw[w];
      ST(upload(ctx, &ctx->pr_prow[w], prow));
      ST(upload(ctx, &ctx->pr_pout[w], pout));
      ST(upload(ctx, &ctx->pr_pne[w], pne));
      ST(upload(ctx, &ctx->pr_pdiag[w], pdiag));
      ST(upload(ctx, &ctx->pr_pcol[w], pcol));
      ST(upload(ctx, &ctx->pr_pval[w], pval));
    }
  }
  ST(upload(ctx, &ctx->pr_diag, diag));
  ctx->prec_nd = nd;
  ctx->prec_ndl = ndl;
  return EKS_OK;
}

// One captured phase of the steady-state s-step SRE-CG outer iteration (eks_options.use_graph).
struct PhaseGraph {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;  // kept for the device-resident loop (use_graph = 2)
  int nb0 = 0;                  // nblocks when it was captured (block indices baked into the kernels)
  long long launches = 0;       // this library's kernels in it
  double bytes = 0, flops = 0;
};

// use_graph value of the options (0 off, 1 phase-graph replay, 2 also the device-resident loop)
static int graphs_on_req(const eks_options* opt) { return opt ? opt->use_graph : 0; }

eks_status ensure_hist(eks_ctx* ctx, size_t count) {
  if (!ctx->d_loop) CK(cudaMalloc((void**)&ctx->d_loop, sizeof(eks::LoopState)));
  if (ctx->hist_cap < count) {
    dfree(ctx->d_hist);
    ctx->hist_cap = 0;
    CK(cudaMalloc((void**)&ctx->d_hist, sizeof(double) * count));
    ctx->hist_cap = count;
  }
  return EKS_OK;
}

// The device-resident loop graph: while(hw) { switch(hs) { phase 0 … P−1 } ; k_loop_check }.
// hw defaults to 1 and hs to 0 at every launch (the host launches it at a phase-0 iteration whose
// loop test it has just evaluated).  Conditional bodies allow kernels, memcpy/memset and child
// graphs (CUDA 12.4+), which is everything a one-rank phase graph holds.
eks_status build_loop_graph(eks_ctx* ctx, const PhaseGraph* pg, int nphase, cudaGraphExec_t* out) {
  *out = nullptr;
  if (!ctx->d_loop || !ctx->d_hist) return fail(ctx, EKS_ERR_STATE, "loop state not allocated");
  cudaGraph_t top = nullptr;
  CK(cudaGraphCreate(&top, 0));
  struct TopGuard {
    cudaGraph_t g;
    ~TopGuard() { cudaGraphDestroy(g); }
  } tg{top};
  cudaGraphConditionalHandle hw, hs;
  CK(cudaGraphConditionalHandleCreate(&hw, top, 1, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&hs, top, 0, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, top, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphNodeParams sp{};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = hs;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  sp.conditional.size = (unsigned)nphase;
  cudaGraphNode_t sn;
  CK(cudaGraphAddNode(&sn, body, nullptr, 0, &sp));
  for (int p = 0; p < nphase; ++p) {
    const cudaGraph_t pgraph = pg[p].graph;
    if (!pgraph) return fail(ctx, EKS_ERR_STATE, "phase graph %d missing", p);
    cudaGraphNode_t cn;
    CK(cudaGraphAddChildGraphNode(&cn, sp.conditional.phGraph_out[p], nullptr, 0, pgraph));
  }
  // the check kernel after the switch, captured into the body
  cudaStream_t cs = ctx->stream;
  CK(cudaStreamBeginCaptureToGraph(cs, body, &sn, nullptr, 1, cudaStreamCaptureModeThreadLocal));
  const cudaError_t le = eks::launch_loop_check(cs, hw, hs, ctx->d_loop, ctx->scal, ctx->flag, ctx->d_hist);
  cudaGraph_t cap = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(cs, &cap);
  CK(le);
  CK(ee);
  CK(cudaGraphInstantiate(out, top, 0));
  return EKS_OK;
}

eks_status eks_solve(eks_ctx* ctx, eks_method method, int s, int t, double tol, const double* b, double* x,
                     eks_mem where, int max_outer, eks_report* rep) {
  eks_options o{};
  o.max_outer = max_outer;
  return eks_solve_ex(ctx, method, s, t, tol, b, x, where, &o, rep);
}

eks_status eks_solve_ex(eks_ctx* ctx, eks_method method, int s, int t, double tol, const double* b, double* x,
                        eks_mem where, const eks_options* opt, eks_report* rep) {
  ST(check_ready(ctx));
  if (method < EKS_SRE_CG || method > EKS_CA_MSDO_CG) return fail(ctx, EKS_ERR_INVALID_ARG, "unknown method");
  const bool ca = method >= EKS_CA_SRE_CG;
  const int base = ca ? method - EKS_CA_SRE_CG : method;
  const int arnoldi = (opt && opt->arnoldi) ? opt->arnoldi : 7;
  if (ca && (arnoldi != 5 && arnoldi != 7)) return fail(ctx, EKS_ERR_INVALID_ARG, "arnoldi must be 5 or 7");
  const int ortho = opt ? opt->ortho : 0;
  const bool restr = opt && opt->restructured;
  if (ortho != 0 && ortho != 1) return fail(ctx, EKS_ERR_INVALID_ARG, "ortho must be 0 (A-CholQR) or 1 (Pre-CholQR)");
  if (ca && ortho) return fail(ctx, EKS_ERR_INVALID_ARG, "Pre-CholQR is for the s-step methods");
  const bool prec = opt && opt->precond;
  if (prec && restr) return fail(ctx, EKS_ERR_INVALID_ARG, "precond is not defined for the restructured methods");
  if (prec && !ctx->prec_nd) return fail(ctx, EKS_ERR_STATE, "eks_setup_precond has not been called");
  if (prec && ctx->prec_nd % t)
    return fail(ctx, EKS_ERR_INVALID_ARG, "precond needs t | ndomains (%d), P:874", ctx->prec_nd);
  if (restr && method != EKS_SRE_CG && method != EKS_SRE_CG2)
    return fail(ctx, EKS_ERR_INVALID_ARG, "restructured exists for SRE-CG and SRE-CG2 only (P:729)");
  if (ca && (s * t > eks::kCaMax || s > eks::kCaMaxBlocks))
    return fail(ctx, EKS_ERR_INVALID_ARG, "CA methods need s*t <= %d and s <= %d", eks::kCaMax, eks::kCaMaxBlocks);
  if (s < 1 || !valid_t(t) || t > ctx->n_global) return fail(ctx, EKS_ERR_INVALID_ARG, "bad s=%d or t=%d", s, t);
  if (!(tol >= 0.0)) return fail(ctx, EKS_ERR_INVALID_ARG, "tol must be >= 0");
  if (!b || !x) return fail(ctx, EKS_ERR_INVALID_ARG, "NULL b or x");
  if (t % ctx->nranks) return fail(ctx, EKS_ERR_INVALID_ARG, "t %% nranks != 0");
  if (ctx->nranks > 1) {  // slab must be a union of domains (reading R1)
    const int64_t dlo = (int64_t)(ctx->rank * (t / ctx->nranks)) * ctx->n_global / t;
    const int64_t dhi = (int64_t)((ctx->rank + 1) * (t / ctx->nranks)) * ctx->n_global / t;
    if (dlo != ctx->row_begin || dhi != ctx->row_end)
      return fail(ctx, EKS_ERR_INVALID_ARG, "rank slab is not the union of its t/nranks domains");
  }
  const int kmax = (opt && opt->max_outer > 0) ? opt->max_outer : 5000;
  begin_run(ctx, opt);
  auto wall0 = std::chrono::steady_clock::now();
  ST(ensure_workspace(ctx, t, s));
  // ring slots: SRE-CG keeps its 2-block window + the new block (restructured: the s blocks of
  // the outer iteration until their updates), CA SRE-CG the (s+1)-block window + s new blocks
  const int ring = (method == EKS_SRE_CG) ? (restr ? std::max(3, s + 1) : 3) : (method == EKS_CA_SRE_CG ? 2 * s + 1 : 0);
  ctx->ortho = ortho;
  ctx->use_prec = prec;
  ctx->mpk_ok = -1;  // the matrix-powers decision depends on the preconditioner option
  // full-basis s-step methods (SRE-CG2, MSDO-CG) keep every W; A·W is cached only with
  // aq_cache = 1 — by default they store Q only (reading R24): the same 4 window sweeps per CGS2, two
  // more SpMMs per block, half the memory per outer iteration
  const int aqc = opt ? opt->aq_cache : 0;
  if (aqc < 0 || aqc > 2) return fail(ctx, EKS_ERR_INVALID_ARG, "aq_cache must be 0 (auto), 1 (on) or 2 (off)");
  // one-synch CGS2 (reading R36) forms A·Z2 = A·Z1 − (AQ)C2: it needs A·Q (auto turns the cache on)
  if (ctx->onesynch && (ca || ortho || restr || aqc == 2))
    return fail(ctx, EKS_ERR_INVALID_ARG, "onesynch is for the s-step methods with A-CholQR, not restructured, "
                                          "with A·Q cached (aq_cache != 2)");
  ctx->aq_off = !ring && !ca && !restr && aqc != 1 && !ctx->onesynch;
  ctx->last_aq_off = ctx->aq_off;
  ctx->lazy = method == EKS_SRE_CG && !restr && eks::sweep_supported(t) && lazy_env();
  ctx->last_lazy = ctx->lazy;
  int plan_fit = -1;  // memory planner: outer iterations the device can hold (full-basis methods)
  if (!ring) {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    double held = 0.0;  // blocks of earlier solves are reused
    for (auto& bk : ctx->Wpool) if (bk.base && bk.owned) held += 8.0 * n_ext(ctx) * t;
    for (auto& bk : ctx->AWpool) if (bk.base && bk.owned) held += 8.0 * ctx->n * t;
    const double per_outer = (double)s * 8.0 * t * ((double)n_ext(ctx) + (ctx->aq_off ? 0.0 : (double)ctx->n));
    plan_fit = (int)(((double)fr - 64.0 * 1024 * 1024 + held) / per_outer);
  }
  EventPair ev;
  CK(ev.create());
  CK(cudaEventRecord(ev.e0, ctx->stream));
  // r0 = b − A x0, ρ0 = ||r0||  (line 1 of Alg 3/4/6)
  ST(copy_in(ctx, ctx->b, b, ctx->n, where));
  ST(copy_in(ctx, ctx->xv.loc, x, ctx->n, where));
  ST(residual(ctx, ctx->r, ctx->scal + 0));
  ST(sync_scalars(ctx, 1));
  const double rho0 = std::sqrt(ctx->h_scal[0]);
  double rho = rho0;
  ctx->hist.assign(1, rho0);
  int k = 1, nblocks = 0, breakdown_block = -1, max_fit = -1;
  eks_status status = EKS_OK;
  // CUDA-graph replay (eks_options.use_graph): steady-state s-step SRE-CG outer iterations (k ≥ 3:
  // the 2-block window is full, the fused next-C1 is running) are the same stream work up to the
  // ring slots (period 3/gcd(3, s) outer iterations) and the r / r_new swap (period 2): one graph
  // per phase of the combined period P ∈ {2, 6} is captured from a normal iteration and replayed
  // after that.  Everything a steady iteration touches is allocated before the first capture
  // (prealloc_steady), so no cudaMalloc/cudaFree can happen inside a capture.
  // Several ranks: the NCCL halo exchanges and allreduces are captured with the kernels (the comm
  // stream forks from and joins the solve stream through events).  Should a capture fail, the outer
  // iteration (which did not execute while captured) runs uncaptured and graphs stay off.
  bool graphs_on = opt && opt->use_graph && method == EKS_SRE_CG && !restr && !prec && !ortho && !ctx->prof_on;
  const int gperiod = (s % 3 == 0) ? 2 : 6;
  PhaseGraph pg[6];
  // Device-resident loop control (use_graph = 2): once every phase is captured, the
  // rest of the solve is ONE graph launch — a while node (condition: the loop test of P:146) around a
  // switch node over the phase graphs (child graphs) followed by k_loop_check, which evaluates the
  // test on the device and selects the next phase.  No host synchronisation per outer iteration.
  bool dloop_on = graphs_on_req(opt) == 2;
  cudaGraphExec_t loop_exec = nullptr;
  struct GraphGuard {
    PhaseGraph* g;
    cudaGraphExec_t* lx;
    ~GraphGuard() {
      for (int i = 0; i < 6; ++i) {
        if (g[i].exec) cudaGraphExecDestroy(g[i].exec);
        if (g[i].graph) cudaGraphDestroy(g[i].graph);
      }
      if (*lx) cudaGraphExecDestroy(*lx);
    }
  } gguard{pg, &loop_exec};
  if (graphs_on) ST(prealloc_steady(ctx, t, ring));
  // One outer iteration's stream work (Alg 3/4/6 lines 3-12, or the CA outer iteration).
  auto outer_body = [&]() -> eks_status {
    ST(reset_flag(ctx));
    if (ca) {
      const int nb0 = nblocks;
      eks_status cs = ca_outer(ctx, t, s, base, arnoldi, k, nblocks, ring);
      if (cs == EKS_ERR_OOM) {
        max_fit = nb0 / s;
        status = EKS_ERR_OOM;
        return EKS_OK;
      }
      ST(cs);
    }
    for (int i = 0; i < (ca ? 0 : s); ++i) {
      Block *Wn = nullptr, *AWn = nullptr;
      const int idx = ring ? nblocks % ring : nblocks;
      eks_status as = slot(ctx, t, idx, &Wn, &AWn);
      if (as == EKS_ERR_OOM) {
        max_fit = nblocks / s;
        status = EKS_ERR_OOM;
        return EKS_OK;
      }
      ST(as);
      const bool seed = (i == 0) && (method == EKS_MSDO_CG || k == 1);
      const double* Zsrc = seed ? nullptr : ctx->AWpool[ring ? (nblocks - 1) % ring : nblocks - 1].loc;
      const int mode = restr ? 4 : (i == 0 ? 1 : 0) | (i == s - 1 ? 2 : 0);
      ST(make_block(ctx, t, method, ring, nblocks, seed, Zsrc, Wn, AWn, i * t, nblocks, mode));
      ++nblocks;
    }
    if (restr) {  // Alg 1/2 lines 14-17: s sequential updates (skipped on a breakdown flag)
      for (int i = 0; i < s; ++i) {
        const int j = nblocks - s + i, idx = ring ? j % ring : j;
        ST(restructured_update(ctx, t, ctx->Wpool[idx].loc, ctx->AWpool[idx].loc, i == 0 ? ctx->r : ctx->rnew,
                               ctx->rnew));
      }
      ctx->rho_fused = false;
    }
    if (ctx->rho_fused) ST(allreduce(ctx, ctx->scal + 1, 1));
    else ST(reduce_scalar(ctx, ctx->scal + 1));
    return EKS_OK;
  };
  int replay_phase = -1;  // phase whose graph ran this outer iteration (for the breakdown index)
  // while (ρ > ε ρ0 and k < k_max)   (reading R7)
  while (rho > tol * rho0 && k < kmax) {
    const int phase = (graphs_on && k >= 3) ? (k - 3) % gperiod : -1;
    replay_phase = -1;
    if (phase == 0 && dloop_on && pg[gperiod - 1].exec) {
      ST(ensure_hist(ctx, (size_t)kmax + 1));  // before the build: the graph bakes d_hist in
      if (!loop_exec) {
        const eks_status bs = build_loop_graph(ctx, pg, gperiod, &loop_exec);
        if (bs != EKS_OK || !loop_exec) {  // not supported here: keep the host-checked replay
          dloop_on = false;
          loop_exec = nullptr;
          cudaGetLastError();
          continue;
        }
      }
      // the rest of the solve on the device: one graph launch, one synchronisation
      eks::LoopState ls{};
      ls.k = k;
      ls.kmax = kmax;
      ls.nphase = gperiod;
      ls.thr = tol * rho0;
      CK(cudaMemcpyAsync(ctx->d_loop, &ls, sizeof(ls), cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaGraphLaunch(loop_exec, ctx->stream));
      CK(cudaMemcpyAsync(&ls, ctx->d_loop, sizeof(ls), cudaMemcpyDeviceToHost, ctx->stream));
      ST(stream_wait(ctx));
      const int k0 = k;
      ctx->hist.resize((size_t)ls.k);
      if (ls.k > k0)
        CK(cudaMemcpy(ctx->hist.data() + k0, ctx->d_hist + k0, sizeof(double) * (ls.k - k0), cudaMemcpyDeviceToHost));
      for (int i = 0; i < ls.iters; ++i) {  // iteration i ran phase i % gperiod
        const PhaseGraph& q = pg[i % gperiod];
        ctx->launches += q.launches + 1;
        ctx->model_bytes += q.bytes;
        ctx->model_flops += q.flops;
      }
      nblocks += s * ls.iters;
      if (ls.stop == 2) {  // breakdown in the last iteration the graph ran (its phase: (iters-1) % P)
        breakdown_block = ls.fl + (nblocks - s - pg[(ls.iters - 1) % gperiod].nb0);
        status = EKS_ERR_BREAKDOWN;
      }
      if ((ls.k - k0) % 2) std::swap(ctx->r, ctx->rnew);
      k = ls.k;
      rho = ctx->hist.back();
      if (ls.stop == 3) status = EKS_ERR_NONFINITE;
      break;
    }
    if (phase >= 0 && pg[phase].exec) {
      CK(cudaGraphLaunch(pg[phase].exec, ctx->stream));
      ctx->launches += pg[phase].launches;
      ctx->model_bytes += pg[phase].bytes;
      ctx->model_flops += pg[phase].flops;
      replay_phase = phase;
      nblocks += s;
    } else if (phase >= 0) {
      const long long l0 = ctx->launches;
      const double b0 = ctx->model_bytes, f0 = ctx->model_flops;
      const int nb0 = nblocks;
      cudaGraph_t g = nullptr;
      const bool c1r0 = ctx->c1_ready;
      eks_status cst = EKS_OK;
      cudaError_t ie = cudaSuccess;
      {
        CaptureGuard cap(ctx->stream);  // ends (and discards) the capture on every exit path
        ie = cap.begin();
        if (ie == cudaSuccess) cst = outer_body();
        if (status == EKS_ERR_OOM) break;  // (cannot happen after prealloc_steady)
        if (ie == cudaSuccess && cst == EKS_OK) ie = cap.end(&g);
      }
      if (ie == cudaSuccess && cst == EKS_OK) {
        ie = cudaGraphInstantiate(&pg[phase].exec, g, 0);
        if (dloop_on) pg[phase].graph = g;
        else cudaGraphDestroy(g);
      } else if (g) {
        cudaGraphDestroy(g);
      }
      if (ie != cudaSuccess || cst != EKS_OK) {  // nothing ran: undo the bookkeeping, run it plainly
        cudaGetLastError();
        if (ctx->nranks == 1 && cst != EKS_OK) return cst;  // one rank: a real error
        graphs_on = false;
        pg[phase].exec = nullptr;
        nblocks = nb0;
        ctx->launches = l0;
        ctx->model_bytes = b0;
        ctx->model_flops = f0;
        ctx->c1_ready = c1r0;  // the fused next-C1 of the last executed block is still in C1
        ST(outer_body());
        goto iteration_done;
      }
      pg[phase].nb0 = nb0;
      pg[phase].launches = ctx->launches - l0;
      pg[phase].bytes = ctx->model_bytes - b0;
      pg[phase].flops = ctx->model_flops - f0;
      CK(cudaGraphLaunch(pg[phase].exec, ctx->stream));
      replay_phase = phase;
    } else {
      ST(outer_body());
      if (status == EKS_ERR_OOM) break;
    }
  iteration_done:
    ST(sync_scalars(ctx, 2));
    const int fl = ctx->h_flag[1];
    if (fl != INT_MAX) {  // A-CholQR breakdown: x stays the last completed iterate
      // a replayed graph carries the block indices of the iteration it was captured from
      breakdown_block = replay_phase >= 0 ? fl + (nblocks - s - pg[replay_phase].nb0) : fl;
      status = EKS_ERR_BREAKDOWN;
      break;
    }
    std::swap(ctx->r, ctx->rnew);  // r_k = r_{k-1} − A V α̃
    rho = std::sqrt(ctx->h_scal[1]);
    ctx->hist.push_back(rho);
    ++k;
    if (!std::isfinite(rho)) {
      status = EKS_ERR_NONFINITE;
      break;
    }
  }
  ctx->last_t = t;
  ctx->last_nblocks = nblocks;
  ctx->last_ring = ring;
  // true residual at exit
  ST(residual(ctx, nullptr, ctx->scal + 2));
  {
    KScope kk(ctx, EKS_K_OTHER);
    CK(eks::launch_sumsq(ctx->stream, ctx->n, ctx->b, ctx->part, ctx->nblk));
    ctx->rho_nblk = ctx->nblk;
  }
  ST(reduce_scalar(ctx, ctx->scal + 3));
  ST(copy_out(ctx, x, ctx->xv.loc, ctx->n, where));
  CK(cudaEventRecord(ev.e1, ctx->stream));
  ST(sync_scalars(ctx, 4));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev.e0, ev.e1);
  (void)wall0;
  const bool converged = rho <= tol * rho0;
  if (status == EKS_OK && !converged) status = EKS_ERR_MAXITER;
  if (rep) {
    rep->outer_iters = k - 1;
    rep->converged = converged;
    rep->breakdown_block = breakdown_block;
    rep->max_outer_fit = (base == EKS_SRE_CG) ? -1 : (max_fit >= 0 ? max_fit : plan_fit);
    rep->rho0 = rho0;
    rep->rho = rho;
    const double nb = std::sqrt(ctx->h_scal[3]);
    rep->true_relres = nb > 0 ? std::sqrt(ctx->h_scal[2]) / nb : 0.0;
    rep->solve_seconds = ms * 1e-3;
    rep->model_bytes = ctx->model_bytes;
    rep->model_flops = ctx->model_flops;
    rep->gpu_launches = (int)ctx->launches;
    rep->rho_history = ctx->hist.data();
  }
  if (status == EKS_ERR_OOM) return fail(ctx, EKS_ERR_OOM, "full basis Q exhausted device memory after %d outer iterations", max_fit);
  if (status == EKS_ERR_BREAKDOWN) return fail(ctx, status, "A-CholQR breakdown in block %d", breakdown_block);
  if (status == EKS_ERR_MAXITER) return fail(ctx, status, "k_max=%d reached, rho/rho0=%.3e", kmax, rho / rho0);
  if (status == EKS_ERR_NONFINITE)
    return fail(ctx, status, "non-finite residual norm after outer iteration %d", k - 1);
  return EKS_OK;
}

eks_status eks_basis_sweep(eks_ctx* ctx, int t, int nblocks_total, const double* X0, double* W_last, eks_mem where,
                           const eks_options* opt, eks_report* rep) {
  ST(check_ready(ctx));
  if (!valid_t(t) || nblocks_total < 1 || !X0 || !W_last || t % ctx->nranks)
    return fail(ctx, EKS_ERR_INVALID_ARG, "bad basis-sweep arguments");
  begin_run(ctx, opt);
  ST(ensure_workspace(ctx, t, 1));
  ctx->use_prec = false;
  ctx->ortho = 0;
  ctx->last_aq_off = false;
  ctx->lazy = eks::sweep_supported(t) && lazy_env();
  ctx->last_lazy = ctx->lazy;
  EventPair ev;
  CK(ev.create());
  CK(cudaEventRecord(ev.e0, ctx->stream));
  ST(reset_flag(ctx));
  const int ring = 3;
  for (int j = 0; j < nblocks_total; ++j) {
    Block *Wn = nullptr, *AWn = nullptr;
    ST(slot(ctx, t, j % ring, &Wn, &AWn));
    const double* Zsrc = nullptr;
    if (j == 0) {
      ST(copy_in(ctx, ctx->Zs.loc, X0, ctx->n * t, where));
      Zsrc = ctx->Zs.loc;
    } else {
      Zsrc = ctx->AWpool[(j - 1) % ring].loc;
    }
    ST(make_block(ctx, t, EKS_SRE_CG, ring, j, false, Zsrc, Wn, AWn, 0, j, 4));
  }
  if (ctx->lazy) {  // W_last = Z2 R⁻¹ of the last slot (through the scratch block Zs)
    ST(materialize_w(ctx, t, (nblocks_total - 1) % ring, ctx->Zs.loc));
    ST(copy_out(ctx, W_last, ctx->Zs.loc, ctx->n * t, where));
  } else {
    ST(copy_out(ctx, W_last, ctx->Wpool[(nblocks_total - 1) % ring].loc, ctx->n * t, where));
  }
  ctx->last_t = t;
  ctx->last_nblocks = nblocks_total;
  ctx->last_ring = ring;
  CK(cudaEventRecord(ev.e1, ctx->stream));
  ST(sync_scalars(ctx, 1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev.e0, ev.e1);
  const int fl = ctx->h_flag[1];
  if (rep) {
    memset(rep, 0, sizeof *rep);
    rep->outer_iters = nblocks_total;
    rep->breakdown_block = fl == INT_MAX ? -1 : fl;
    rep->max_outer_fit = -1;
    rep->solve_seconds = ms * 1e-3;
    rep->model_bytes = ctx->model_bytes;
    rep->model_flops = ctx->model_flops;
    rep->gpu_launches = (int)ctx->launches;
  }
  if (fl != INT_MAX) return fail(ctx, EKS_ERR_BREAKDOWN, "A-CholQR breakdown in block %d", fl);
  return EKS_OK;
}

eks_status eks_plan_halo(int rank, int nranks, const int64_t* ranges, const int64_t* row_ptr, const int32_t* col,
                         int32_t* ext_col, int64_t* need, int64_t* geom) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !ranges || !row_ptr || !col || !ext_col || !need || !geom)
    return EKS_ERR_INVALID_ARG;
  for (int q = 0; q < nranks; ++q)
    if (ranges[2 * q] > ranges[2 * q + 1] || (q > 0 && ranges[2 * q] != ranges[2 * q - 1]) || ranges[0] != 0)
      return EKS_ERR_INVALID_ARG;
  const int64_t n = ranges[2 * rank + 1] - ranges[2 * rank];
  for (int64_t p = 0; p < row_ptr[n]; ++p)
    if (col[p] < 0 || col[p] >= ranges[2 * nranks - 1]) return EKS_ERR_BAD_MATRIX;
  HaloPlan P;
  plan_halo(rank, nranks, ranges, n, row_ptr, col, P);
  if (P.ecol.empty()) memcpy(ext_col, col, sizeof(int32_t) * row_ptr[n]);  // one rank: unchanged
  else memcpy(ext_col, P.ecol.data(), sizeof(int32_t) * P.ecol.size());
  memcpy(need, P.need.data(), sizeof(int64_t) * P.need.size());
  geom[0] = P.halo_before;
  geom[1] = P.halo_after;
  geom[2] = P.int_lo;
  geom[3] = P.int_hi;
  return EKS_OK;
}

eks_status eks_plan_grid(int64_t row_begin, int64_t row_end, const int64_t* row_ptr, const int32_t* col,
                         const double* vals, int64_t halo_before, int64_t halo_after, int64_t* geom, double* sv) {
  if (!row_ptr || !col || !vals || !geom || row_end <= row_begin) return EKS_ERR_INVALID_ARG;
  std::vector<double> v;
  if (!grid_plan_host(row_end - row_begin, row_ptr, col, vals, row_begin, halo_before, halo_after, geom, v)) {
    for (int k = 0; k < 6; ++k) geom[k] = 0;
    return EKS_OK;
  }
  if (sv) memcpy(sv, v.data(), sizeof(double) * v.size());
  return EKS_OK;
}

eks_status eks_get_profile(const eks_ctx* ctx, eks_profile* out) {
  if (!ctx || !out) return EKS_ERR_INVALID_ARG;
  *out = ctx->prof;
  return EKS_OK;
}

eks_status eks_destroy(eks_ctx* ctx) {
  if (!ctx) return EKS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_workspace(ctx);
  free_precond(ctx);
  dfree(ctx->d_rp);
  dfree(ctx->d_col);
  dfree(ctx->d_val);
  dfree(ctx->d_ecol);
  dfree(ctx->d_eval);
  dfree(ctx->d_tmax);
  dfree(ctx->d_seg);
  dfree(ctx->d_segrows);
  dfree(ctx->d_segown);
  dfree(ctx->d_lidx);
  dfree(ctx->d_sval);
  dfree(ctx->d_sv);
  dfree(ctx->mpk_sv);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& p : ctx->prof_pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
  dfree(ctx->d_hist);
  if (ctx->d_loop) cudaFree(ctx->d_loop);
  delete ctx;
  return EKS_OK;
}

const char* eks_error_string(const eks_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

// ============================================================================
// Kernel-level ABI (include/eks_kernels.h)
// ============================================================================
static eks_status k_ready(eks_ctx* ctx, int t) {
  ST(check_ready(ctx));
  if (ctx->nranks != 1) return fail(ctx, EKS_ERR_INVALID_ARG, "kernel-level calls are single-rank");
  if (!valid_t(t)) return fail(ctx, EKS_ERR_INVALID_ARG, "t=%d not in {1,2,4,...,64}", t);
  begin_run(ctx, nullptr);
  return ensure_workspace(ctx, t, 1);
}

eks_status eks_k_split(eks_ctx* ctx, int t, const double* r, double* Z) {
  ST(k_ready(ctx, t));
  CK(eks::launch_split(ctx->stream, t, ctx->n, ctx->row_begin, ctx->n_global, r, Z));
  CK(cudaStreamSynchronize(ctx->stream));
  return EKS_OK;
}

eks_status eks_k_spmm(eks_ctx* ctx, int t, const double* X, double* Y, double* G, const double* v, double* g) {
  ST(k_ready(ctx, t));
  Block xb;
  xb.base = const_cast<double*>(X);
  xb.loc = xb.base;
  if (!(G || g)) ST(spmm(ctx, xb, Y, t));
  if (G || g) {
    ST(spmm_gram(ctx, xb, Y, t, g ? v : nullptr, ctx->Bg));
    if (G) CK(cudaMemcpyAsync(G, ctx->Bg, sizeof(double) * t * t, cudaMemcpyDeviceToDevice, ctx->stream));
    if (g && v) CK(cudaMemcpyAsync(g, ctx->Bg + t * t, sizeof(double) * t, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return EKS_OK;
}

eks_status eks_plan_mpk(int nz, int d, int db, int da, int* steps) {
  if (nz < 1 || d < 1 || db < 0 || da < 0 || db > d || da > d || !steps) return EKS_ERR_INVALID_ARG;
  std::vector<MpkStep> st(d);
  mpk_plan(nz, d, db, da, st.data());
  for (int i = 0; i < d; ++i) {
    steps[4 * i] = st[i].zlo;
    steps[4 * i + 1] = st[i].zhi;
    steps[4 * i + 2] = st[i].gb;
    steps[4 * i + 3] = st[i].ga;
  }
  return EKS_OK;
}

eks_status eks_k_matrix_powers(eks_ctx* ctx, int t, int s, int z0, int z1, const double* X, double* V) {
  ST(k_ready(ctx, t));
  if (!eks::sweep_supported(t) || spmm_path_for(ctx, t) != 4)
    return fail(ctx, EKS_ERR_INVALID_ARG, "matrix powers need the plane-marching SpMM (stencil operator, t >= 8)");
  const int nzg = ctx->gplan.nz, d = s - 1;
  if (d < 1 || z0 < 0 || z1 <= z0 || z1 > nzg || !X || !V) return fail(ctx, EKS_ERR_INVALID_ARG, "bad slab or s");
  const int64_t plane = (int64_t)ctx->gplan.nx * ctx->gplan.ny;
  const int VS = (ctx->gplan.w + 1) & ~1;
  const int nz = z1 - z0, db = std::min(d, z0), da = std::min(d, nzg - z1);
  const size_t rows = (size_t)(db + nz + da) * plane;
  double* buf = nullptr;
  ST(dalloc(ctx, &buf, rows * t * (d + 1)));
  // every ghost or slab row a power may not read is NaN: a wrong plane range shows up in the slab rows
  CK(cudaMemsetAsync(buf, 0xFF, sizeof(double) * rows * t * (d + 1), ctx->stream));
  CK(cudaMemcpyAsync(buf, X + (size_t)(z0 - db) * plane * t, sizeof(double) * rows * t, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  std::vector<double*> L(d + 1);
  for (int i = 0; i <= d; ++i) L[i] = buf + (size_t)i * rows * t + (size_t)db * plane * t;
  eks_status stt = mpk_local(ctx, t, d, nz, db, da, ctx->gplan.sv + (size_t)(z0 - db) * plane * VS, L.data());
  if (stt == EKS_OK)
    for (int i = 1; i <= d && stt == EKS_OK; ++i)
      if (cudaMemcpyAsync(V + (size_t)(i - 1) * nz * plane * t, L[i], sizeof(double) * nz * plane * t,
                          cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
        stt = fail(ctx, EKS_ERR_CUDA, "matrix powers: copy failed");
  cudaStreamSynchronize(ctx->stream);
  dfree(buf);
  return stt;
}

eks_status eks_k_cgs2(eks_ctx* ctx, int t, int nq, const double* const* Q, const double* const* AQ, double* Z,
                      double* C1, double* C2) {
  ST(k_ready(ctx, t));
  if (nq < 1 || !Q || !AQ || !Z) return fail(ctx, EKS_ERR_INVALID_ARG, "bad cgs2 arguments");
  std::vector<const double*> q(Q, Q + nq), aq(AQ, AQ + nq);
  ST(cgs2(ctx, t, q, aq, Z, Z));
  if (C1) CK(cudaMemcpyAsync(C1, ctx->C1, sizeof(double) * nq * t * t, cudaMemcpyDeviceToDevice, ctx->stream));
  if (C2) CK(cudaMemcpyAsync(C2, ctx->C2, sizeof(double) * nq * t * t, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return EKS_OK;
}

eks_status eks_k_acholqr(eks_ctx* ctx, int t, const double* Z, double* W, double* AW, double* R, double* B) {
  ST(k_ready(ctx, t));
  if (!Z || !W || !AW) return fail(ctx, EKS_ERR_INVALID_ARG, "NULL argument");
  ST(reset_flag(ctx));
  Block wb;
  wb.base = W;
  wb.loc = W;
  if (W != Z) CK(cudaMemcpyAsync(W, Z, sizeof(double) * ctx->n * t, cudaMemcpyDeviceToDevice, ctx->stream));
  ST(spmm_gram(ctx, wb, AW, t, nullptr, ctx->Bg));
  CK(eks::launch_chol_fast(ctx->stream, t, ctx->Bg, nullptr, ctx->Rm, ctx->Rinv, nullptr, ctx->flag, 0));  // solve path
  if (eks::sweep_supported(t))
    CK(eks::launch_apply_tc(ctx->stream, t, ctx->n, W, AW, ctx->Rinv, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, 4, ctx->nblk, 0, nullptr, ctx->part2, eks::Tail{}));
  else
    CK(eks::launch_apply(ctx->stream, t, ctx->n, W, AW, ctx->Rinv, nullptr, nullptr, nullptr, nullptr, nullptr,
                         nullptr, nullptr, 4, ctx->nblk));
  if (R) CK(cudaMemcpyAsync(R, ctx->Rm, sizeof(double) * t * t, cudaMemcpyDeviceToDevice, ctx->stream));
  if (B) CK(cudaMemcpyAsync(B, ctx->Bg, sizeof(double) * t * t, cudaMemcpyDeviceToDevice, ctx->stream));
  ST(sync_scalars(ctx, 1));
  if (ctx->h_flag[1] != INT_MAX) return fail(ctx, EKS_ERR_BREAKDOWN, "A-CholQR breakdown");
  return EKS_OK;
}

eks_status eks_k_time_spmm(eks_ctx* ctx, int t, const double* X, double* Y, const double* v, int variant, int reps,
                           double* ms) {
  ST(k_ready(ctx, t));
  if (!X || !Y || !ms || reps < 1 || variant < 0 || variant > 7)
    return fail(ctx, EKS_ERR_INVALID_ARG, "bad eks_k_time_spmm arguments");
  if (variant > 0 && !eks::sweep_supported(t))
    return fail(ctx, EKS_ERR_INVALID_ARG, "fused SpMM+Gram needs t in {8,16,32,64}");
  ST(reset_flag(ctx));
  const size_t stride = eks::sweep_part_stride(t, 1, true);
  ST(ensure_part(ctx, stride * ctx->nblk));
  eks::CholArgs ch{};
  ch.on = variant == 3 && eks::spmm_gram_fused_chol(t);
  ch.R = ctx->Rm;
  ch.Rinv = ctx->Rinv;
  ch.alpha = v ? ctx->alpha : nullptr;
  ch.flag = ctx->flag;
  const eks::Tail tl = variant >= 2 ? tail(ctx, 2, ctx->Bg, stride) : eks::Tail{};
  int path = variant <= 3 ? spmm_path_for(ctx, t) : (variant == 4 && ctx->ell_w ? 1 : 2);
  if (variant == 6) {
    if (!(ctx->grid_ok && eks::spmm_grid_fits(t, ctx->gplan)))
      return fail(ctx, EKS_ERR_INVALID_ARG, "matrix is not stencil-structured (no grid plan)");
    path = 4;
  }
  const bool use_seg = path == 0, use_ell = path == 1;
  Block xb7;
  xb7.base = const_cast<double*>(X);
  xb7.loc = xb7.base;
  auto run = [&]() -> cudaError_t {
    if (variant == 7)  // exactly the solve's SpMM-block step (spmm_gram): fused, or SpMM + Gram sweep at t = 64
      return spmm_gram(ctx, xb7, Y, t, v, ctx->Bg) == EKS_OK ? cudaSuccess : cudaErrorUnknown;
    if (variant == 0)
      return eks::launch_spmm(ctx->stream, t, 0, (int)ctx->n, ctx->d_rp, ctx->d_col, ctx->d_val, X, Y, ctx->sms);
    if (path == 4) {
      cudaError_t e = eks::launch_spmm_grid(ctx->stream, t, ctx->gplan, X, Y, v, ctx->part, ctx->nblk, tl, ch);
      if (e == cudaSuccess && variant == 3 && !ch.on)
        e = eks::launch_chol(ctx->stream, t, ctx->Bg, v ? ctx->Bg + t * t : nullptr, ctx->Rm, ctx->Rinv,
                             v ? ctx->alpha : nullptr, ctx->flag, 0);
      return e;
    }
    if (use_seg) {
      cudaError_t e = eks::launch_spmm_seg(ctx->stream, t, ctx->n, ctx->seg, ctx->ell_w, X, Y, v, ctx->part, ctx->nblk,
                                           tl, ch);
      if (e == cudaSuccess && variant == 3 && !ch.on)
        e = eks::launch_chol(ctx->stream, t, ctx->Bg, v ? ctx->Bg + t * t : nullptr, ctx->Rm, ctx->Rinv,
                             v ? ctx->alpha : nullptr, ctx->flag, 0);
      return e;
    }
    cudaError_t e = use_ell ? eks::launch_spmm_gram_ell(ctx->stream, t, ctx->n, ctx->d_ecol, ctx->d_eval,
                                                           ctx->ell_w, ctx->d_tmax, ctx->n, X, 0, Y, v, ctx->part,
                                                           ctx->nblk, tl, ch)
                               : eks::launch_spmm_gram(ctx->stream, t, ctx->n, ctx->d_rp, ctx->d_col, ctx->d_val,
                                                       (int)ctx->maxrow, X, 0, Y, v, ctx->part, ctx->nblk, tl, ch);
    if (e == cudaSuccess && variant == 3 && !ch.on)
      e = eks::launch_chol(ctx->stream, t, ctx->Bg, v ? ctx->Bg + t * t : nullptr, ctx->Rm, ctx->Rinv,
                           v ? ctx->alpha : nullptr, ctx->flag, 0);
    return e;
  };
  CK(run());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  for (int i = 0; i < reps; ++i) CK(run());
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float f = 0.f;
  cudaEventElapsedTime(&f, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = (double)f / reps;
  return EKS_OK;
}

eks_status eks_k_last_basis(eks_ctx* ctx, int j, double* W, double* AW) {
  ST(check_ready(ctx));
  const int t = ctx->last_t, nb = ctx->last_nblocks, ring = ctx->last_ring;
  if (!W || t == 0 || j < 0 || j >= nb || (ring && j < nb - ring))
    return fail(ctx, EKS_ERR_INVALID_ARG, "basis block %d not resident (%d blocks built, ring %d)", j, nb, ring);
  const int idx = ring ? j % ring : j;
  if (idx >= (int)ctx->Wpool.size() || !ctx->Wpool[idx].base) return fail(ctx, EKS_ERR_INVALID_ARG, "no basis block %d", j);
  if (ctx->last_lazy) ST(materialize_w(ctx, t, idx, W));  // the slot holds Z2 and R⁻¹
  else CK(cudaMemcpyAsync(W, ctx->Wpool[idx].loc, sizeof(double) * ctx->n * t, cudaMemcpyDeviceToDevice, ctx->stream));
  if (AW && ctx->last_aq_off && !ring && j < nb - 2)
    return fail(ctx, EKS_ERR_INVALID_ARG, "A·W of block %d is not kept (store-Q-only solve: the last 2 blocks)", j);
  if (AW)
    CK(cudaMemcpyAsync(AW, ctx->AWpool[idx].loc, sizeof(double) * ctx->n * t, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return EKS_OK;
}

eks_status eks_k_last_residual(eks_ctx* ctx, double* r) {
  ST(check_ready(ctx));
  if (!r || !ctx->r) return fail(ctx, EKS_ERR_INVALID_ARG, "no residual (solve first)");
  CK(cudaMemcpyAsync(r, ctx->r, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return EKS_OK;
}

eks_status eks_k_chol(eks_ctx* ctx, int t, const double* B, double* R) {
  ST(k_ready(ctx, t));
  ST(reset_flag(ctx));
  ST(chol(ctx, t, B, nullptr, R, ctx->Rinv, nullptr, 0));
  ST(sync_scalars(ctx, 1));
  if (ctx->h_flag[1] != INT_MAX) return fail(ctx, EKS_ERR_BREAKDOWN, "Cholesky breakdown");
  return EKS_OK;
}

}  // extern "C"
