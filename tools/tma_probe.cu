// tma_probe.cu — bandwidth of a persistent-CTA ring of cp.async.bulk copies (global → shared,
// mbarrier completion) vs. copy size, stage count and copies per stage.  Diagnostic for the
// segment-staged SpMM: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   sa(b)),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b))
               : "memory");
}

// Each CTA streams its share of `total` bytes in stages of `per` copies of `csz` bytes.
__global__ void __launch_bounds__(288, 1) k_probe(const char* src, size_t total, int csz, int per, int NS,
                                                  double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const size_t SB = (size_t)csz * per;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * SB);
  uint64_t* empty = full + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nst = total / SB;  // stages in total
  const size_t my = nst > blockIdx.x ? (nst - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    for (size_t j = 0; j < my; ++j) {
      const int s = (int)(j % NS);
      if (j >= NS) mbar_wait(empty + s, (uint32_t)((j / NS - 1) & 1));
      const char* g = src + (blockIdx.x + j * gridDim.x) * SB;
      if (lane == 0) mbar_expect_tx(full + s, (uint32_t)SB);
      __syncwarp();
      for (int c = lane; c < per; c += 32) bulk(sm + s * SB + (size_t)c * csz, g + (size_t)c * csz, csz, full + s);
    }
    return;
  }
  double acc = 0.0;
  for (size_t j = 0; j < my; ++j) {
    const int s = (int)(j % NS);
    mbar_wait(full + s, (uint32_t)((j / NS) & 1));
    const double* d = reinterpret_cast<const double*>(sm + s * SB);
    for (size_t e = threadIdx.x; e < SB / 8; e += 256 * 8) acc += d[e];
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)8 << 30;  // 8 GB
  char* src;
  double* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int cs[] = {512, 2048, 8192, 32768};
  for (int csz : cs)
    for (int stage_kb : {16, 48}) {
      const int per = stage_kb * 1024 / csz;
      if (per < 1) continue;
      for (int NS : {2, 4}) {
        const size_t sb = (size_t)csz * per;
        if (NS * sb + 256 > 220 * 1024) continue;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_probe<<<sms, 288, NS * sb + 256>>>(src, total, csz, per, NS, sink);
        cudaEventRecord(a);
        for (int it = 0; it < 3; ++it) k_probe<<<sms, 288, NS * sb + 256>>>(src, total, csz, per, NS, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("copy %6d B x %3d per stage (%3d KB), NS=%d: %7.1f GB/s  %s\n", csz, per, stage_kb, NS,
               3.0 * total / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
