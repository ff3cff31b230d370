// chol_probe.cu — device-clock latency of the warp Cholesky (chol_warp_core) and of chained
// fp64 div / sqrt on one warp.  Diagnostic: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_1804_10629_b200/csrc
#include <cstdio>
#include "eks_device.cuh"

template <int T>
__global__ void k_probe(const double* B, double* out, long long* cyc) {
  double a[T], y[T];
  long long t0 = clock64();
  bool f = eks::chol_warp_core<T>(B, a, y);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < T; ++i) s += a[i] + y[i];
  out[threadIdx.x] = s + f;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  t0 = clock64();
  f = eks::chol_warp_fast<T>(B, a, y);
  t1 = clock64();
  s = 0;
  for (int i = 0; i < T; ++i) s += a[i] + y[i];
  out[100 + threadIdx.x] = s + f;
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // chained division and sqrt
  double x = B[0] + 1.0, z = 1.0;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) z = __ddiv_rn(x, z + 1.0);
  t1 = clock64();
  out[32 + threadIdx.x] = z;
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / 64;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) z = __dsqrt_rn(z + 2.0);
  t1 = clock64();
  out[64 + threadIdx.x] = z;
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / 64;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64();
  out[96 + threadIdx.x] = z;
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / 64;
}

template <int T>
void run() {
  double hB[T * T];
  for (int i = 0; i < T; ++i)
    for (int j = 0; j < T; ++j) hB[i * T + j] = (i == j ? T + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *B, *out;
  long long* cyc;
  cudaMalloc(&B, sizeof hB);
  cudaMalloc(&out, 160 * 8);
  cudaMalloc(&cyc, 5 * 8);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) k_probe<T><<<1, 32>>>(B, out, cyc);
  long long h[5];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  printf("T=%2d chol_warp_fast: %lld cycles\n", T, h[4]);
  printf("T=%2d chol_warp_core: %lld cycles; ddiv %lld, dsqrt %lld, shfl+add %lld cycles each (%s)\n", T, h[0], h[1],
         h[2], h[3], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<8>();
  run<16>();
  run<32>();
  return 0;
}
