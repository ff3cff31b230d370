// Micro-benchmark for the fp64 roofline denominators that MEASURED_PEAKS.json
// does not carry: DFMA (CUDA-core fp64 FMA) and DMMA (mma.sync .f64) throughput,
// plus an fp64 stream-read and copy bandwidth. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[4][2];
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DMMA and DFMA issued by the same warps: is the fp64 tensor path a separate pipe from the FMA pipe?
// Per iteration: 4 DMMA (4·512 flop per warp) and 32 DFMA per thread (32·2·32 = 2048 flop per warp).
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  double ma = 1.0 + threadIdx.x * 1e-9, mb = 1.0 - threadIdx.x * 1e-9;
  double c[4][2];
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(ma), "d"(mb));
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ x, size_t n2, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(x + i); s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ x, double2* __restrict__ y, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"clock_khz\": %d, \"mem_bytes\": %zu}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk, p.totalGlobalMem);
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 32 * 256));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 64 * iters * (double)blocks * threads;
      if (fl / (ms * 1e-3) > best) best = fl / (ms * 1e-3);
    }
    printf("{\"dfma_tflops\": %.3f}\n", best / 1e12);
  }
  // DMMA m8n8k4: 2*8*8*4 = 512 flop per warp-instruction
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    dmma_kernel<<<blocks, threads>>>(out, 16);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 512.0 * 4 * iters * (double)blocks * (threads / 32);
      if (fl / (ms * 1e-3) > best) best = fl / (ms * 1e-3);
    }
    printf("{\"dmma_tflops\": %.3f}\n", best / 1e12);
  }
  // DMMA + DFMA interleaved in the same warps
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    mixed_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); mixed_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = (512.0 * 4 + 2.0 * 32 * 32) * iters * (double)blocks * (threads / 32);
      if (fl / (ms * 1e-3) > best) best = fl / (ms * 1e-3);
    }
    printf("{\"mixed_dmma_dfma_tflops\": %.3f}\n", best / 1e12);
  }
  // fp64 read and copy bandwidth over 4 GiB
  {
    size_t bytes = (size_t)4 << 30; size_t n2 = bytes / 16;
    double2 *x, *y; CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&y, bytes));
    CK(cudaMemset(x, 0, bytes)); CK(cudaMemset(y, 0, bytes));
    int blocks = sms * 8, threads = 512;
    double bestr = 0, bestc = 0;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); read_kernel<<<blocks, threads>>>(x, n2, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      if (r && bytes / (ms * 1e-3) > bestr) bestr = bytes / (ms * 1e-3);
      cudaEventRecord(e0); copy_kernel<<<blocks, threads>>>(x, y, n2); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      if (r && 2.0 * bytes / (ms * 1e-3) > bestc) bestc = 2.0 * bytes / (ms * 1e-3);
    }
    printf("{\"read_gbs\": %.1f, \"copy_gbs\": %.1f}\n", bestr / 1e9, bestc / 1e9);
  }
  return 0;
}
