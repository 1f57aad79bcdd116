// FP64 FMA throughput microbenchmark (measured ALU peak for the "alu" roofline).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  int iters = 4096, blocks = sms * 8, threads = 256;
  k<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); k<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf("{\"fp64_fma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms, best);
  return 0;
}
