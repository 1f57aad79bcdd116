// Memory-system microbenchmarks that decide the 2-D tile shapes:
//  (1) strided-segment copy: R rows of N complex128 each; CTA b copies columns [b T, (b+1) T) of
//      every row (the access pattern of an all-l x all-m time tile), T = 1, 2, 4, 8 -> segment
//      bytes 16 T.  Reports read+write GB/s.
//  (2) L2-resident read+write bandwidth: the same copy on a footprint that fits in L2, repeated.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void seg_copy(const double2 *__restrict__ src, double2 *__restrict__ dst, int rows, int N, int T) {
  const int n0 = blockIdx.x * T;
  const int items = rows * T;
  for (int base = threadIdx.x; base < items; base += 8 * blockDim.x) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int it = base + k * blockDim.x;
      if (it < items) {
        const int t = it % T, r = it / T;
        v[k] = __ldg(src + (size_t)r * N + n0 + t);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int it = base + k * blockDim.x;
      if (it < items) {
        const int t = it % T, r = it / T;
        dst[(size_t)r * N + n0 + t] = v[k];
      }
    }
  }
}

__global__ void lin_copy(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      dst[i] = __ldg(src + i);
}

int main() {
  const int rows = 2048;
  const int N = 1 << 20;       // 2048 x 1M x 16 B = 32 GiB per array... use 1/4: N = 256K
  const int Nn = N / 4;
  const size_t elems = (size_t)rows * Nn;
  double2 *a, *b;
  if (cudaMalloc(&a, elems * sizeof(double2)) != cudaSuccess || cudaMalloc(&b, elems * sizeof(double2)) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 0, elems * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"seg_copy\": {");
  for (int T = 1; T <= 16; T *= 2) {
    for (int thr = 256; thr <= 512; thr *= 2) {
      seg_copy<<<Nn / T, thr>>>(a, b, rows, Nn, T);
      float best = 1e9f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        seg_copy<<<Nn / T, thr>>>(a, b, rows, Nn, T);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%s\"T%d_thr%d_GBs\": %.1f", (T == 1 && thr == 256) ? "" : ", ", T, thr,
             2.0 * elems * sizeof(double2) / best / 1e6);
    }
  }
  printf("}, \"l2_copy\": {");
  for (int mb = 16; mb <= 128; mb *= 2) {
    const size_t n = ((size_t)mb << 20) / sizeof(double2) / 2;   // src + dst = mb MiB
    lin_copy<<<148 * 8, 256>>>(a, b, n, 2);
    float best = 1e9f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      lin_copy<<<148 * 8, 256>>>(a, b, n, 20);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%s\"%dMiB_GBs\": %.1f", mb == 16 ? "" : ", ", mb, 2.0 * 20 * n * sizeof(double2) / best / 1e6);
  }
  {
    const size_t n = elems;
    float best = 1e9f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      lin_copy<<<148 * 8, 256>>>(a, b, n, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf(", \"hbm_linear_GBs\": %.1f", 2.0 * n * sizeof(double2) / best / 1e6);
  }
  printf("}}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
