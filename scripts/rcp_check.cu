// Accuracy of the spectral divide's reciprocal (device_common.cuh rcp_pos) against 1.0 / q over
// q in [1e-7, 1e4] (log-uniform) : max relative error and max ulp distance.
#include <cstdio>
#include <cmath>
#include <cstdint>
#include "../paper_2103_12571_b200/csrc/device_common.cuh"

using namespace pint;
__global__ void k(double *out_rel, unsigned long long *out_ulp, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double q = exp(log(1e-7) + (log(1e4) - log(1e-7)) * (i + 0.5) / n);
  const double a = rcp_pos(q), b = 1.0 / q;
  out_rel[i] = fabs(a - b) / b;
  long long d = __double_as_longlong(a) - __double_as_longlong(b);
  out_ulp[i] = (unsigned long long)(d < 0 ? -d : d);
}

int main() {
  const int n = 1 << 24;
  double *r; unsigned long long *u;
  cudaMallocManaged(&r, n * sizeof(double));
  cudaMallocManaged(&u, n * sizeof(unsigned long long));
  k<<<n / 256, 256>>>(r, u, n);
  cudaDeviceSynchronize();
  double mr = 0; unsigned long long mu = 0;
  for (int i = 0; i < n; ++i) { if (r[i] > mr) mr = r[i]; if (u[i] > mu) mu = u[i]; }
  printf("rcp_pos: max rel err %.3e, max ulp %llu over %d samples\n", mr, mu, n);
  return mr < 1e-15 ? 0 : 1;
}
