// Generic-grid path: the iteration on 7-smooth grid sizes n = 2^a 3^b 5^c 7^d (the paper's
// Table 1/2 sizes N = 300 ... 800) in 1-D and 2-D, one rank,
// correction form.  Same steps as the power-of-two path, with the spatial solves done by a
// mixed-radix Stockham FFT (radices 4, 2, 3, 5, 7) instead of PCR / the radix-16/32 engine:
//   (i)   resid_any_kernel:   X = alpha^{l/L} (w - C u)          (residual_point, modular wraps)
//   (ii)  tfft_fwd_kernel:    L-point DFT along time              (kernels.cu, T | N)
//   (iii) node_any_kernel:    x1 = S_p^{-1} x per frequency slot
//   (iv)  fft_any_kernel rows (+ columns), divide_any_kernel, inverse columns (+ rows):
//         x2 = F^{-1} [F x1 / (1 - d_km dT lambda)]  (A circulant: diagonal in Fourier)
//   (v)   node_any_kernel:    y = G_p^{-1} S_p x2; tfft_bwd_kernel: inverse DFT, unscale, u += c
// These grids are small (at most 800^2 points in the paper's tables): one CTA per line, all
// passes through shared memory; tuned for correctness and clarity, not for the HBM roof.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"
#include "internal.h"
#include "residual.cuh"

namespace pint {

namespace {

constexpr int kGenThreads = 256;

template <int M>
__global__ void __launch_bounds__(kGenThreads) resid_any_kernel(Geometry g, StaticTables st, AlphaTables at,
                                                                 const double2 *__restrict__ u,
                                                                 double2 *__restrict__ X) {
  const long long total = (long long)g.L * g.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(i / g.N), n = (int)(i - (long long)l * g.N);
    double2 r[M];
    residual_point<M, false, 3, false>(g, st, u, l, n, r);
    const double sc = __ldg(at.scale_fwd + l);   // alpha^{l/L} (J^{-1})
#pragma unroll
    for (int m = 0; m < M; ++m) X[((size_t)l * M + m) * g.N + n] = cscale(r[m], sc);
  }
}

// X[p][m][n] <- sum_j A[p][m][j] X[p][j][n] for every slot p and point n (in place)
template <int M>
__global__ void __launch_bounds__(kGenThreads) node_any_kernel(Geometry g, const double2 *__restrict__ A,
                                                                double2 *__restrict__ X) {
  const long long total = (long long)g.L * g.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(i / g.N), n = (int)(i - (long long)p * g.N);
    double2 *base = X + (size_t)p * M * g.N + n;
    const double2 *ap = A + (size_t)p * M * M;
    double2 v[M];
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = base[(size_t)j * g.N];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < M; ++j) acc = cfma(__ldg(ap + m * M + j), v[j], acc);
      base[(size_t)m * g.N] = acc;
    }
  }
}

// One Stockham pass of radix R over the n points of `src` into `dst` (shared memory): butterfly j
// reads src[j + t n/R], twiddles by w_{Ns R}^{t k} (k = j mod Ns), R-point DFT, writes
// dst[(j / Ns) Ns R + k + s Ns].  tw[q] = e^{-2 pi i q / n} (host long double, integer-reduced
// indices); INV conjugates every root.  Natural order in, natural order out after all passes.
template <int R, bool INV>
__device__ __forceinline__ void stockham_pass(const double2 *src, double2 *dst, int n, int Ns,
                                              const double2 *__restrict__ tw) {
  const int m = n / R;
  const int rstep = n / R;            // index step of the R-th roots of unity in tw
  const int twstep = n / (Ns * R);    // index step of the (Ns R)-th roots
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const int k = j % Ns;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      double2 x = src[j + t * m];
      if (t > 0 && k > 0) {
        double2 w = __ldg(tw + (long long)t * k * twstep % n);
        if (INV) w.y = -w.y;
        x = cmul(x, w);
      }
      v[t] = x;
    }
    const int o = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      double2 acc = v[0];
#pragma unroll
      for (int t = 1; t < R; ++t) {
        double2 w = __ldg(tw + ((t * s) % R) * rstep);
        if (INV) w.y = -w.y;
        acc = cfma(w, v[t], acc);
      }
      dst[o + s * Ns] = acc;
    }
  }
}

// One CTA per line.  Line i: element t at X[(i / lpp) pstride + (i % lpp) lstride + t es].
// fac: the radices of n (product = n), nf of them.  Unnormalised both ways.
template <bool INV>
__global__ void __launch_bounds__(kGenThreads) fft_any_kernel(double2 *__restrict__ X, int n, int es, int lpp,
                                                               long long lstride, long long pstride, int4 fac0,
                                                               int4 fac1, int nf, const double2 *__restrict__ tw) {
  extern __shared__ double2 smg[];
  double2 *a = smg, *b = smg + n;
  const int i = blockIdx.x;
  double2 *line = X + (size_t)(i / lpp) * pstride + (size_t)(i % lpp) * lstride;
  for (int t = threadIdx.x; t < n; t += blockDim.x) a[t] = line[(size_t)t * es];
  __syncthreads();
  const int f[8] = {fac0.x, fac0.y, fac0.z, fac0.w, fac1.x, fac1.y, fac1.z, fac1.w};
  int Ns = 1;
  for (int q = 0; q < nf; ++q) {
    const int R = f[q];
    switch (R) {
      case 2: stockham_pass<2, INV>(a, b, n, Ns, tw); break;
      case 3: stockham_pass<3, INV>(a, b, n, Ns, tw); break;
      case 4: stockham_pass<4, INV>(a, b, n, Ns, tw); break;
      case 5: stockham_pass<5, INV>(a, b, n, Ns, tw); break;
      default: stockham_pass<7, INV>(a, b, n, Ns, tw); break;
    }
    __syncthreads();
    double2 *tmp = a;
    a = b;
    b = tmp;
    Ns *= R;
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) line[(size_t)t * es] = a[t];
}

// x2 = x1 / ((1 - s_q (lambda_x(kx) + lambda_y(ky))) nx ny) on natural-order spectra
__global__ void __launch_bounds__(kGenThreads) divide_any_kernel(Geometry g, StaticTables st, AlphaTables at,
                                                                  double2 *__restrict__ X) {
  const long long total = (long long)g.L * g.M * g.N;
  const double inv_n = 1.0 / ((double)g.nx * (double)g.ny);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(i / g.N), n = (int)(i - (long long)q * g.N);
    const int kx = n % g.nx, ky = n / g.nx;
    const double2 s = __ldg(at.shift + q);
    const double2 lam = cadd(__ldg(st.lamx + kx), __ldg(st.lamy + ky));
    const double2 sl = cmul(s, lam);
    const double dr = 1.0 - sl.x, di = -sl.y;
    const double den = inv_n / (dr * dr + di * di);   // > 0 (|1 - s lambda| bounded below)
    X[i] = cmul(X[i], make_double2(dr * den, -di * den));
  }
}

int grid_for(long long items) {
  long long b = (items + kGenThreads - 1) / kGenThreads;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

bool radices(int n, int f[8], int &nf) {
  nf = 0;
  while (n % 4 == 0 && nf < 8) { f[nf++] = 4; n /= 4; }
  for (int r : {2, 3, 5, 7})
    while (n % r == 0 && nf < 8) { f[nf++] = r; n /= r; }
  return n == 1;
}

cudaError_t launch_fft_lines(double2 *X, int n, int es, int lpp, long long lstride, long long pstride, int lines,
                             bool inverse, const double2 *tw, cudaStream_t s) {
  int f[8] = {1, 1, 1, 1, 1, 1, 1, 1}, nf = 0;
  if (!radices(n, f, nf)) return cudaErrorInvalidValue;
  const size_t smem = 2 * (size_t)n * sizeof(double2);
  const void *fn = inverse ? (const void *)fft_any_kernel<true> : (const void *)fft_any_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int4 f0 = make_int4(f[0], f[1], f[2], f[3]), f1 = make_int4(f[4], f[5], f[6], f[7]);
  if (inverse)
    fft_any_kernel<true><<<lines, kGenThreads, smem, s>>>(X, n, es, lpp, lstride, pstride, f0, f1, nf, tw);
  else
    fft_any_kernel<false><<<lines, kGenThreads, smem, s>>>(X, n, es, lpp, lstride, pstride, f0, f1, nf, tw);
  record_launch(s);
  return cudaGetLastError();
}

}  // namespace

bool grid_is_smooth(long long n) {
  if (n < 1) return false;
  for (int r : {2, 3, 5, 7})
    while (n % r == 0) n /= r;
  return n == 1;
}

int generic_launches(const Geometry &g) { return g.dim == 2 ? 10 : 8; }

const char *generic_kernel_name(const Geometry &g, int i) {
  static const char *k1[] = {"resid_any_kernel", "tfft_fwd_kernel", "node_any_kernel<Sinv>", "fft_any_kernel<fwd x>",
                             "divide_any_kernel", "fft_any_kernel<inv x>", "node_any_kernel<SG>", "tfft_bwd_kernel"};
  static const char *k2[] = {"resid_any_kernel", "tfft_fwd_kernel", "node_any_kernel<Sinv>", "fft_any_kernel<fwd x>",
                             "fft_any_kernel<fwd y>", "divide_any_kernel", "fft_any_kernel<inv y>",
                             "fft_any_kernel<inv x>", "node_any_kernel<SG>", "tfft_bwd_kernel"};
  if (i < 0 || i >= generic_launches(g)) return "";
  return g.dim == 2 ? k2[i] : k1[i];
}

cudaError_t launch_generic_residual(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                                    const double2 *u, double2 *X, cudaStream_t s) {
  const int grid = grid_for((long long)g.L * g.N);
#define PINT_RANY(MM) resid_any_kernel<MM><<<grid, kGenThreads, 0, s>>>(g, st, at, u, X)
  switch (g.M) {
    case 1: PINT_RANY(1); break;
    case 2: PINT_RANY(2); break;
    case 3: PINT_RANY(3); break;
    case 4: PINT_RANY(4); break;
    case 5: PINT_RANY(5); break;
    case 6: PINT_RANY(6); break;
    case 7: PINT_RANY(7); break;
    default: PINT_RANY(8); break;
  }
#undef PINT_RANY
  record_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_generic_solve(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                                 cudaStream_t s) {
  const int grid = grid_for((long long)g.L * g.N);
  auto node = [&](const double2 *A) -> cudaError_t {
#define PINT_NANY(MM) node_any_kernel<MM><<<grid, kGenThreads, 0, s>>>(g, A, X)
    switch (g.M) {
      case 1: PINT_NANY(1); break;
      case 2: PINT_NANY(2); break;
      case 3: PINT_NANY(3); break;
      case 4: PINT_NANY(4); break;
      case 5: PINT_NANY(5); break;
      case 6: PINT_NANY(6); break;
      case 7: PINT_NANY(7); break;
      default: PINT_NANY(8); break;
    }
#undef PINT_NANY
    record_launch(s);
    return cudaGetLastError();
  };
  const int planes = g.L * g.M;
  cudaError_t e;
  if ((e = node(at.Sinv)) != cudaSuccess) return e;   // x1 = S_p^{-1} x
  // rows: line (plane, y) at plane N + y nx, contiguous; columns: (plane, x) at plane N + x, stride nx
  if ((e = launch_fft_lines(X, g.nx, 1, g.ny, g.nx, g.N, planes * g.ny, false, st.twx, s)) != cudaSuccess) return e;
  if (g.dim == 2 &&
      (e = launch_fft_lines(X, g.ny, g.nx, g.nx, 1, g.N, planes * g.nx, false, st.twy, s)) != cudaSuccess)
    return e;
  divide_any_kernel<<<grid_for((long long)planes * g.N), kGenThreads, 0, s>>>(g, st, at, X);
  record_launch(s);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (g.dim == 2 &&
      (e = launch_fft_lines(X, g.ny, g.nx, g.nx, 1, g.N, planes * g.nx, true, st.twy, s)) != cudaSuccess)
    return e;
  if ((e = launch_fft_lines(X, g.nx, 1, g.ny, g.nx, g.N, planes * g.ny, true, st.twx, s)) != cudaSuccess) return e;
  return node(at.SG);                                  // y = G_p^{-1} S_p x2
}

}  // namespace pint
