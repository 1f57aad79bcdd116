// The residual of step (i) at one point (north star (i)): r[m] = (w - C u)[l][m][n]
// for all M nodes, shared by the time-tile kernels (kernels.cu) and the generic-grid path
// (generic.cu).
#pragma once
#include "device_common.cuh"
#include "internal.h"

namespace pint {

// H-term source (last node of the previous global step) of local step l at point n
__device__ __forceinline__ double2 prev_value(const StaticTables &st, int l, int n) {
  const int jj = l - st.prev_shift;
  return jj < 0 ? __ldg(st.u0 + n) : __ldg(st.prev_base + (long long)jj * st.prev_stride + n);
}

// Hermitian (packed) mode stores the iterate as real fp64 u[l][m][n] in the first L M N doubles
// of u_dev (its imaginary parts are zero in exact arithmetic)
__device__ __forceinline__ double2 u_at(const double2 *__restrict__ u, size_t i, bool real) {
  return real ? make_double2(__ldg((const double *)u + i), 0.0) : __ldg(u + i);
}

// P2 = false: any grid (the 7-smooth non-power-of-two sizes of Tables 1-2): modular wraps
template <int M, bool REAL = false, int HW = 3, bool P2 = true>
__device__ __forceinline__ void residual_point(const Geometry &g, const StaticTables &st,
                                               const double2 *__restrict__ u, int l, int n, double2 r[M]) {
  constexpr bool real = REAL;   // Hermitian mode: real storage (st.packed)
  const size_t plane = (size_t)M * g.N;
  const size_t ul = (size_t)l * plane;
  const int x = P2 ? (n & (g.nx - 1)) : n % g.nx;
  const int y = P2 ? (n >> g.lognx) : n / g.nx;
  const int row = P2 ? (y << g.lognx) : y * g.nx;
  double2 uc[M], Au[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const size_t uj = ul + (size_t)j * g.N;
    const double2 c = u_at(u, uj + n, real);
    uc[j] = c;
    double2 s = make_double2(g.wx[3] * c.x, g.wx[3] * c.y);
    // unrolled over the halo HW (1: the 3-point operators, whose missing offsets carry weight 0;
    // 3: any stencil, offsets outside [-h0, h1] skipped by uniform predicates)
#pragma unroll
    for (int o = -HW; o <= HW; ++o) {
      if (o == 0 || (HW > 1 && (o < -g.hx0 || o > g.hx1))) continue;
      const double2 v = u_at(u, uj + row + (P2 ? ((x + o) & (g.nx - 1)) : (x + o + g.nx) % g.nx), real);
      s.x = fma(g.wx[3 + o], v.x, s.x);
      s.y = fma(g.wx[3 + o], v.y, s.y);
    }
    if (g.dim == 2) {
#pragma unroll
      for (int o = -HW; o <= HW; ++o) {
        if (o == 0 || (HW > 1 && (o < -g.hy0 || o > g.hy1))) continue;
        const double2 v = u_at(u, uj + (P2 ? ((((y + o) & (g.ny - 1)) << g.lognx) + x)
                                             : (size_t)((y + o + g.ny) % g.ny) * g.nx + x), real);
        s.x = fma(g.wy[3 + o], v.x, s.x);
        s.y = fma(g.wy[3 + o], v.y, s.y);
      }
    }
    Au[j] = s;
  }
  // w (global l = 0) or the H-term u_{l-1, M-1} (real storage: one rank, previous local step)
  const double2 base = real ? (l == 0 ? __ldg(st.u0 + n) : u_at(u, ul - g.N + n, true)) : prev_value(st, l, n);
#pragma unroll
  for (int m = 0; m < M; ++m) {
    double2 acc = csub(base, uc[m]);
    if (st.v) acc = cadd(acc, __ldg(st.v + ((size_t)l * M + m) * g.N + n));   // forcing part of w
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double q = g.dTQ[m * M + j];
      acc.x = fma(q, Au[j].x, acc.x);
      acc.y = fma(q, Au[j].y, acc.y);
    }
    r[m] = acc;
  }
}

}  // namespace pint
