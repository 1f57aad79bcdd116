// 2-D spatial solves (north star step (iv), Alg. 1) on the register FFT
// engine of fft_reg.cuh.
//
// Spatial solves: for every line q = (slot p, node m) x2 = F^{-1}[F x1 / (1 - s_q lambda)] as
// three plane passes over the frequency batch of slot p (all M nodes):
//   R  rows:    x1 = S_p^{-1} x (node transform in shared memory), x-DIF; spectral rows
//               stored in the S-layout of fft_reg.cuh (coalesced)
//   C  columns: y-DIF, x2 = x1 / ((1 - s_q (lambda_x + lambda_y)) nx ny), y-DIT, in registers
//   I  rows:    x-DIT, y = G_p^{-1} S_p x2 applied while copying the rows out
// run as ONE persistent kernel that software-pipelines the batches (round j: R(j), C(j-1),
// I(j-2)) so intermediate planes are re-read while they are still in L2.
//
// Work distribution: the global item sequence (round by round, stage segments in the order
// R, C, I) is claimed item by item from one device counter by the co-resident CTAs of a
// cooperative launch (the next claim is issued when an item starts and read when it ends).  An
// item of C(b) waits until all items of R(b) have been counted done (I(b): all of C(b)); every
// dependency points to an item that comes earlier in the sequence, already claimed by a running
// CTA, so the earliest unfinished item can always run (no deadlock while all CTAs are resident,
// which the cooperative launch guarantees).  Producers publish with bar.sync +
// red.release.gpu; consumers acquire with ld.acquire.gpu and then load with cp.async.cg /
// ld.global.cg (L2; never a stale L1 line).
//
// Direct form (Alg. 1 as printed): the C stage synthesizes its input spectrum sig_q * r0hat (no
// R stage); see launch_direct_front in kernels.cu.
//
// Units: st.slots[0 .. nsolve) (every slot; Hermitian mode: the L/2 + 1 slots with k <= L/2,
// whose R stage unpacks X_k from the packed real-data spectra Z_k, Z_{L-k} and whose planes live in
// the unit area of X, internal.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "device_common.cuh"
#include "fft_reg.cuh"
#include "internal.h"

namespace pint {

namespace {

constexpr int kSpThreads = 256;
enum { kStR = 0, kStC = 1, kStI = 2 };

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_cg(const double2 *p) {
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void wait_count(const unsigned *ctr, unsigned need) {
  if (threadIdx.x == 0) {
    while (ld_acquire_gpu(ctr) < need) __nanosleep(64);
  }
  __syncthreads();
}

// all threads' stores of the item are ordered before the barrier; thread 0's release-add makes
// them visible at gpu scope to the consumer that acquires the counter (PTX release/acquire)
__device__ __forceinline__ void publish(unsigned *ctr) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
}

__device__ __forceinline__ void copy_table(double2 *dst, const double2 *src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

// 1 / ((1 - s lambda) nx ny) for natural frequencies (kx, ky)
__device__ __forceinline__ double2 inv_symbol(const StaticTables &st, double2 s, double inv_n, int kx, int ky) {
  const double2 lam = cadd(__ldg(st.lamx + kx), __ldg(st.lamy + ky));
  const double2 sl = cmul(s, lam);
  const double dr = 1.0 - sl.x, di = -sl.y;
  const double q = dr * dr + di * di;   // > 0: |1 - s lambda| >= 7.7e-4 on every config
  double rq = __drcp_rn(q);
  rq = fma(rq, fma(-q, rq, 1.0), rq);
  const double den = inv_n * rq;
  return make_double2(dr * den, -di * den);   // conj(1 - s lambda) / |1 - s lambda|^2 / (nx ny)
}

// M x M complex matvec over the M lines (stride ls) of every column x of `rows` rows in shared
// memory: v_m <- sum_j A[m][j] v_j (A row-major in shared memory, compile-time M; the A reads
// are warp-uniform broadcasts, issued inside the loop so they do not pin M^2 registers)
template <class PX, int MM>
__device__ __forceinline__ void node_transform_m(double2 *sm, int ls, int rows, const double2 *A) {
  constexpr int LX = PX::LOGN, NX = 1 << LX;
  double2 ar[MM <= 4 ? MM * MM : 1];   // M <= 4: A in registers (nothing else is live here)
  if constexpr (MM <= 4) {
#pragma unroll
    for (int i = 0; i < MM * MM; ++i) ar[i] = A[i];
  }
  for (int i = threadIdx.x; i < rows * NX; i += blockDim.x) {
    const int x = i & (NX - 1), r = i >> LX;
    double2 *base = sm + (size_t)r * MM * ls + rfft::F<PX>(x);
    double2 v[MM];
#pragma unroll
    for (int j = 0; j < MM; ++j) v[j] = base[j * ls];
#pragma unroll (MM <= 4 ? MM : 1)
    for (int m = 0; m < MM; ++m) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < MM; ++j) {
        double2 a;
        if constexpr (MM <= 4) {
          a = ar[m * MM + j];
        } else {
          const volatile double2 *av = (const volatile double2 *)(A + m * MM + j);
          a = make_double2(av->x, av->y);
        }
        acc = cfma(a, v[j], acc);
      }
      base[m * ls] = acc;
    }
  }
}
template <class PX>
__device__ __forceinline__ void node_transform(double2 *sm, int ls, int M, int rows, const double2 *A) {
  switch (M) {
    case 1: node_transform_m<PX, 1>(sm, ls, rows, A); break;
    case 2: node_transform_m<PX, 2>(sm, ls, rows, A); break;
    case 3: node_transform_m<PX, 3>(sm, ls, rows, A); break;
    case 4: node_transform_m<PX, 4>(sm, ls, rows, A); break;
    case 5: node_transform_m<PX, 5>(sm, ls, rows, A); break;
    case 6: node_transform_m<PX, 6>(sm, ls, rows, A); break;
    case 7: node_transform_m<PX, 7>(sm, ls, rows, A); break;
    default: node_transform_m<PX, 8>(sm, ls, rows, A); break;
  }
}

// Copy-out of the I item with the node matrix applied: for every (row yy, column x) the M lines'
// values (tile[(yy M + j) NX + F(x)]) -> out_m = sum_j A[m][j] v_j -> xp[m N + (y0 + yy) NX + x].
// A (M x M, shared memory) is held in registers for M <= 4 (the FFT's registers are free here).
template <class PX, int MM>
__device__ __forceinline__ void node_copyout(const double2 *tile, const double2 *A, int YR,
                                             double2 *__restrict__ xp, int N, int y0) {
  constexpr int LX = PX::LOGN, NX = 1 << LX;
  double2 ar[MM <= 4 ? MM * MM : 1];
  if constexpr (MM <= 4) {
#pragma unroll
    for (int i = 0; i < MM * MM; ++i) ar[i] = A[i];
  }
  for (int i = threadIdx.x; i < YR * NX; i += blockDim.x) {
    const int x = i & (NX - 1), yy = i >> LX;
    const double2 *base = tile + (size_t)yy * MM * NX + rfft::F<PX>(x);
    double2 v[MM];
#pragma unroll
    for (int j = 0; j < MM; ++j) v[j] = base[j * NX];
    double2 *dst = xp + ((size_t)(y0 + yy) << LX) + x;
#pragma unroll (MM <= 4 ? MM : 1)
    for (int m = 0; m < MM; ++m) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < MM; ++j) {
        double2 a;
        if constexpr (MM <= 4) {
          a = ar[m * MM + j];
        } else {
          const volatile double2 *av = (const volatile double2 *)(A + m * MM + j);
          a = make_double2(av->x, av->y);
        }
        acc = cfma(a, v[j], acc);
      }
      dst[(size_t)m * N] = acc;
    }
  }
}

// ---- R item: rows y0 .. y0 + YR - 1 of slot p, all M nodes ---------------------------------
template <class PX>
__device__ __forceinline__ void r_item(const Geometry &g, const AlphaTables &at, double2 *tile, double2 *nt,
                                       const double2 *twx, double2 *__restrict__ xp, int p, int y0, int YR,
                                       bool node, const double2 *__restrict__ za, const double2 *__restrict__ zb) {
  constexpr int LX = PX::LOGN, NX = PX::N;
  const int M = g.M, nl = M * YR;
  if (za) {
    // Hermitian (packed) mode: unpack X_k from Z_k = za, Z_{L-k} = zb ([m][N/2] each):
    // top half rows X_k = (Z_k + conj Z_{L-k}) / 2, bottom half X_k = (Z_k - conj Z_{L-k}) / 2i;
    // za == zb (k = 0, L/2): X_k = Re Z_k (top), Im Z_k (bottom)
    const int hy = g.ny / 2;
    constexpr int kL = 4;   // loads batched for memory-level parallelism
    for (int i0 = threadIdx.x; i0 < nl * NX; i0 += kL * blockDim.x) {
      double2 a[kL], b[kL];
#pragma unroll
      for (int k = 0; k < kL; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < nl * NX) {
          const int x = i & (NX - 1), l = i >> LX;
          const int yy = l / M, m = l - yy * M;
          const int y = y0 + yy;
          const size_t off = (size_t)m * (g.N / 2) + ((size_t)(y < hy ? y : y - hy) << LX) + x;
          a[k] = __ldg(za + off);
          b[k] = __ldg(zb + off);
        }
      }
#pragma unroll
      for (int k = 0; k < kL; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < nl * NX) {
          const int x = i & (NX - 1), l = i >> LX;
          const int top = y0 + l / M < hy;
          double2 v;
          if (za == zb) v = top ? make_double2(a[k].x, 0.0) : make_double2(a[k].y, 0.0);
          else if (top) v = make_double2(0.5 * (a[k].x + b[k].x), 0.5 * (a[k].y - b[k].y));
          else v = make_double2(0.5 * (a[k].y + b[k].y), 0.5 * (b[k].x - a[k].x));   // (a - conj b) / (2i)
          tile[(size_t)l * NX + rfft::F<PX>(x)] = v;
        }
      }
    }
  } else if (NX >= kSpThreads) {
    for (int l = 0; l < nl; ++l) {   // line-major: the (row, node) split once per line
      const int yy = l / M, m = l - yy * M;
      const double2 *src = xp + (size_t)m * g.N + ((size_t)(y0 + yy) << LX);
      double2 *dst = tile + (size_t)l * NX;
      for (int x = threadIdx.x; x < NX; x += kSpThreads) cp_async16(dst + rfft::F<PX>(x), src + x);
    }
  } else {
    for (int i = threadIdx.x; i < nl * NX; i += blockDim.x) {
      const int x = i & (NX - 1), l = i >> LX;
      const int yy = l / M, m = l - yy * M;
      cp_async16(tile + (size_t)l * NX + rfft::F<PX>(x), xp + (size_t)m * g.N + ((size_t)(y0 + yy) << LX) + x);
    }
  }
  if (node && threadIdx.x < M * M) nt[threadIdx.x] = __ldg(at.Sinv + (size_t)p * M * M + threadIdx.x);
  cp_async_wait_all();
  __syncthreads();
  if (node) {
    node_transform<PX>(tile, NX, M, YR, nt);
    __syncthreads();
  }
  const int l = threadIdx.x / PX::TPL, tau = threadIdx.x - l * PX::TPL;
  // warps without a line skip; surplus lanes of a partly used warp (TPL < 32) run on the dummy
  // line nl (never read back, never stored) so that their exchanges cannot touch a real line
  if ((int)(threadIdx.x & ~31) / PX::TPL >= nl) return;
  const int lc = l < nl ? l : nl;
  double2 v[PX::E];
  rfft::forward_from_smem<PX>(v, tile + (size_t)lc * NX, lc, tau, twx);
  if (l < nl) {
    const int yy = l / M, m = l - yy * M;
    double2 *dst = xp + (size_t)m * g.N + ((size_t)(y0 + yy) << LX);
    constexpr int R = 1 << PX::BL;
#pragma unroll
    for (int u = 0; u < PX::E / R; ++u)
#pragma unroll
      for (int t = 0; t < R; ++t) dst[rfft::s_slot<PX>(tau, u, t)] = v[u * R + t];
  }
}

// ---- I item: inverse rows ------------------------------------------------------------------
template <class PX>
__device__ __forceinline__ void i_item(const Geometry &g, const AlphaTables &at, double2 *tile, double2 *nt,
                                       const double2 *twx, double2 *__restrict__ xp, int p, int y0, int YR,
                                       bool node) {
  constexpr int LX = PX::LOGN, NX = PX::N;
  constexpr int R = 1 << PX::BL;
  const int M = g.M, nl = M * YR;
  const int l = threadIdx.x / PX::TPL, tau = threadIdx.x - l * PX::TPL;
  const bool wrun = (int)(threadIdx.x & ~31) / PX::TPL < nl;   // warp holds at least one line
  const int lc = l < nl ? l : nl;                                 // nl: dummy line (see r_item)
  const int ls_ = l < nl ? l : nl - 1;                            // line whose data the loads read
  const int yy = ls_ / M, m = ls_ - yy * M;
  const double2 *src = xp + (size_t)m * g.N + ((size_t)(y0 + yy) << LX);
  double2 v[PX::E];
#pragma unroll
  for (int u = 0; u < PX::E / R; ++u)
#pragma unroll
    for (int t = 0; t < R; ++t) v[u * R + t] = ld_cg(src + rfft::s_slot<PX>(tau, u, t));
  double2 *line = tile + (size_t)lc * NX;
  if (wrun) {
    rfft::inverse_in_regs<PX>(v, line, lc, tau, twx);
    if (l < nl) rfft::to_smem<PX, 0>(v, line, tau);
  }
  if (node && threadIdx.x < M * M) nt[threadIdx.x] = __ldg(at.SG + (size_t)p * M * M + threadIdx.x);
  __syncthreads();
  if (node) {   // y = G_p^{-1} S_p x2 applied on the way out (one smem pass and barrier fewer)
    switch (M) {
      case 1: node_copyout<PX, 1>(tile, nt, YR, xp, g.N, y0); break;
      case 2: node_copyout<PX, 2>(tile, nt, YR, xp, g.N, y0); break;
      case 3: node_copyout<PX, 3>(tile, nt, YR, xp, g.N, y0); break;
      case 4: node_copyout<PX, 4>(tile, nt, YR, xp, g.N, y0); break;
      case 5: node_copyout<PX, 5>(tile, nt, YR, xp, g.N, y0); break;
      case 6: node_copyout<PX, 6>(tile, nt, YR, xp, g.N, y0); break;
      case 7: node_copyout<PX, 7>(tile, nt, YR, xp, g.N, y0); break;
      default: node_copyout<PX, 8>(tile, nt, YR, xp, g.N, y0); break;
    }
    return;
  }
  for (int i = threadIdx.x; i < nl * NX; i += blockDim.x) {
    const int x = i & (NX - 1), li = i >> LX;
    const int y2 = li / M, m2 = li - y2 * M;
    xp[(size_t)m2 * g.N + ((size_t)(y0 + y2) << LX) + x] = tile[(size_t)li * NX + rfft::F<PX>(x)];
  }
}

// ---- C item: columns (S-slots) kx0 .. kx0 + TC - 1 of line q -----------------------------------
template <class PX, class PY>
__device__ __forceinline__ void c_item(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                                       double2 *tile, const double2 *twy, double2 *__restrict__ xl,
                                       const double2 *__restrict__ spec, int q, int kx0, int TC) {
  constexpr int LX = PX::LOGN, LY = PY::LOGN;
  constexpr int NX = 1 << LX, NY = PY::N;
  constexpr int R = 1 << PY::BL;
  const int pad = TC >= 8 ? 1 : 8 / TC;
  const int ls = NY + pad;
  const int lT = 31 - __clz(TC);
  const int l = threadIdx.x / PY::TPL, tau = threadIdx.x - l * PY::TPL;
  const bool wrun = (int)(threadIdx.x & ~31) / PY::TPL < TC;   // warp holds at least one column
  const int lc = l < TC ? l : TC;                                 // TC: dummy line (see r_item)
  double2 *line = tile + (size_t)lc * ls;
  const double2 s = __ldg(at.shift + q);
  const double inv_n = 1.0 / ((double)NX * (double)NY);
  const int pxs = rfft::slot_to_pos<PX>(kx0 + (l < TC ? l : TC - 1));   // x position of the column (S-slot)
  const int kx = brev(pxs, LX);
  double2 v[PY::E];
  if (spec) {
    // direct form: x1 spectrum = sig_q * r0hat, r0hat[py][px] in position order (P -> bitrev(P))
    const double2 sg = __ldg(at.sig + q);
#pragma unroll
    for (int u = 0; u < PY::E / R; ++u)
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int P = rfft::last_pos<PY>(tau, u, t);
        const double2 w = cmul(sg, __ldg(spec + ((size_t)P << LX) + pxs));
        v[u * R + t] = cmul(w, inv_symbol(st, s, inv_n, kx, brev(P, LY)));
      }
  } else {
    for (int i = threadIdx.x; i < TC * NY; i += blockDim.x) {
      const int c = i & (TC - 1), y = i >> lT;
      cp_async16(tile + (size_t)c * ls + rfft::F<PY>(y), xl + ((size_t)y << LX) + kx0 + c);
    }
    cp_async_wait_all();
    __syncthreads();
    if (wrun) {
      rfft::forward_from_smem<PY>(v, line, lc, tau, twy);
#pragma unroll
      for (int u = 0; u < PY::E / R; ++u)
#pragma unroll
        for (int t = 0; t < R; ++t) {
          const int P = rfft::last_pos<PY>(tau, u, t);
          v[u * R + t] = cmul(v[u * R + t], inv_symbol(st, s, inv_n, kx, brev(P, LY)));
        }
    }
  }
  if (wrun) {
    rfft::inverse_in_regs<PY>(v, line, lc, tau, twy);
    if (l < TC) rfft::to_smem<PY, 0>(v, line, tau);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TC * NY; i += blockDim.x) {
    const int c = i & (TC - 1), y = i >> lT;
    xl[((size_t)y << LX) + kx0 + c] = tile[(size_t)c * ls + rfft::F<PY>(y)];
  }
}

}  // namespace

template <int LX, int LY, int MB>
__global__ void __launch_bounds__(kSpThreads, MB == 4 ? 2 : 1)
    spatial2d_kernel(const Geometry g, StaticTables st, AlphaTables at, SpatialPlan sp, double2 *__restrict__ X,
                     const double2 *__restrict__ spec, unsigned *__restrict__ sync) {
  using PX = rfft::Plan<LX, MB>;
  using PY = rfft::Plan<LY, MB>;
  extern __shared__ double2 sm[];
  constexpr int TWX = PX::twsize(), TWY = PY::twsize();
  double2 *twx = sm, *twy = sm + TWX, *nt = sm + TWX + TWY, *tile = nt + 64;   // nt: M x M node table
  copy_table(twx, st.ptwx, TWX);
  copy_table(twy, st.ptwy, TWY);
  __syncthreads();
  const int riPerBatch = g.ny / sp.YR, cPerLine = g.nx / sp.TC;
  const bool node = st.P == 1;   // P > 1: the node transforms live in the cross-rank DFT kernels
  const int first = sp.synth ? kStC : kStR;
  // Items are claimed dynamically in sequence order (round j: the active stage segments, stage
  // index si works on batch j - si; R(j), C(j-1), I(j-2)) from one device counter.  Every item
  // depends only on items of earlier rounds (lower sequence numbers), all of which were claimed
  // before it by CTAs that are running (cooperative launch), so the waits cannot deadlock.  The
  // next claim is issued at the start of an item and consumed at its end (latency hidden).
  unsigned *claim = sync + 3 * sp.nbatch;
  __shared__ unsigned s_next[2];   // double-buffered: consecutive items use alternate slots
  auto round_count = [&](int j) {
    const int slo = j - (sp.nbatch - 1) > 0 ? j - (sp.nbatch - 1) : 0;
    const int shi = j < sp.nstage - 1 ? j : sp.nstage - 1;
    int rn = 0;
    for (int si = slo; si <= shi; ++si) rn += (first + si == kStC) ? sp.nC : sp.nRI;
    return rn;
  };
  if (threadIdx.x == 0) s_next[0] = sp.claim ? atomicAdd(claim, 1u) : blockIdx.x;
  __syncthreads();
  unsigned t = s_next[0];
  int par = 1;
  int j = 0;
  long long rs = 0;            // sequence number of round j's first item
  int rn = round_count(0);
  for (;;) {
    while (j < sp.rounds && (long long)t >= rs + rn) {
      rs += rn;
      ++j;
      if (j < sp.rounds) rn = round_count(j);
    }
    if (j >= sp.rounds) break;
    unsigned nxt = 0;
    if (threadIdx.x == 0) nxt = sp.claim ? atomicAdd(claim, 1u) : t + gridDim.x;   // static: t = cta mod G
    const int slo = j - (sp.nbatch - 1) > 0 ? j - (sp.nbatch - 1) : 0;
    {
      const int k = (int)((long long)t - rs);
      int si = slo, kk = k;
      for (;;) {
        const int n = (first + si == kStC) ? sp.nC : sp.nRI;
        if (kk < n) break;
        kk -= n;
        ++si;
      }
      const int stage = first + si, b = j - si;
      if ((sp.skip >> stage) & 1) {
        // timing experiments only (PINT_SP_SKIP): the stage's items do no work
      } else if (stage == kStC) {
        if (!sp.synth) wait_count(sync + kStR * sp.nbatch + b, (unsigned)sp.nRI);
        const int li = kk / cPerLine;                       // line within the batch
        const int un = b * sp.B + li / g.M, m = li % g.M;   // unit, node
        const int q = __ldg(st.slots + un) * g.M + m;       // table line (slot, node)
        double2 *plane = (st.packed ? unit_planes(g, X) + (size_t)un * g.M * g.N : X + (size_t)q / g.M * g.M * g.N) +
                         (size_t)m * g.N;
        c_item<PX, PY>(g, st, at, tile, twy, plane, sp.synth ? spec : nullptr, q, (kk - li * cPerLine) * sp.TC, sp.TC);
      } else {
        if (stage == kStI) wait_count(sync + kStC * sp.nbatch + b, (unsigned)sp.nC);
        const int pi = kk / riPerBatch;                     // slot within the batch
        const int y0 = (kk - pi * riPerBatch) * sp.YR;
        const int un = b * sp.B + pi;                       // unit
        const int slot = __ldg(st.slots + un);
        double2 *xp = st.packed ? unit_planes(g, X) + (size_t)un * g.M * g.N : X + (size_t)slot * g.M * g.N;
        if (stage == kStR) {
          const double2 *za = nullptr, *zb = nullptr;
          if (st.packed) {   // Z_k and Z_{L-k} (slot of the conjugate frequency) in the packed first half
            const int k = brev(slot, g.logL), pc = brev((g.L - k) & (g.L - 1), g.logL);
            za = X + (size_t)slot * g.M * (g.N / 2);
            zb = X + (size_t)pc * g.M * (g.N / 2);
          }
          r_item<PX>(g, at, tile, nt, twx, xp, slot, y0, sp.YR, node, za, zb);
        } else {
          i_item<PX>(g, at, tile, nt, twx, xp, slot, y0, sp.YR, node);
        }
      }
      // slot par was last read before the previous item's publish barrier, which thread 0 has
      // passed: no thread can still be reading it
      if (threadIdx.x == 0) s_next[par] = nxt;
      publish(sync + stage * sp.nbatch + b);   // its barrier also publishes s_next[par] to the CTA
      t = s_next[par];
      par ^= 1;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// host side

int spatial_maxb(const Geometry &g) {
  // Radix-16 plans (E = 16 values per thread, two CTAs per SM).  A radix-32 plan for the
  // 512/1024-point axes (one exchange instead of two, but 246 registers -> one CTA of 8 warps per
  // SM) measured 95.5 ms vs 79.1 ms per config-5 spatial launch: latency hiding wins here.
  (void)g;
  return 4;
}

SpatialPlan make_spatial_plan(const Geometry &g, int lines, bool synth) {
  SpatialPlan sp{};
  sp.lines = lines;
  const int mb = spatial_maxb(g);
  const int ex = g.lognx < mb ? g.nx : (1 << mb), ey = g.logny < mb ? g.ny : (1 << mb);
  const int tplx = g.nx / ex, tply = g.ny / ey;
  sp.YR = kSpThreads / (tplx * g.M);         // rows per R/I item: M*YR lines of TPLx threads
  if (sp.YR < 1) sp.YR = 1;
  while (sp.YR > 1 && (g.ny % sp.YR)) sp.YR >>= 1;
  if (sp.YR > g.ny) sp.YR = g.ny;
  sp.TC = kSpThreads / tply;                 // columns per C item
  if (sp.TC > g.nx) sp.TC = g.nx;
  if (sp.TC < 1) sp.TC = 1;
  // batch = one frequency slot (all M nodes: the node transforms sit in R and I)
  const int slots = lines / g.M;
  sp.B = 1;
  const size_t slot_bytes = (size_t)g.M * g.N * sizeof(double2);
  while ((size_t)sp.B * slot_bytes < ((size_t)16 << 20) && slots % (2 * sp.B) == 0) sp.B *= 2;
  sp.nbatch = slots / sp.B;
  sp.nRI = sp.B * (g.ny / sp.YR);
  sp.nC = sp.B * g.M * (g.nx / sp.TC);
  sp.synth = synth ? 1 : 0;
  sp.nstage = synth ? 2 : 3;
  const char *sk = getenv("PINT_SP_SKIP");   // timing experiments only: bit s skips stage s (R, C, I)
  sp.skip = sk ? atoi(sk) : 0;
  const char *cl = getenv("PINT_SP_CLAIM");  // A/B experiments: 0 = static round-robin assignment
  sp.claim = cl ? atoi(cl) : 1;
  sp.rounds = sp.nbatch + sp.nstage - 1;
  return sp;
}

size_t spatial_sync_bytes(int lines) { return (size_t)(3 * lines + 1) * sizeof(unsigned); }   // + claim counter

bool spatial2d_supported(const Geometry &g) {
  const int d = g.lognx - g.logny;
  return g.dim == 2 && g.lognx >= 2 && g.lognx <= 12 && g.logny >= 2 && g.logny <= 12 && d >= -1 && d <= 1 &&
         (g.nx >= 16 ? g.nx / 16 : 1) * g.M <= kSpThreads;
}

namespace {
template <int LX, int LY, int MB>
cudaError_t launch_sp(const Geometry &g, const StaticTables &st, const AlphaTables &at, const SpatialPlan &sp,
                      double2 *X, const double2 *spec, unsigned *sync, cudaStream_t s) {
  const void *fn = (const void *)spatial2d_kernel<LX, LY, MB>;
  // tile + one dummy line for the surplus lanes of partly used warps
  const size_t tile_r = (size_t)(sp.YR * g.M + 1) * g.nx, tile_c = (size_t)(sp.TC + 1) * (g.ny + 8);
  const size_t tile = tile_r > tile_c ? tile_r : tile_c;
  const size_t smem =
      (rfft::Plan<LX, MB>::twsize() + rfft::Plan<LY, MB>::twsize() + 64 + tile) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kSpThreads, smem)) != cudaSuccess) return e;
  if (per < 1) return cudaErrorInvalidConfiguration;
  Geometry gg = g;
  StaticTables sst = st;
  AlphaTables aat = at;
  SpatialPlan ssp = sp;
  double2 *xx = X;
  const double2 *ss = spec;
  unsigned *sy = sync;
  void *args[] = {&gg, &sst, &aat, &ssp, &xx, &ss, &sy};
  return cudaLaunchCooperativeKernel(fn, dim3(sms * per), dim3(kSpThreads), args, smem, s);
}

}  // namespace

cudaError_t launch_spatial2d(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                             const double2 *spec, unsigned *sync, int lines, cudaStream_t s) {
  if (!spatial2d_supported(g)) return cudaErrorInvalidValue;
  const SpatialPlan sp = make_spatial_plan(g, lines, spec != nullptr);
  cudaError_t e = cudaMemsetAsync(sync, 0, (size_t)(3 * sp.nbatch + 1) * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
#define PINT_SP(LXX, LYY) \
  if (g.lognx == LXX && g.logny == LYY) return launch_sp<LXX, LYY, 4>(g, st, at, sp, X, spec, sync, s);
#define PINT_SP3(L_) PINT_SP(L_, L_) PINT_SP(L_, L_ - 1) PINT_SP(L_ - 1, L_)
  PINT_SP(2, 2)
  PINT_SP3(3) PINT_SP3(4) PINT_SP3(5) PINT_SP3(6) PINT_SP3(7) PINT_SP3(8) PINT_SP3(9) PINT_SP3(10)
  PINT_SP3(11) PINT_SP3(12)
#undef PINT_SP3
#undef PINT_SP
  return cudaErrorInvalidValue;
}

}  // namespace pint
