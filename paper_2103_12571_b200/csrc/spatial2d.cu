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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "device_common.cuh"
#include "fft_reg.cuh"
#include "host_numerics.h"
#include "internal.h"

namespace pint {

namespace {

constexpr int kSpThreads = 256;
constexpr int kColScal = 16;   // per-group scalar slot of cols_pipe_kernel: shift, sig, <= 8 x-symbols (+ pad)
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
  const char *sk = experiment_env("PINT_SP_SKIP");   // timing experiments only: bit s skips stage s (R, C, I)
  sp.skip = sk ? atoi(sk) : 0;
  const char *cl = experiment_env("PINT_SP_CLAIM");  // A/B experiments: 0 = static round-robin assignment
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
  if (st.sm_reserve > 0 && sms > 2 * st.sm_reserve) sms -= st.sm_reserve;   // leave SMs to NCCL
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

// =============================================================================================
// Pipelined plane passes (one persistent launch per stage; the default 2-D solve for the large
// grids).  Same arithmetic as the R / C / I items above, restructured so that the
// memory stream never waits for the FFT arithmetic and DRAM only sees whole 128-byte lines:
//   * every CTA (one per SM) runs G consumer groups (one item each) over a ring of NS
//     shared-memory slots filled by the TMA unit (1-D cp.async.bulk of contiguous rows for R,
//     tensor-map tiles for C and I) that complete on one mbarrier per slot;
//   * the group that finishes reading slot s refills it with the CTA's item k + NS at once (ring
//     order = item order, every wait points to an earlier item: no deadlock);
//   * the spectral planes between R, C and I are stored COLUMN-BLOCKED: S-slot q of row y of a
//     plane lives at blk(q) ny 8 + y 8 + (q mod 8), blocks of 8 S-slot columns (128 bytes per
//     row).  R writes whole 128-byte block rows, C reads and writes block columns (a CTA takes
//     both 4-column halves of a block back to back, so the two 64-byte halves of every line meet
//     in L2), I reads a row as one tensor-map box of all blocks;
//   * results leave from registers (R, coalesced) or through the slot (I: node transform on the
//     way out; C: the column transpose).
// Items are assigned statically: CTA b takes b, b + grid, ... (grid = one CTA per SM).

namespace {

constexpr int kBW = 8;   // S-slot columns per block of the blocked spectral layout (128 bytes)

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// Wait for CTA-local item k in ring slot s = k mod NS.  The slot's previous item k - NS may belong
// to another group, and item k is only issued once that item is processed: a group that runs
// ahead must not test item k's phase parity while the barrier still sits in item k - NS's phase
// (equal parity two phases apart: try_wait.parity would pass at once on stale data).  The issuing
// thread records the item it put into the slot (slot_item[s]); once that reads k, item k - NS's
// phase has completed and the barrier's current phase is item k's, so the parity wait is exact.
__device__ __forceinline__ void ring_wait(uint64_t *bar, volatile int *slot_item, int k, int NS) {
  while (slot_item[k % NS] != k) __nanosleep(32);
  mbar_wait(bar, (unsigned)((k / NS) & 1));
}

// first 1024-byte aligned address (shared window) at or after p
__device__ __forceinline__ unsigned char *align_smem_1024(unsigned char *p) {
  const unsigned a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

// blocked offset of S-slot q in row y of a plane with ny rows
__device__ __forceinline__ size_t blocked(int q, int y, int logny) {
  return ((size_t)(q >> 3) << (logny + 3)) + ((size_t)y << 3) + (q & 7);
}

// y_m = sum_j A[m][j] x_j over the MM lines (stride NX) of each of the `rows` row groups of a
// natural-order tile, in place (A: M x M complex, global, L1-resident broadcast reads)
template <int MM>
__device__ __forceinline__ void node_natural(double2 *tile, const double2 *__restrict__ A, int rows, int NX, int t,
                                             int GT) {
  double2 ar[MM * MM];
#pragma unroll
  for (int i = 0; i < MM * MM; ++i) ar[i] = __ldg(A + i);
  for (int i = t; i < rows * NX; i += GT) {
    const int r = i / NX, x = i - r * NX;
    double2 *base = tile + (size_t)r * MM * NX + x;
    double2 v[MM];
#pragma unroll
    for (int j = 0; j < MM; ++j) v[j] = base[j * NX];
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < MM; ++j) acc = cfma(ar[m * MM + j], v[j], acc);
      base[m * NX] = acc;
    }
  }
}

// R (INV = false) and I (INV = true) stage.  Item = YR rows y0.. of all MM node planes of one
// unit (frequency slot p): LINES = YR MM lines of NX points, TPL threads per line, GT = LINES TPL
// threads per group.  R loads natural rows of X (1-D bulk copies) and stores blocked spectral
// rows into Yb (a second vector: a blocked row is spread over the whole plane, so R cannot work
// in place); I loads blocked rows of Yb through the tensor map `tmi` (box: all blocks of one
// row) and stores natural rows into X.  Named barriers: 1 + line id (exchanges, TPL > 32), then
// one per group.
template <class PX, int MM, bool INV, bool NODE>
__global__ void __launch_bounds__(PX::E == 32 ? 256 : 512, 1)
    rows_pipe_kernel(const __grid_constant__ CUtensorMap tmi, const Geometry g, StaticTables st, AlphaTables at,
                     double2 *__restrict__ X, double2 *__restrict__ Yb, int YR, int G, int NS, int nitems) {
  constexpr int NX = PX::N, TPL = PX::TPL, E = PX::E, R = 1 << PX::BL, TW = PX::twsize();
  constexpr int NBLK = NX / kBW, IBOX = NBLK < 256 ? NBLK : 256;
  extern __shared__ __align__(1024) unsigned char smraw_[];
  unsigned char *smraw = align_smem_1024(smraw_);   // the launch adds 1 KB of slack
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smraw + 64);   // item held by slot s (ring_wait)
  double2 *twx = reinterpret_cast<double2 *>(smraw + 128);
  double2 *ring = reinterpret_cast<double2 *>(smraw + 1024 + (((size_t)TW * sizeof(double2) + 1023) & ~(size_t)1023));
  const int LINES = YR * MM, GT = LINES * TPL, slot_elems = LINES * NX;
  const int gid = threadIdx.x / GT, t = threadIdx.x - gid * GT;
  const int l = t / TPL, tau = t - l * TPL;
  const int lid = gid * LINES + l;
  const int gbar = 1 + (TPL > 32 ? G * LINES : 0) + gid;   // after the line barriers (TPL > 32)
  const int ygroups = g.ny / YR;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      slot_item[s] = -1;
    }
    mbar_init_fence();
    if (INV) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmi) : "memory");
  }
  copy_table(twx, PX::E == 32 ? st.ptwx5 : st.ptwx, TW);
  __syncthreads();
  // fill the ring slot of CTA-local item k (one elected thread)
  auto issue = [&](int k) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= nitems) return;
    const int un = it / ygroups, y0 = (it - un * ygroups) * YR;
    const int p = __ldg(st.slots + un);
    uint64_t *bar = full + k % NS;
    double2 *dst = ring + (size_t)(k % NS) * slot_elems;
    mbar_arrive_expect_tx(bar, (unsigned)(slot_elems * sizeof(double2)));
    for (int yy = 0; yy < YR; ++yy)
      for (int m = 0; m < MM; ++m) {
        double2 *d = dst + (size_t)(yy * MM + m) * NX;
        if constexpr (INV) {
          for (int b = 0; b < NBLK; b += IBOX)
            tma_load_3d(d + b * kBW, &tmi, 0, y0 + yy, (p * MM + m) * NBLK + b, bar);
        } else if (st.packed) {
          // packed spectra (pairs (y, x), (y, x + nx/2)): row y of Z_k and of Z_{L-k} side by side
          const int kf = brev(p, g.logL), pc = brev((g.L - kf) & (g.L - 1), g.logL);
          const size_t ro = (size_t)(y0 + yy) << (PX::LOGN - 1);
          bulk_g2s(d, X + ((size_t)p * MM + m) * (g.N / 2) + ro, NX / 2 * sizeof(double2), bar);
          bulk_g2s(d + NX / 2, X + ((size_t)pc * MM + m) * (g.N / 2) + ro, NX / 2 * sizeof(double2), bar);
        } else {
          bulk_g2s(d, X + ((size_t)p * MM + m) * g.N + ((size_t)(y0 + yy) << PX::LOGN), NX * sizeof(double2), bar);
        }
      }
    slot_item[k % NS] = k;   // after the barrier's arm (ring_wait)
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  for (int k = gid;; k += G) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= nitems) break;
    const int s = k % NS;
    double2 *tile = ring + (size_t)s * slot_elems;
    double2 *line = tile + (size_t)l * NX;
    const int un = it / ygroups, y0 = (it - un * ygroups) * YR;
    const int p = __ldg(st.slots + un);
    // I output: the natural planes of slot p, or (packed mode) the unit planes behind Z
    double2 *xp = st.packed ? unit_planes(g, X) + (size_t)un * MM * g.N : X + (size_t)p * MM * g.N;
    const int yy = l / MM, m = l - yy * MM;
    ring_wait(full + s, slot_item, k, NS);
    double2 v[E];
    if constexpr (!INV) {
      if (st.packed) {   // X_k = (Z_k + conj Z_{L-k}) / 2 at x, (Z_k - conj Z_{L-k}) / 2i at x + nx/2
        for (int i = t; i < LINES * (NX / 2); i += GT) {
          const int li = i / (NX / 2), x = i - li * (NX / 2);
          double2 *a_ = tile + (size_t)li * NX + x;
          const double2 a = a_[0], b = a_[NX / 2];
          a_[0] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
          a_[NX / 2] = make_double2(0.5 * (a.y + b.y), 0.5 * (b.x - a.x));
        }
        named_sync(gbar, GT);
      }
      if constexpr (NODE) {   // x1 = S_p^{-1} x on the natural rows, in place
        node_natural<MM>(tile, at.Sinv + (size_t)p * MM * MM, YR, NX, t, GT);
        named_sync(gbar, GT);
      }
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = line[rfft::natural_pos<PX>(tau, i)];
      rfft::line_sync<PX>(lid);   // the engine's exchanges write swizzled positions
      rfft::forward_regs<PX>(v, line, lid, tau, twx);
      fence_proxy_async_smem();   // this thread's generic smem accesses before the refill's async ones
      named_sync(gbar, GT);       // every line of the slot has done its last read
      if (t == 0) issue(k + NS);
      double2 *dst = Yb + ((size_t)p * MM + m) * g.N;
#pragma unroll
      for (int u = 0; u < E / R; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) dst[blocked(rfft::s_slot<PX>(tau, u, r), y0 + yy, g.logny)] = v[u * R + r];
    } else {
#pragma unroll
      for (int u = 0; u < E / R; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) v[u * R + r] = line[rfft::s_slot<PX>(tau, u, r)];
      rfft::line_sync<PX>(lid);
      rfft::inverse_in_regs<PX>(v, line, lid, tau, twx);
      rfft::to_smem<PX, 0>(v, line, tau);
      named_sync(gbar, GT);
      if constexpr (NODE) {   // y = G_p^{-1} S_p x2 on the way out
        const double2 *A = at.SG + (size_t)p * MM * MM;
        double2 ar[MM * MM];
#pragma unroll
        for (int i = 0; i < MM * MM; ++i) ar[i] = __ldg(A + i);
        for (int i = t; i < YR * NX; i += GT) {
          const int x = i & (NX - 1), r2 = i >> PX::LOGN;
          const double2 *base = tile + (size_t)r2 * MM * NX + rfft::F<PX>(x);
          double2 w[MM];
#pragma unroll
          for (int j = 0; j < MM; ++j) w[j] = base[j * NX];
          double2 *o = xp + ((size_t)(y0 + r2) << PX::LOGN) + x;
#pragma unroll
          for (int mm = 0; mm < MM; ++mm) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < MM; ++j) acc = cfma(ar[mm * MM + j], w[j], acc);
            o[(size_t)mm * g.N] = acc;
          }
        }
      } else {
        for (int i = t; i < LINES * NX; i += GT) {
          const int x = i & (NX - 1), li = i >> PX::LOGN;
          const int y2 = li / MM, m2 = li - y2 * MM;
          xp[(size_t)m2 * g.N + ((size_t)(y0 + y2) << PX::LOGN) + x] = tile[(size_t)li * NX + rfft::F<PX>(x)];
        }
      }
      fence_proxy_async_smem();
      named_sync(gbar, GT);
      if (t == 0) issue(k + NS);
    }
  }
}

// C stage, in place on the blocked planes Yb.  Item = TC consecutive S-slot columns (one half of
// a block, or the whole block when TC = 8) of one plane (unit, node), loaded by the tensor map
// `tmc` (box {2 TC doubles, BR rows, 1 block}, 16-byte swizzle of the TC*16-byte rows:
// conflict-free column reads).  GC groups of TC TPL threads over a ring of NS slots; the CTA's
// items k, k+1 are the two halves of one block (with two groups they run side by side).  Then
// lines of stride ls for the engine's exchanges: y-DIF, x2 = x1 / ((1 - s lambda) nx ny) with the
// y-symbol table staged in shared memory, y-DIT; the transpose back to block rows goes through
// the slot.  Named barriers: 1 + group, then 1 + GC + line (TPL > 32).
//
// SYN (direct form, Alg. 1 as printed): the x1 spectrum of every plane q is sig_q r0hat, so the
// tile loaded is the item's block of r0hat itself (the same for every plane; `tmc` then maps the
// blocked spectrum of r0, plane 0, L2-resident) read at the DIF output positions, times sig_q; no
// y-DIF, the divide and the y-DIT follow.
// the C item geometry is fixed by the column plan (pipe_plan makes the same choice at run time and
// launch_pipe checks it): 8 columns per item if 8 lines of ny/16 threads fit 256 threads and the
// tile 64 KB, else 4; line stride ny + 8/TC (+1 for TC = 8); TMA boxes of min(ny, 256) rows
template <class PY>
__host__ __device__ constexpr int cols_lt() { return (8 * (PY::N / 16) <= 256 && 8 * PY::N * 16 <= 64 * 1024) ? 3 : 2; }
template <class PY>
__host__ __device__ constexpr int cols_ls() { return PY::N + ((1 << cols_lt<PY>()) >= 8 ? 1 : 8 / (1 << cols_lt<PY>())); }

template <class PX, class PY, int GC, bool SYN = false>
__global__ void __launch_bounds__(GC * 256 / (PY::TPL == 32 && PY::E == 32 ? 2 : 1), 1)
    cols_pipe_kernel(const __grid_constant__ CUtensorMap tmc, const Geometry g, StaticTables st, AlphaTables at,
                     double2 *__restrict__ Yb, int NS, int nitems) {
  constexpr int NY = PY::N, TPL = PY::TPL, E = PY::E, R = 1 << PY::BL, TW = PY::twsize();
  constexpr int LX = PX::LOGN, LY = PY::LOGN, NX = PX::N, NBLK = NX / kBW;
  static_assert(GC <= 2, "the scalar area holds two groups");
  extern __shared__ __align__(1024) unsigned char smraw_[];
  unsigned char *smraw = align_smem_1024(smraw_);   // swizzled TMA tiles need 1 KB-aligned slots
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smraw + 64);   // item held by slot s (ring_wait)
  double2 *twy = reinterpret_cast<double2 *>(smraw + 128);
  double2 *lamy = twy + TW;
  double2 *scal = lamy + NY;   // per group: the current item's shift, sig and TC x-symbols (kColScal)
  double2 *ring = reinterpret_cast<double2 *>(
      smraw + 1024 + (((size_t)(TW + NY + 2 * kColScal) * sizeof(double2) + 1023) & ~(size_t)1023));
  constexpr int lT = cols_lt<PY>(), ls = cols_ls<PY>(), BR = NY < 256 ? NY : 256;
  constexpr int TC = 1 << lT, NH = kBW >> lT;   // columns per item, items per block
  constexpr int slot_elems = ((TC * ls * (int)sizeof(double2) + 1023) & ~1023) / (int)sizeof(double2);
  constexpr int GT = TC * TPL;
  const int gid = threadIdx.x / GT, t = threadIdx.x - gid * GT, c = t / TPL, tau = t - c * TPL;
  const int gbar = 1 + gid, lid = GC + gid * TC + c;   // line_sync uses barrier 1 + lid
  const int M = g.M;
  const double inv_n = 1.0 / ((double)NX * (double)NY);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      slot_item[s] = -1;
    }
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmc) : "memory");
  }
  copy_table(twy, PY::E == 32 ? st.ptwy5 : st.ptwy, TW);
  // y symbols by spectral position P (frequency bitrev(P)), stored at P ^ ((P >> SH) & 7): the last
  // pass reads positions R_L g + r with lanes on consecutive g, which this XOR spreads over the
  // eight 16-byte bank slots (a plain bit-reversed table read was 8-way conflicted)
  constexpr int SH = PY::BL > 3 ? PY::BL : 3;
  for (int P = threadIdx.x; P < NY; P += blockDim.x) lamy[P ^ ((P >> SH) & 7)] = __ldg(st.lamy + brev(P, LY));
  // CTA-local item k: block pair b = blockIdx + (k / NH) grid, half k mod NH
  auto item_of = [&](int k) { return (blockIdx.x + (k / NH) * gridDim.x) * NH + (k % NH); };
  // the per-item scalars (plane shift s_q, sig_q, the x-symbol of each column) of the group's item
  // kk, loaded by the column leaders one item ahead into the group's scal slot: the divide reads
  // them from shared memory instead of waiting on dependent global loads in the middle of the item
  double2 *my_scal = scal + gid * kColScal;
  auto scal_load = [&](int kk, double2 &a, double2 &b, double2 &x) {
    const int it2 = item_of(kk);
    if (it2 >= nitems) return false;
    const int bi2 = it2 / NH, half2 = it2 - bi2 * NH;
    const int li2 = bi2 / NBLK, blk2 = bi2 - li2 * NBLK;
    const int un2 = li2 / M, mm2 = li2 - un2 * M;
    const int q2 = __ldg(st.slots + un2) * M + mm2;
    a = __ldg(at.shift + q2);
    b = SYN ? __ldg(at.sig + q2) : make_double2(0.0, 0.0);
    x = __ldg(st.lamx + brev(rfft::slot_to_pos<PX>(blk2 * kBW + half2 * TC + c), LX));
    return true;
  };
  auto scal_store = [&](const double2 &a, const double2 &b, const double2 &x) {
    if (c == 0) {
      my_scal[0] = a;
      my_scal[1] = b;
    }
    my_scal[2 + c] = x;
  };
  if (tau == 0) {
    double2 a, b, x;
    if (scal_load(gid, a, b, x)) scal_store(a, b, x);
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int it = item_of(k);
    if (it >= nitems) return;
    const int bi = it / NH, half = it - bi * NH;
    const int li = bi / NBLK, blk = bi - li * NBLK;
    const int un = li / M, mm = li - un * M;
    const int plane = __ldg(st.slots + un) * M + mm;
    uint64_t *bar = full + k % NS;
    double2 *dst = ring + (size_t)(k % NS) * slot_elems;
    mbar_arrive_expect_tx(bar, (unsigned)(NY * TC * sizeof(double2)));
    for (int b = 0; b < NY; b += BR)
      tma_load_3d(dst + (size_t)b * TC, &tmc, 2 * TC * half, b, (SYN ? 0 : plane) * NBLK + blk, bar);
    slot_item[k % NS] = k;   // after the barrier's arm (ring_wait)
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  for (int k = gid;; k += GC) {
    const int it = item_of(k);
    if (it >= nitems) break;
    const int s = k % NS;
    double2 *tile = ring + (size_t)s * slot_elems;
    const int bi = it / NH, half = it - bi * NH;
    const int li = bi / NBLK, blk = bi - li * NBLK;
    const int un = li / M, mm = li - un * M;
    const int q = __ldg(st.slots + un) * M + mm;   // table line (slot, node) == plane index
    const int q0 = blk * kBW + half * TC;          // first S-slot column of the item
    double2 *xb = Yb + (size_t)q * g.N + ((size_t)blk << (LY + 3)) + half * TC;
    (void)q0;
    ring_wait(full + s, slot_item, k, NS);
    double2 v[E];
    double2 *line = tile + (size_t)c * ls;
    // column c, row y of the swizzled TMA tile: 16-byte chunk c ^ ((y TC / 8) mod TC) of row y
    if constexpr (SYN) {   // the x1 spectrum sig_q r0hat at the DIF output positions (rows = P)
      // read in the natural arrangement (consecutive rows on consecutive lanes: conflict free) and
      // regroup through the exchange line; reading the last pass's rows R_L g + r straight from the
      // tile put all eight lanes of a quarter warp on one bank slot
      const double2 sg = my_scal[1];
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int y = rfft::natural_pos<PY>(tau, i);
        v[i] = cmul(sg, tile[(y << lT) + (c ^ (((y << lT) >> 3) & (TC - 1)))]);
      }
      named_sync(gbar, GT);   // the slot is re-used as TC exchange lines of stride ls
      rfft::to_smem<PY, 0>(v, line, tau);
      rfft::line_sync<PY>(lid);
#pragma unroll
      for (int u = 0; u < E / R; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) v[u * R + r] = line[rfft::F<PY>(rfft::last_pos<PY>(tau, u, r))];
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int y = rfft::natural_pos<PY>(tau, i);
        v[i] = tile[(y << lT) + (c ^ (((y << lT) >> 3) & (TC - 1)))];
      }
      named_sync(gbar, GT);   // the slot is re-used as TC exchange lines of stride ls
      rfft::forward_regs<PY>(v, line, lid, tau, twy);
    }
    const double2 sh = my_scal[0], lx = my_scal[2 + c];
#pragma unroll
    for (int u = 0; u < E / R; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        // 1 / ((1 - s lambda) nx ny), lambda = lambda_x + lambda_y (|1 - s lambda| >= 7.7e-4)
        const int P = rfft::last_pos<PY>(tau, u, r);
        const double2 lam = cadd(lx, lamy[P ^ ((P >> SH) & 7)]);
        const double2 sl = cmul(sh, lam);
        const double dr = 1.0 - sl.x, di = -sl.y;
        const double qq = dr * dr + di * di;
        const double den = inv_n * rcp_pos(qq);
        v[u * R + r] = cmul(v[u * R + r], make_double2(dr * den, -di * den));
      }
    rfft::inverse_in_regs<PY>(v, line, lid, tau, twy);
    rfft::to_smem<PY, 0>(v, line, tau);
    named_sync(gbar, GT);   // also: every divide of this item has read my_scal
    double2 na, nb, nx;
    const bool more = tau == 0 && scal_load(k + GC, na, nb, nx);   // in flight during the copy-out
    {   // element (column cc, row y) of the item -> blocked row y; thread t: cc = t mod TC, rows t/TC + j TPL
      const int cc = t & (TC - 1), y0 = t >> lT;
      double2 *xo = xb + cc + ((size_t)y0 << 3);
      const double2 *ti = tile + (size_t)cc * ls;
#pragma unroll 8
      for (int j = 0; j < NY / TPL; ++j) xo[(size_t)j * TPL * 8] = ti[rfft::F<PY>(y0 + j * TPL)];
    }
    if (more) scal_store(na, nb, nx);
    fence_proxy_async_smem();
    named_sync(gbar, GT);
    if (t == 0) issue(k + NS);
  }
}

// ---------------------------------------------------------------------------------------------
// Fused plane passes (1024^2 grids, radix-32 plans on both axes, one rank): R, C and I items of
// consecutive frequency slots interleaved in ONE persistent launch, so the SM runs fp64-heavy C
// items beside memory-heavy R / I items and the blocked spectra of a slot are re-read while still
// largely in L2.  Global item sequence, round j: R(j), C(j - 1), I(j - 2) (batch = one slot, all M
// nodes); CTA c takes items c, c + grid, ...; two groups of 128 threads alternate over a ring of
// three slots (sized for the largest item).  Dependencies: C(b) reads what all R(b) items wrote,
// I(b) what all C(b) items wrote: completion counters done[stage][b] (bar.sync + red.release.gpu
// after the item's stores; ld.acquire.gpu + proxy fence before the TMA load that reads them).  A
// refill whose dependency is not met yet is deferred to the group that will consume the item
// (it waits once it holds no other unfinished item), so every wait points to items of an earlier
// round that are never blocked behind a wait of a later round: deadlock free with all CTAs
// resident (one per SM, launched as a cooperative grid).
namespace fused {

struct Seq {
  int nb, nR, nC, nI;
};

__device__ __forceinline__ long long round_size(const Seq &q, int j) {
  return (j < q.nb ? q.nR : 0) + (j >= 1 && j <= q.nb ? q.nC : 0) + (j >= 2 && j <= q.nb + 1 ? q.nI : 0);
}

// global item index -> (stage 0 R / 1 C / 2 I, batch, index within the stage segment)
__device__ __forceinline__ void decode(const Seq &q, long long g, int &stage, int &b, int &idx) {
  long long rs = 0;
  int j = 0;
  const long long s0 = round_size(q, 0), s1 = round_size(q, 1);
  if (q.nb >= 3 && g >= s0 + s1) {   // skip whole middle rounds (all three segments present)
    const long long S = (long long)q.nR + q.nC + q.nI;
    long long jj = (g - s0 - s1) / S;
    if (jj > q.nb - 2) jj = q.nb - 2;
    j = 2 + (int)jj;
    rs = s0 + s1 + jj * S;
  }
  for (;;) {
    const long long rn = round_size(q, j);
    if (g < rs + rn) break;
    rs += rn;
    ++j;
  }
  long long off = g - rs;
  if (j < q.nb) {
    if (off < q.nR) { stage = 0; b = j; idx = (int)off; return; }
    off -= q.nR;
  }
  if (j >= 1 && j <= q.nb) {
    if (off < q.nC) { stage = 1; b = j - 1; idx = (int)off; return; }
    off -= q.nC;
  }
  stage = 2;
  b = j - 2;
  idx = (int)off;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void release_add(unsigned *p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

}  // namespace fused

template <int MM>
__global__ void __launch_bounds__(256, 1)
    spatial_fused_kernel(const __grid_constant__ CUtensorMap tmi, const __grid_constant__ CUtensorMap tmc,
                         const Geometry g, StaticTables st, AlphaTables at, double2 *__restrict__ X,
                         double2 *__restrict__ Yb, int YR, int nb, unsigned *__restrict__ done) {
  using PL = rfft::Plan<10, 5>;   // both axes: 1024 points, 32 values x 32 threads per line
  constexpr int N1 = PL::N, TPL = PL::TPL, E = PL::E, R = 1 << PL::BL, TW = PL::twsize();
  constexpr int LG = PL::LOGN, NBLK = N1 / kBW, TC = 4, LT = 2, LS = N1 + 2, NS = 3, GT = 128;
  constexpr int SH = PL::BL > 3 ? PL::BL : 3;
  constexpr int SLOT = ((TC * LS * 16 + 1023) & ~1023) / 16;   // >= R / I items (4 lines x 1024)
  extern __shared__ __align__(1024) unsigned char smraw_[];
  unsigned char *smraw = align_smem_1024(smraw_);
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smraw + 64);
  double2 *tw = reinterpret_cast<double2 *>(smraw + 128);
  double2 *lamy = tw + TW;
  double2 *ring = reinterpret_cast<double2 *>(smraw + 1024 + (((size_t)(TW + N1) * 16 + 1023) & ~(size_t)1023));
  const int LINES = YR * MM;
  const int gid = threadIdx.x / GT, t = threadIdx.x - gid * GT, l = t / TPL, tau = t - l * TPL;
  const int gbar = 1 + gid;   // lines are warps (TPL = 32): __syncwarp exchanges, no line barriers
  const fused::Seq q{nb, g.ny / YR, MM * (g.nx / TC), g.ny / YR};
  const long long total = (long long)nb * (q.nR + q.nC + q.nI);
  const double inv_n = 1.0 / ((double)g.nx * (double)g.ny);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      slot_item[s] = -1;
    }
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmi) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmc) : "memory");
  }
  copy_table(tw, st.ptwx5, TW);
  for (int P = threadIdx.x; P < N1; P += blockDim.x) lamy[P ^ ((P >> SH) & 7)] = __ldg(st.lamy + brev(P, LG));
  __syncthreads();
  auto item = [&](int k) { return (long long)blockIdx.x + (long long)k * gridDim.x; };
  auto dep_ready = [&](int stage, int b) {
    if (stage == 0) return true;
    const unsigned need = stage == 1 ? (unsigned)q.nR : (unsigned)q.nC;
    return fused::ld_acquire(done + (stage - 1) * nb + b) >= need;
  };
  auto issue_now = [&](int k) {   // dependency met (or none): arm the slot and start the copies
    int stage, b, idx;
    fused::decode(q, item(k), stage, b, idx);
    const int p = __ldg(st.slots + b);
    uint64_t *bar = full + k % NS;
    double2 *dst = ring + (size_t)(k % NS) * SLOT;
    if (stage == 1) {   // C: 4 S-slot columns (a half block) of plane (p, m)
      const int bi = idx >> 1, half = idx & 1;
      const int mm = bi / NBLK, blk = bi - mm * NBLK;
      mbar_arrive_expect_tx(bar, (unsigned)(N1 * TC * 16));
      for (int y = 0; y < N1; y += 256) tma_load_3d(dst + (size_t)y * TC, &tmc, 2 * TC * half, y, (p * MM + mm) * NBLK + blk, bar);
    } else {            // R: natural rows of X; I: blocked rows of Yb
      const int y0 = idx * YR;
      mbar_arrive_expect_tx(bar, (unsigned)(LINES * N1 * 16));
      for (int yy = 0; yy < YR; ++yy)
        for (int m = 0; m < MM; ++m) {
          double2 *d = dst + (size_t)(yy * MM + m) * N1;
          if (stage == 0)
            bulk_g2s(d, X + ((size_t)p * MM + m) * g.N + ((size_t)(y0 + yy) << LG), N1 * 16, bar);
          else
            tma_load_3d(d, &tmi, 0, y0 + yy, (p * MM + m) * NBLK, bar);
        }
    }
    slot_item[k % NS] = k;
  };
  auto issue = [&](int k) {       // refill: start the copies now, or defer to the consumer of k
    if (item(k) >= total) return;
    int stage, b, idx;
    fused::decode(q, item(k), stage, b, idx);
    if (dep_ready(stage, b)) {
      fused::fence_proxy_async_global();
      issue_now(k);
    } else {
      slot_item[k % NS] = -(k + 2);
    }
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  for (int k = gid;; k += 2) {
    const long long gi = item(k);
    if (gi >= total) break;
    int stage, b, idx;
    fused::decode(q, gi, stage, b, idx);
    const int s = k % NS;
    double2 *tile = ring + (size_t)s * SLOT;
    const int p = __ldg(st.slots + b);
    // wait for the slot to hold item k (doing a deferred refill ourselves) and for its bytes
    for (;;) {
      const int v = slot_item[s];
      if (v == k) break;
      if (v == -(k + 2)) {
        if (t == 0) {
          const unsigned need = stage == 1 ? (unsigned)q.nR : (unsigned)q.nC;
          while (fused::ld_acquire(done + (stage - 1) * nb + b) < need) __nanosleep(128);
          fused::fence_proxy_async_global();
          issue_now(k);
        }
        while (slot_item[s] != k) __nanosleep(32);
        break;
      }
      __nanosleep(32);
    }
    mbar_wait(full + s, (unsigned)((k / NS) & 1));
    double2 v[E];
    if (stage == 0) {   // ---- R: S_p^{-1} over the natural rows, x-DIF, blocked store into Yb
      const int y0 = idx * YR;
      node_natural<MM>(tile, at.Sinv + (size_t)p * MM * MM, YR, N1, t, GT);
      named_sync(gbar, GT);
      const bool act = l < LINES;
      double2 *line = tile + (size_t)(act ? l : 0) * N1;
      if (act) {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = line[rfft::natural_pos<PL>(tau, i)];
        __syncwarp();
        rfft::forward_regs<PL>(v, line, 0, tau, tw);
      }
      fence_proxy_async_smem();
      named_sync(gbar, GT);
      if (t == 0) issue(k + NS);
      if (act) {
        const int yy = l / MM, m = l - yy * MM;
        double2 *dst = Yb + ((size_t)p * MM + m) * g.N;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[blocked(rfft::s_slot<PL>(tau, 0, r), y0 + yy, LG)] = v[r];
      }
      fused::fence_proxy_async_global();
      named_sync(gbar, GT);
      if (t == 0) fused::release_add(done + 0 * nb + b);
    } else if (stage == 1) {   // ---- C: y-DIF, divide, y-DIT on 4 columns, in place in Yb
      const int bi = idx >> 1, half = idx & 1;
      const int mm = bi / NBLK, blk = bi - mm * NBLK;
      const int qq = p * MM + mm;
      const int c = l;   // 4 columns = the group's 4 warps
      const int q0 = blk * kBW + half * TC;
      double2 *xb = Yb + (size_t)qq * g.N + ((size_t)blk << (LG + 3)) + half * TC;
      const double2 sh = __ldg(at.shift + qq);
      const double2 lx = __ldg(st.lamx + brev(rfft::slot_to_pos<PL>(q0 + c), LG));
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int y = rfft::natural_pos<PL>(tau, i);
        v[i] = tile[(y << LT) + (c ^ (((y << LT) >> 3) & (TC - 1)))];
      }
      named_sync(gbar, GT);
      double2 *line = tile + (size_t)c * LS;
      rfft::forward_regs<PL>(v, line, 0, tau, tw);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int P = rfft::last_pos<PL>(tau, 0, r);
        const double2 lam = cadd(lx, lamy[P ^ ((P >> SH) & 7)]);
        const double2 sl = cmul(sh, lam);
        const double dr = 1.0 - sl.x, di = -sl.y;
        const double q2 = dr * dr + di * di;
        const double den = inv_n * __drcp_rn(q2);
        v[r] = cmul(v[r], make_double2(dr * den, -di * den));
      }
      rfft::inverse_in_regs<PL>(v, line, 0, tau, tw);
      rfft::to_smem<PL, 0>(v, line, tau);
      named_sync(gbar, GT);
      for (int i = t; i < (N1 << LT); i += GT) {
        const int cc = i & (TC - 1), y = i >> LT;
        xb[((size_t)y << 3) + cc] = tile[(size_t)cc * LS + rfft::F<PL>(y)];
      }
      fence_proxy_async_smem();
      fused::fence_proxy_async_global();
      named_sync(gbar, GT);
      if (t == 0) {
        fused::release_add(done + 1 * nb + b);
        issue(k + NS);
      }
    } else {   // ---- I: x-DIT of the blocked rows, G_p^{-1} S_p on the way out to X
      const int y0 = idx * YR;
      const bool act = l < LINES;
      double2 *line = tile + (size_t)(act ? l : 0) * N1;
      if (act) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = line[rfft::s_slot<PL>(tau, 0, r)];
        __syncwarp();
        rfft::inverse_in_regs<PL>(v, line, 0, tau, tw);
        rfft::to_smem<PL, 0>(v, line, tau);
      }
      named_sync(gbar, GT);
      const double2 *A = at.SG + (size_t)p * MM * MM;
      double2 ar[MM * MM];
#pragma unroll
      for (int i = 0; i < MM * MM; ++i) ar[i] = __ldg(A + i);
      double2 *xp = X + (size_t)p * MM * g.N;
      for (int i = t; i < YR * N1; i += GT) {
        const int x = i & (N1 - 1), r2 = i >> LG;
        const double2 *base = tile + (size_t)r2 * MM * N1 + rfft::F<PL>(x);
        double2 w[MM];
#pragma unroll
        for (int j = 0; j < MM; ++j) w[j] = base[j * N1];
        double2 *o = xp + ((size_t)(y0 + r2) << LG) + x;
#pragma unroll
        for (int m2 = 0; m2 < MM; ++m2) {
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < MM; ++j) acc = cfma(ar[m2 * MM + j], w[j], acc);
          o[(size_t)m2 * g.N] = acc;
        }
      }
      fence_proxy_async_smem();
      named_sync(gbar, GT);
      if (t == 0) issue(k + NS);
    }
  }
}

struct PipePlan {
  int YR, G, NS;           // R / I: rows per item, groups, slots
  int lT, GC, NSC, ls, BR; // C: log2 columns per item, groups (1: 255 registers, 2: 128), slots, line stride, box rows
  int rx32, ry32;          // radix-32 plans for the 1024-point x (R, I) / y (C) axes
  size_t rsmem, csmem;
};

bool pipe_plan(const Geometry &g, PipePlan &pp) {
  if (g.dim != 2 || g.lognx < 9 || g.logny < 9 || g.lognx > 11 || g.logny > 11) return false;
  if (g.lognx - g.logny > 1 || g.logny - g.lognx > 1 || g.M > 4) return false;
  // radix-32 row plan for the R / I passes (1024^2 grids; the C pass must use the same x plan):
  // R 16.3 -> 13.8 ms, I 13.1 -> 11.8 ms on config 5
  pp.rx32 = g.lognx == 10 && g.logny == 10 ? 1 : 0;
  if (const char *e = experiment_env("PINT_R_RADIX32")) pp.rx32 = atoi(e) && g.lognx == 10 && g.logny == 10 ? 1 : 0;
  const int tplx = pp.rx32 ? 32 : g.nx / 16, tply = g.ny / 16;
  // R / I: items of YR rows x M nodes, <= 256 threads and <= 64 KB, two groups, three slots
  int YR = 1;
  while (2 * YR * g.M * tplx <= 256 && 2 * YR * g.M * g.nx * 16 <= 64 * 1024 && g.ny % (2 * YR) == 0) YR *= 2;
  if (YR * g.M * tplx > 256 || (size_t)YR * g.M * g.nx * 16 > 64 * 1024) return false;
  pp.YR = YR;
  pp.G = 512 / (YR * g.M * tplx);
  if (pp.G > 2) pp.G = 2;
  pp.NS = pp.G + 1;
  const size_t tw_r = ((size_t)pass_twiddle_count(g.lognx, pp.rx32 ? 5 : 4) * 16 + 1023) & ~(size_t)1023;
  pp.rsmem = 1024 + 1024 + tw_r + (size_t)pp.NS * YR * g.M * g.nx * 16;
  // C: a whole 8-column block per item if it fits 256 threads and 64 KB, else half blocks
  int lT = 3;
  while (lT > 2 && ((1 << lT) * tply > 256 || (size_t)(1 << lT) * g.ny * 16 > 64 * 1024)) --lT;
  const int TC = 1 << lT;
  if (TC * tply > 256) return false;
  pp.lT = lT;
  pp.GC = 1;
  if (const char *e = experiment_env("PINT_C_GROUPS")) pp.GC = atoi(e) == 2 ? 2 : 1;
  // radix-32 column plan (32 threads x 32 values per line, one exchange per transform, two groups
  // of 128 threads at <= 255 registers): C 31 -> 24 ms on config 5
  pp.ry32 = g.logny == 10 && g.lognx == 10 ? 1 : 0;
  if (const char *e = experiment_env("PINT_C_RADIX32")) pp.ry32 = atoi(e) && g.logny == 10 && g.lognx == 10 ? 1 : 0;
  if (pp.ry32) pp.GC = 2;
  pp.NSC = pp.GC + 1 > 3 ? pp.GC + 1 : 3;
  pp.ls = g.ny + (TC >= 8 ? 1 : 8 / TC);
  pp.BR = g.ny < 256 ? g.ny : 256;
  const size_t tw_c =
      ((size_t)(pass_twiddle_count(g.logny, pp.ry32 ? 5 : 4) + g.ny + 2 * kColScal) * 16 + 1023) & ~(size_t)1023;
  const size_t cslot = ((size_t)TC * pp.ls * 16 + 1023) & ~(size_t)1023;
  pp.csmem = 1024 + 1024 + tw_c + (size_t)pp.NSC * cslot;
  const int lbr = tplx > 32 && !pp.rx32 ? pp.G * YR * g.M : 0, lbc = tply > 32 && !pp.ry32 ? pp.GC * TC : 0;   // named barrier ids
  if (lbr + pp.G + 1 > 16 || lbc + pp.GC + 1 > 16) return false;
  return pp.rsmem <= 227 * 1024 && pp.csmem <= 227 * 1024;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  }
  return fn;
}

// tensor map over the blocked spectral planes Yb: dims {16 doubles (one block row), ny rows,
// planes * nx/8 blocks}
bool blocked_map(const Geometry &g, double2 *Yb, unsigned box0, unsigned box1, unsigned box2, CUtensorMapSwizzle swz,
                 CUtensorMap &tm) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * kBW, (cuuint64_t)g.ny, (cuuint64_t)g.L * g.M * (g.nx / kBW)};
  const cuuint64_t strides[2] = {(cuuint64_t)kBW * 16, (cuuint64_t)kBW * 16 * g.ny};
  const cuuint32_t box[3] = {box0, box1, box2};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)Yb, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// direct form: r0hat (position order, [py][px]) -> the blocked S-slot layout of the C pass
// (S-slot q of row py at blocked(q, py)) in `out` (one plane)
template <class PX>
__global__ void spec_blocked_kernel(const Geometry g, const double2 *__restrict__ spec, double2 *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.N; i += gridDim.x * blockDim.x) {
    const int q = i & (g.nx - 1), py = i >> g.lognx;
    out[blocked(q, py, g.logny)] = __ldg(spec + ((size_t)py << g.lognx) + rfft::slot_to_pos<PX>(q));
  }
}

template <class PX, class PY, int MM, int GC>
cudaError_t launch_pipe(const Geometry &g, const StaticTables &st, const AlphaTables &at, const PipePlan &pp,
                        double2 *X, double2 *Yb, int units, bool node, cudaStream_t s,
                        const double2 *spec = nullptr) {   // spec: direct form (no R pass, C synthesized)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (st.sm_reserve > 0 && sms > 2 * st.sm_reserve) sms -= st.sm_reserve;   // leave SMs to NCCL
  cudaError_t e;
  const int TC = 1 << pp.lT;
  const unsigned nblk = g.nx / kBW;
  CUtensorMap tmi, tmc;
  // direct form: the blocked spectrum of r0 goes to the first plane of X (X is written only by the
  // I pass, after the C pass has read it)
  if (!blocked_map(g, Yb, 2 * kBW, 1, nblk < 256 ? nblk : 256, CU_TENSOR_MAP_SWIZZLE_NONE, tmi) ||
      !blocked_map(g, spec ? X : Yb, 2 * TC, pp.BR, 1, TC == 4 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   tmc))
    return cudaErrorNotSupported;
  if (spec) {
    spec_blocked_kernel<PX><<<sms * 4, 256, 0, s>>>(g, spec, X);
    record_launch(s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const int rthreads = pp.G * pp.YR * MM * PX::TPL;
  const int ritems = units * (g.ny / pp.YR);
  auto rows = [&](auto fn) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.rsmem);
    if (e2 != cudaSuccess) return e2;
    fn<<<sms, rthreads, pp.rsmem, s>>>(tmi, g, st, at, X, Yb, pp.YR, pp.G, pp.NS, ritems);
    record_launch(s);
    return cudaGetLastError();
  };
  if (!spec) {
    e = node ? rows(rows_pipe_kernel<PX, MM, false, true>) : rows(rows_pipe_kernel<PX, MM, false, false>);
    if (e != cudaSuccess) return e;
  }
  {
    const void *fn = spec ? (const void *)cols_pipe_kernel<PX, PY, GC, true> : (const void *)cols_pipe_kernel<PX, PY, GC>;
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.csmem)) != cudaSuccess)
      return e;
    if (pp.lT != cols_lt<PY>() || pp.ls != cols_ls<PY>() || pp.BR != (PY::N < 256 ? PY::N : 256))
      return cudaErrorInvalidValue;   // the kernel's compile-time item geometry must match the plan
    const int cthreads = GC * TC * PY::TPL;
    const int citems = units * g.M * (g.nx / TC);
    if (spec)
      cols_pipe_kernel<PX, PY, GC, true><<<sms, cthreads, pp.csmem, s>>>(tmc, g, st, at, Yb, pp.NSC, citems);
    else
      cols_pipe_kernel<PX, PY, GC><<<sms, cthreads, pp.csmem, s>>>(tmc, g, st, at, Yb, pp.NSC, citems);
    record_launch(s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return node ? rows(rows_pipe_kernel<PX, MM, true, true>) : rows(rows_pipe_kernel<PX, MM, true, false>);
}

// plans: radix-32 passes (Plan<10, 5>: 32 values per thread, one exchange per transform) for
// 1024-point axes when selected, radix-16 (Plan<L, 4>) otherwise
template <int LX, int LY, int MM>
cudaError_t launch_pipe_dispatch(const Geometry &g, const StaticTables &st, const AlphaTables &at, const PipePlan &pp,
                                 double2 *X, double2 *Yb, int units, bool node, cudaStream_t s,
                                 const double2 *spec = nullptr) {
  using PX4 = rfft::Plan<LX, 4>;
  using PY4 = rfft::Plan<LY, 4>;
  if constexpr (LX == 10 && LY == 10) {
    using P5 = rfft::Plan<10, 5>;
    if (pp.rx32 && pp.ry32) return launch_pipe<P5, P5, MM, 2>(g, st, at, pp, X, Yb, units, node, s, spec);
    if (pp.ry32) return launch_pipe<PX4, P5, MM, 2>(g, st, at, pp, X, Yb, units, node, s, spec);
    if (pp.rx32) return launch_pipe<P5, PY4, MM, 1>(g, st, at, pp, X, Yb, units, node, s, spec);
  }
  return pp.GC == 2 ? launch_pipe<PX4, PY4, MM, 2>(g, st, at, pp, X, Yb, units, node, s, spec)
                    : launch_pipe<PX4, PY4, MM, 1>(g, st, at, pp, X, Yb, units, node, s, spec);
}

// ---------------------------------------------------------------------------------------------
// Pipelined 2-D time transforms (north star step (ii) and the inverse of (v)): item = one node m
// and T consecutive points n0.. over all L steps (rows at stride M N).  Tiles arrive by TMA in
// 128-byte column boxes (8 points x up to 256 steps, 128-byte swizzle: conflict-free column
// reads), two consumer groups run the register FFT engine on the T columns over a ring of three
// slots, results are put back into the slot in the boxes' layout and leave by the TMA unit.
//   forward: X[p][m][n] = DIF_L(alpha^{l/L} r_l)[p]  (slot p holds frequency bitrev(p); the scale
//            was applied by the residual kernel), P > 1: times the four-step twiddle twr[p];
//            one tensor store per box.
//   inverse: u[l][m][n] += alpha^{-l/L} / L * DIT_L(x2)[l]: the update is a TMA tensor
//            REDUCTION (cp.reduce.async.bulk.tensor .add on the FLOAT64 map of u, UTMAREDG: the
//            fp64 add happens at the L2, u never enters the SM); overwrite: a tensor store, the
//            old last-step value read by the one thread per column that needs it; the last-step
//            difference; optionally (pf) an L2 prefetch of the u tile when the x2 tile is issued.
template <class PL, bool INV>
__global__ void __launch_bounds__(PL::E == 32 ? 256 : 512, 1)
    tfft_pipe_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmu,
                     const Geometry g, StaticTables st, AlphaTables at, double2 *__restrict__ X,
                     double2 *__restrict__ u, int lT, int G, int NS, int ls, int nitems,
                     unsigned long long *diff_slot, int overwrite, int pf, int pair) {
  constexpr int NL = PL::N, TPL = PL::TPL, E = PL::E, R = 1 << PL::BL, TW = PL::twsize(), NP = PL::NP;
  constexpr int LB = NL < 256 ? NL : 256;   // steps per TMA box
  extern __shared__ __align__(1024) unsigned char smraw_[];
  unsigned char *smraw = align_smem_1024(smraw_);
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smraw + 64);   // item held by slot s (ring_wait)
  double2 *twl = reinterpret_cast<double2 *>(smraw + 128);
  constexpr size_t kTwBytes = ((size_t)TW * sizeof(double2) + 1023) & ~(size_t)1023;
  constexpr size_t kScBytes = ((size_t)NL * sizeof(double) + 1023) & ~(size_t)1023;
  double *sbw = reinterpret_cast<double *>(smraw + 1024 + kTwBytes);   // inverse: alpha^{-l/L} / L
  double2 *ring = reinterpret_cast<double2 *>(smraw + 1024 + kTwBytes + kScBytes);
  __shared__ double red[16];
  const int T = 1 << lT, GT = T * TPL;
  const int tile_elems = NL * T, line_elems = T * ls;
  const int slot_elems = (((tile_elems > line_elems ? tile_elems : line_elems) * (int)sizeof(double2) + 1023) & ~1023) /
                         (int)sizeof(double2);
  const int gid = threadIdx.x / GT, t = threadIdx.x - gid * GT, c = t / TPL, tau = t - c * TPL;
  const int gbar = 1 + gid, lid = G + gid * T + c;   // line_sync: barrier 1 + lid (TPL > 32)
  const int per = g.N >> lT;
  const size_t lstride = (size_t)g.M * g.N;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      slot_item[s] = -1;
    }
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmx) : "memory");
    if (INV) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmu) : "memory");
  }
  copy_table(twl, st.ptwL, TW);
  if (INV)
    for (int i = threadIdx.x; i < NL; i += blockDim.x) sbw[i] = __ldg(at.scale_bwd + i);
  __syncthreads();
  // pair: the CTA's items k, k + 1 are neighbours in n (256 contiguous bytes per step between them)
  auto item_of = [&](int k) {
    return pair ? 2 * ((int)blockIdx.x + (k >> 1) * (int)gridDim.x) + (k & 1) : (int)blockIdx.x + k * (int)gridDim.x;
  };
  auto issue = [&](int k) {
    const int it = item_of(k);
    if (it >= nitems) return;
    const int m = it / per, n0 = (it - m * per) << lT;
    uint64_t *bar = full + k % NS;
    double2 *dst = ring + (size_t)(k % NS) * slot_elems;
    mbar_arrive_expect_tx(bar, (unsigned)(tile_elems * sizeof(double2)));
    for (int cb = 0; cb < T; cb += 8)
      for (int lb = 0; lb < NL; lb += LB) {
        tma_load_3d(dst + (size_t)cb * NL + lb * 8, &tmx, 2 * (n0 + cb), m, lb, bar);
        if (INV && !overwrite && pf)   // the reduction's read of u: start it towards L2 now
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(&tmu),
                       "r"(2 * (n0 + cb)), "r"(m), "r"(lb)
                       : "memory");
      }
    slot_item[k % NS] = k;   // after the barrier's arm (ring_wait)
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  double dmax = 0.0;
  for (int k = gid;; k += G) {
    const int it = item_of(k);
    if (it >= nitems) break;
    const int s = k % NS;
    double2 *tile = ring + (size_t)s * slot_elems;
    const int m = it / per, n0 = (it - m * per) << lT;
    // column c of the tile: box c / 8, row l, 16-byte chunk (c mod 8) ^ (l mod 8)
    double2 *col = tile + (size_t)(c >> 3) * NL * 8;
    const int cc = c & 7;
    double2 *line = tile + (size_t)c * ls;
    double2 uold = make_double2(0.0, 0.0);
    if (INV && overwrite && diff_slot && tau == TPL - 1)   // overwrite form: the old last-step value
      uold = u[(size_t)(NL - 1) * lstride + (size_t)m * g.N + n0 + c];
    ring_wait(full + s, slot_item, k, NS);
    double2 v[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int l = rfft::natural_pos<PL>(tau, i);
      v[i] = col[l * 8 + (cc ^ (l & 7))];
    }
    named_sync(gbar, GT);   // the slot becomes T exchange lines of stride ls
    if constexpr (!INV) {
      rfft::forward_regs<PL>(v, line, lid, tau, twl);
      // slot order out: through the line once more so that every thread holds the slots
      // tau + TPL i (the arrangement whose box rows are bank-conflict free)
      rfft::to_smem<PL, NP - 1>(v, line, tau);
      rfft::line_sync<PL>(lid);
      rfft::from_smem<PL, 0>(v, line, tau);
      if (st.twr) {   // P > 1: four-step twiddle
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = cmul(v[i], __ldg(st.twr + rfft::natural_pos<PL>(tau, i)));
      }
    } else {
      // slot order in, natural steps out: place the values at their swizzled line positions,
      // re-read them at the last pass's positions, then the inverse transform
      rfft::to_smem<PL, 0>(v, line, tau);
      rfft::line_sync<PL>(lid);
#pragma unroll
      for (int uu = 0; uu < E / R; ++uu)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int P = rfft::last_pos<PL>(tau, uu, r);
          double2 w = line[rfft::F<PL>(P)];
          if (st.twr) w = cmulc(w, __ldg(st.twr + P));   // P > 1: inverse four-step twiddle
          v[uu * R + r] = w;
        }
      rfft::line_sync<PL>(lid);
      rfft::inverse_in_regs<PL>(v, line, lid, tau, twl);   // v[i]: step tau + TPL i
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = cscale(v[i], sbw[rfft::natural_pos<PL>(tau, i)]);
      if (tau == TPL - 1) {   // step L - 1
        const double2 dd = overwrite ? csub(v[E - 1], uold) : v[E - 1];
        dmax = nanmax(dmax, hypot(dd.x, dd.y));
      }
    }
    named_sync(gbar, GT);   // every line of the group read: the slot becomes the boxes again
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int l = rfft::natural_pos<PL>(tau, i);
      col[l * 8 + (cc ^ (l & 7))] = v[i];
    }
    fence_proxy_async_smem();
    named_sync(gbar, GT);
    if (t == 0) {
      for (int cb = 0; cb < T; cb += 8)
        for (int lb = 0; lb < NL; lb += LB) {
          const double2 *src = tile + (size_t)cb * NL + lb * 8;
          if (INV && !overwrite) tma_reduce_add_3d(&tmu, 2 * (n0 + cb), m, lb, src);
          else tma_store_3d(INV ? &tmu : &tmx, 2 * (n0 + cb), m, lb, src);
        }
      bulk_commit();
      bulk_wait_read();   // the TMA unit has read the slot: refill it
      issue(k + NS);
    }
  }
  if (INV && diff_slot) {
    for (int o = 16; o > 0; o >>= 1) dmax = nanmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double vmax = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) vmax = nanmax(vmax, red[w]);
      atomicMax(diff_slot, (unsigned long long)__double_as_longlong(vmax));
    }
  }
}

// A/B (experiments build): PINT_TFFT_PF=1 prefetches the u tile towards the L2 when the x2 tile is issued
static int tfft_prefetch() {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_TFFT_PF");
    v = (e && atoi(e)) ? 1 : 0;
  }
  return v;
}

static int tfft_pair() {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_TFFT_PAIR");
    v = (e && atoi(e)) ? 1 : 0;
  }
  return v;
}
static int tfft_promo256() {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_TFFT_PROMO");
    v = (e && atoi(e)) ? 1 : 0;
  }
  return v;
}

struct TfftPlan {
  int lT, G, NS, ls;
  size_t smem;
};

template <class PL>
bool tfft_plan(const Geometry &g, TfftPlan &tp) {
  // T points per item: 64 KB tiles (L T 16 bytes), 8 <= T <= 64, 128 threads per group (E = 32)
  // or 256 (E = 16); two groups, three slots
  int T = (64 * 1024) / (16 * PL::N);
  if (T > 64) T = 64;
  if (T < 8 || g.N % T) return false;
  tp.lT = 31 - __builtin_clz((unsigned)T);
  tp.G = 2;
  tp.NS = 3;
  tp.ls = PL::N + 2;
  if (T * PL::TPL > 256) return false;
  if (PL::TPL > 32 && tp.G * T + tp.G + 1 > 16) return false;   // named barrier ids
  const size_t tile = (size_t)PL::N * T * 16, lines = (size_t)T * tp.ls * 16;
  const size_t slot = ((tile > lines ? tile : lines) + 1023) & ~(size_t)1023;
  tp.smem = 1024 + 1024 + (((size_t)PL::twsize() * 16 + 1023) & ~(size_t)1023) +
            (((size_t)PL::N * 8 + 1023) & ~(size_t)1023) + tp.NS * slot;
  return tp.smem <= 227 * 1024;
}

// 3-D map over X[l][m][n] as doubles {2N, M, L}, box {16 doubles (8 points), 1 node, min(L, 256)}
bool time_map(const Geometry &g, double2 *base, CUtensorMap &tm) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * g.N, (cuuint64_t)g.M, (cuuint64_t)g.L};
  const cuuint64_t strides[2] = {(cuuint64_t)g.N * 16, (cuuint64_t)g.M * g.N * 16};
  const cuuint32_t box[3] = {16, 1, (cuuint32_t)(g.L < 256 ? g.L : 256)};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             tfft_promo256() ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LL>
cudaError_t launch_tfft_l(const Geometry &g, const StaticTables &st, const AlphaTables *at, double2 *X,
                          const double2 *x2, double2 *u, bool inverse, unsigned long long *diff_slot, int overwrite,
                          cudaStream_t s) {
  using PL = rfft::Plan<LL, 5>;
  TfftPlan tp;
  if (!tfft_plan<PL>(g, tp)) return cudaErrorInvalidValue;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CUtensorMap tmx, tmu;
  if (!time_map(g, inverse ? (double2 *)x2 : X, tmx) || !time_map(g, u, tmu)) return cudaErrorNotSupported;
  const void *fn = inverse ? (const void *)tfft_pipe_kernel<PL, true> : (const void *)tfft_pipe_kernel<PL, false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tp.smem);
  if (e != cudaSuccess) return e;
  const int threads = tp.G * (1 << tp.lT) * PL::TPL;
  const int nitems = g.M * (g.N >> tp.lT);
  AlphaTables a = at ? *at : AlphaTables{};
  if (inverse)
    tfft_pipe_kernel<PL, true><<<sms, threads, tp.smem, s>>>(tmx, tmu, g, st, a, X, u, tp.lT, tp.G, tp.NS, tp.ls,
                                                             nitems, diff_slot, overwrite, tfft_prefetch(), tfft_pair());
  else
    tfft_pipe_kernel<PL, false><<<sms, threads, tp.smem, s>>>(tmx, tmu, g, st, a, X, u, tp.lT, tp.G, tp.NS, tp.ls,
                                                              nitems, nullptr, 0, 0, tfft_pair());
  return cudaGetLastError();
}

template <int MM>
cudaError_t launch_fused(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X, double2 *Yb,
                         unsigned *done, cudaStream_t s) {
  using PL = rfft::Plan<10, 5>;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int YR = MM == 3 ? 1 : 4 / MM;
  int nb = st.nsolve;
  CUtensorMap tmi, tmc;
  if (!blocked_map(g, Yb, 2 * kBW, 1, g.nx / kBW, CU_TENSOR_MAP_SWIZZLE_NONE, tmi) ||
      !blocked_map(g, Yb, 8, 256, 1, CU_TENSOR_MAP_SWIZZLE_64B, tmc))
    return cudaErrorNotSupported;
  const size_t slot = ((size_t)4 * (1024 + 2) * 16 + 1023) & ~(size_t)1023;
  const size_t smem = 1024 + 1024 + (((size_t)(PL::twsize() + 1024) * 16 + 1023) & ~(size_t)1023) + 3 * slot;
  const void *fn = (const void *)spatial_fused_kernel<MM>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, smem)) != cudaSuccess) return e;
  if (per < 1) return cudaErrorInvalidConfiguration;
  if ((e = cudaMemsetAsync(done, 0, 2 * (size_t)nb * sizeof(unsigned), s)) != cudaSuccess) return e;
  Geometry gg = g;
  StaticTables sst = st;
  AlphaTables aat = at;
  double2 *xx = X, *yy = Yb;
  int yr = YR;
  unsigned *dd = done;
  void *args[] = {(void *)&tmi, (void *)&tmc, &gg, &sst, &aat, &xx, &yy, &yr, &nb, &dd};
  // cooperative: all CTAs resident (the cross-CTA dependency waits need it)
  e = cudaLaunchCooperativeKernel(fn, dim3(sms), dim3(256), args, smem, s);
  record_launch(s);
  return e;
}

}  // namespace

// Measured on config 5: 63 ms against 46-50 ms for the three launches — ncu shows the same
// 206 GB of DRAM traffic (three 64 MB slots in flight do not stay in the 126 MB L2), 38 % fp64,
// instruction-cache stalls from the three unrolled item bodies.  Kept as an A/B option only
// (PINT_FUSED=1, experiments build).
bool spatial_fused_supported(const Geometry &g, const StaticTables &st) {
  const char *e = experiment_env("PINT_FUSED");
  if (!e || !atoi(e)) return false;
  return g.dim == 2 && g.pow2 && g.lognx == 10 && g.logny == 10 && g.M <= 4 && st.P == 1 && !st.packed &&
         st.nsolve >= 1;
}

cudaError_t launch_spatial_fused(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                                 double2 *Yb, unsigned *sync, cudaStream_t s) {
  if (!spatial_fused_supported(g, st) || Yb == X) return cudaErrorInvalidValue;
  switch (g.M) {
    case 1: return launch_fused<1>(g, st, at, X, Yb, sync, s);
    case 2: return launch_fused<2>(g, st, at, X, Yb, sync, s);
    case 3: return launch_fused<3>(g, st, at, X, Yb, sync, s);
    default: return launch_fused<4>(g, st, at, X, Yb, sync, s);
  }
}

bool spatial_pipe_geometry(const Geometry &g) {
  PipePlan pp;
  return pipe_plan(g, pp);
}

bool spatial_pipe_supported(const Geometry &g, const StaticTables &st) {
  return (!st.packed || st.xpair) && spatial_pipe_geometry(g);
}

cudaError_t launch_spatial_pipe(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                                double2 *Yb, cudaStream_t s, const double2 *spec) {
  PipePlan pp;
  if ((st.packed && !st.xpair) || !pipe_plan(g, pp) || Yb == X) return cudaErrorInvalidValue;
  const bool node = st.P == 1;
  const int units = st.nsolve;
#define PINT_PIPE(LXX, LYY, MMM) \
  if (g.lognx == LXX && g.logny == LYY && g.M == MMM) return launch_pipe_dispatch<LXX, LYY, MMM>(g, st, at, pp, X, Yb, units, node, s, spec);
#define PINT_PIPE_M(LXX, LYY) PINT_PIPE(LXX, LYY, 1) PINT_PIPE(LXX, LYY, 2) PINT_PIPE(LXX, LYY, 3) PINT_PIPE(LXX, LYY, 4)
  PINT_PIPE_M(9, 9) PINT_PIPE_M(10, 10) PINT_PIPE_M(9, 10) PINT_PIPE_M(10, 9) PINT_PIPE_M(11, 11) PINT_PIPE_M(10, 11)
  PINT_PIPE_M(11, 10)
#undef PINT_PIPE_M
#undef PINT_PIPE
  return cudaErrorInvalidValue;
}

bool tfft_pipe_supported(const Geometry &g, const StaticTables &st) {
  if (g.dim != 2 || st.packed || g.logL < 7 || g.logL > 10) return false;
  TfftPlan tp;
  switch (g.logL) {
    case 7: return tfft_plan<rfft::Plan<7, 5>>(g, tp);
    case 8: return tfft_plan<rfft::Plan<8, 5>>(g, tp);
    case 9: return tfft_plan<rfft::Plan<9, 5>>(g, tp);
    default: return tfft_plan<rfft::Plan<10, 5>>(g, tp);
  }
}

cudaError_t launch_tfft_pipe(const Geometry &g, const StaticTables &st, const AlphaTables *at, double2 *X,
                             const double2 *x2, double2 *u, bool inverse, unsigned long long *diff_slot, int overwrite,
                             cudaStream_t s) {
  switch (g.logL) {
    case 7: return launch_tfft_l<7>(g, st, at, X, x2, u, inverse, diff_slot, overwrite, s);
    case 8: return launch_tfft_l<8>(g, st, at, X, x2, u, inverse, diff_slot, overwrite, s);
    case 9: return launch_tfft_l<9>(g, st, at, X, x2, u, inverse, diff_slot, overwrite, s);
    case 10: return launch_tfft_l<10>(g, st, at, X, x2, u, inverse, diff_slot, overwrite, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pint
