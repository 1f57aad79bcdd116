// sm_100a kernels of libpint: one alpha-circulant preconditioned Richardson iteration
// (arXiv 2103.12571, Alg. 1, correction form) on complex fp64 data u[l][m][n].
//
//   fwd_kernel        (i)+(ii)+(iii): residual w - C u, alpha^{l/L} scale,
//                     L-point DIF FFT along time in shared memory (Lemma P:164-171),
//                     S_k^{-1} node transform                         u -> X
//   pcr_*_kernel      (iv) 1-D: (I - d_km dT A) x2 = x1 by parallel cyclic reduction on
//                     the constant-coefficient cyclic tridiagonal, row-sum carried   X -> X|Y
//   fft2d_*_kernel    (iv) 2-D: x2 = F^{-1}[F x1 / (1 - s lambda)] (3 passes)        X -> X
//   bwd_kernel        (v): G_k^{-1} S_k, inverse DIT FFT along time from
//                     bit-reversed order, alpha^{-l/L}/L, u += c    X -> u
//
// Design notes: the arithmetic intensity is low (< 4 flop/B, fp64), so the
// kernels are organised around full-tile shared-memory staging with 16-byte coalesced global
// accesses and are measured against the HBM roof; the FFT-heavy ones end up latency bound on
// shared memory and fp64 dependencies (§5b).  No tensor cores: no dense contraction on this path.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "device_common.cuh"
#include "internal.h"
#include "residual.cuh"   // residual_point (shared with generic.cu)

namespace pint {

// ---------------------------------------------------------------------------------------------
// residual of one (l, n) for all nodes: r_m = w_m - u_m + dT sum_j Q_mj (A u_j) + u_{l-1, M-1}
// (C = I_L (x) C_coll + E (x) H; w_0 = u0 replicated, w_{l>0} = 0 since b == 0)

// ---------------------------------------------------------------------------------------------
// Time-transform tile kernels.  Tile: all l x all m x T consecutive n, element (l, m, t) at
// sm[sidx<false>((l*M + m)*T + t)] (row index l*M + m; a "row" is T consecutive n of one (l, m)).
//
// fwd_kernel<M, RESID=true,  NODE=true>   1-D:  u -> X = S_p^{-1} FFT_l(alpha^{l/L} (w - C u))
// fwd_kernel<M, RESID=false, NODE=false>  2-D:  X (= alpha^{l/L} r from residual2d_kernel) -> FFT_l in place
// bwd_kernel<M, NODE=true>                1-D:  u += alpha^{-l/L}/L IFFT_p(G_p^{-1} S_p X2)
// bwd_kernel<M, NODE=false>               2-D:  u += alpha^{-l/L}/L IFFT_p(X2)  (G^{-1}S applied in the row pass)

constexpr int kTileThreads = 256;
constexpr int kTileMinBlocks = 3;   // time tiles: radix <= 8, 80 registers
constexpr int kSpaceMinBlocks = 2;  // spatial FFT passes: radix <= 16, 128 registers

// PACK (Hermitian mode, real data, 1 rank): column t of the tile is the complex time series
// r(n') + i r(n' + N/2), n' = n0 + t < N/2; after the FFT the node step unpacks X_k from the slots
// of k and L - k (both in the tile), applies S_k^{-1} and writes unit q's lines (X + q M N) at n'
// and n' + N/2.
template <int M, bool RESID, bool NODE, bool PACK = false, int HW = 1>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    fwd_kernel(Geometry g, StaticTables st, AlphaTables at, const double2 *__restrict__ u,
               double2 *__restrict__ X, int T) {
  extern __shared__ double2 sm[];
  const int lT = 31 - __clz(T);
  const int n0 = blockIdx.x * T;
  const int L = g.L;
  const size_t plane = (size_t)M * g.N;
  const int rows = L * M;
  const int all = rows * T;
  for (int i = threadIdx.x; i < g.L; i += blockDim.x) sm[all + i] = __ldg(st.twL + i);   // time twiddles
  if (RESID) {
    // (i) residual + alpha^{l/L} scale, one (l, t) per work item
    const int items = L * T;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int t = it & (T - 1), l = it >> lT;
      double2 r[M];
      residual_point<M, PACK, HW>(g, st, u, l, n0 + t, r);
      const double sc = __ldg(at.scale_fwd + l);
      if (PACK) {
        double2 r2[M];
        residual_point<M, PACK, HW>(g, st, u, l, n0 + t + g.N / 2, r2);
#pragma unroll
        for (int m = 0; m < M; ++m) sm[sidx<false>((l * M + m) * T + t)] = make_double2(r[m].x * sc, r2[m].x * sc);
      } else {
#pragma unroll
        for (int m = 0; m < M; ++m) sm[sidx<false>((l * M + m) * T + t)] = cscale(r[m], sc);
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
      const int t = idx & (T - 1), row = idx >> lT;
      cp_async16(sm + sidx<false>(idx), X + (size_t)row * g.N + n0 + t);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  // (ii) L-point DIF FFT along l for the M*T columns
  fft_dif<3, false>(sm, M * T, 1, M * T, L, g.logL, sm + all);   // twiddles staged behind the tile
  if (PACK) {
    // (iii) unpack X_k (k <= L/2) from the slots of k and L - k, then S_k^{-1}; one (unit, m) per item
    for (int it = threadIdx.x; it < st.nsolve * M; it += blockDim.x) {
      const int m = it % M, q = it / M;
      const int p = __ldg(st.slots + q), kf = brev(p, g.logL), pc = brev((L - kf) & (L - 1), g.logL);
      double2 srow[M];
#pragma unroll
      for (int j = 0; j < M; ++j) srow[j] = __ldg(at.Sinv + ((size_t)p * M + m) * M + j);
      double2 *dst = X + ((size_t)q * M + m) * g.N + n0;
      for (int t = 0; t < T; ++t) {
        double2 at_ = make_double2(0.0, 0.0), ab = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const double2 a = sm[sidx<false>((p * M + j) * T + t)], b = sm[sidx<false>((pc * M + j) * T + t)];
          double2 xt, xb;
          if (pc == p) {
            xt = make_double2(a.x, 0.0);
            xb = make_double2(a.y, 0.0);
          } else {
            xt = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
            xb = make_double2(0.5 * (a.y + b.y), 0.5 * (b.x - a.x));
          }
          at_ = cfma(srow[j], xt, at_);
          ab = cfma(srow[j], xb, ab);
        }
        dst[t] = at_;
        dst[t + g.N / 2] = ab;
      }
    }
  } else if (NODE) {
    // (iii) node transform, one (p, m) row of T outputs per work item (row m of S_p^{-1} loaded once)
    for (int it = threadIdx.x; it < rows; it += blockDim.x) {
      const int m = it % M, p = it / M;
      double2 srow[M];
#pragma unroll
      for (int j = 0; j < M; ++j) srow[j] = __ldg(at.Sinv + ((size_t)p * M + m) * M + j);
      double2 *dst = X + (size_t)p * plane + (size_t)m * g.N + n0;
      for (int t = 0; t < T; ++t) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) acc = cfma(srow[j], sm[sidx<false>((p * M + j) * T + t)], acc);
        dst[t] = acc;
      }
    }
  } else {
    // (P > 1: the node transform runs after the cross-rank DFT) four-step twiddle e^{-2 pi i rank kappa/L}
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
      const int t = idx & (T - 1), row = idx >> lT;
      double2 v = sm[sidx<false>(idx)];
      if (st.twr) v = cmul(v, __ldg(st.twr + row / M));
      X[(size_t)row * g.N + n0 + t] = v;
    }
  }
}

// 1-D forward tile with the u tile staged by the TMA unit (one rank, complex storage, 3-point
// stencils, T = 4): same arithmetic as fwd_kernel<M, true, true> without its per-thread stencil
// loads (which kept the L1 data pipe at 90 %, half of it global-load wavefronts for 64-byte rows).
// Persistent (one CTA per SM) with two consumer groups of 256 threads over a ring of NS slots:
// slot = the tile [l][m][t] (box {T, M, L} of the tensor map over u, 64-byte swizzle: element a
// at swz64(a)), then the halo columns n0 - 1 and n0 + T as [l][m] arrays (16-byte box columns;
// wrapped column indices make the line periodic).  The group that finishes tile k refills its
// slot with tile k + NS (ring order = tile order).  Thread l of a group evaluates the residual of
// step l for all t and m with a sliding window along t (it first reads the H-term row l - 1 into
// registers; a group barrier separates those reads from the in-place writes of r), then the
// group runs the L-point DIF FFT on the swizzled tile (twiddles staged once per CTA) and
// S_p^{-1} writes X.
constexpr int kFwdTmaGT = 256, kFwdTmaG = 2;

template <int M>
__global__ void __launch_bounds__(kFwdTmaGT * kFwdTmaG, 1)
    fwd1d_tma_kernel(const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmh,
                     const __grid_constant__ CUtensorMap tmx, Geometry g, StaticTables st, AlphaTables at, int NS,
                     int ntiles) {
  constexpr int T = 4;
  extern __shared__ __align__(16) unsigned char smraw_[];
  unsigned char *smb;   // 1024-byte aligned (the 64-byte swizzle pattern follows smem address bits 7-8)
  {
    const unsigned a = (unsigned)__cvta_generic_to_shared(smraw_);
    smb = smraw_ + (((a + 1023u) & ~1023u) - a);
  }
  const int L = g.L, N = g.N;
  const int rows = L * M, all = rows * T;
  const size_t slot_elems = (size_t)rows * (T + 2);
  uint64_t *full = reinterpret_cast<uint64_t *>(smb);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smb + 64);
  double2 *tw = reinterpret_cast<double2 *>(smb + 1024);
  double2 *ring = reinterpret_cast<double2 *>(smb + 1024 + (((size_t)L * sizeof(double2) + 1023) & ~(size_t)1023));
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < NS; ++s2) {
      mbar_init(full + s2, 1);
      slot_item[s2] = -1;
    }
    mbar_init_fence();
  }
  for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = __ldg(st.twL + i);
  __syncthreads();
  auto issue = [&](int k) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= ntiles) return;
    const int n0 = it * T;
    uint64_t *bar = full + k % NS;
    double2 *sl = ring + (size_t)(k % NS) * slot_elems;
    mbar_arrive_expect_tx(bar, (unsigned)((all + 2 * rows) * sizeof(double2)));
    tma_load_3d(sl, &tmu, 2 * n0, 0, 0, bar);
    tma_load_3d(sl + all, &tmh, 2 * ((n0 - 1 + N) & (N - 1)), 0, 0, bar);
    tma_load_3d(sl + all + rows, &tmh, 2 * ((n0 + T) & (N - 1)), 0, 0, bar);
    slot_item[k % NS] = k;
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  const int gid = threadIdx.x / kFwdTmaGT;
  const Grp gp{(int)threadIdx.x - gid * kFwdTmaGT, kFwdTmaGT, 1 + gid};
  const int l = gp.tid;
  const double wl = g.wx[2], wc = g.wx[3], wr = g.wx[4];
  for (int k = gid;; k += kFwdTmaG) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= ntiles) break;
    const int n0 = it * T;
    double2 *sm = ring + (size_t)(k % NS) * slot_elems;
    const double2 *hl = sm + all, *hr = hl + rows;
    auto U = [&](int ll, int m, int t) -> double2 & { return sm[swz64((ll * M + m) * T + t)]; };
    while (slot_item[k % NS] != k) __nanosleep(32);
    mbar_wait(full + k % NS, (unsigned)((k / NS) & 1));
    // (i) residual + alpha^{l/L}, one step l per thread
    double2 h[T];
    if (l < L) {
#pragma unroll
      for (int t = 0; t < T; ++t) h[t] = l == 0 ? __ldg(st.u0 + n0 + t) : U(l - 1, M - 1, t);
    }
    gp.sync();   // every H-term read of row l - 1 precedes the writes of row l - 1
    if (l < L) {
      const double sc = __ldg(at.scale_fwd + l);
      double2 lv[M], cv[M], rv[M];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        lv[j] = hl[l * M + j];
        cv[j] = U(l, j, 0);
      }
#pragma unroll
      for (int t = 0; t < T; ++t) {
#pragma unroll
        for (int j = 0; j < M; ++j) rv[j] = t + 1 < T ? U(l, j, t + 1) : hr[l * M + j];
        double2 Au[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
          Au[j].x = fma(wl, lv[j].x, fma(wc, cv[j].x, wr * rv[j].x));
          Au[j].y = fma(wl, lv[j].y, fma(wc, cv[j].y, wr * rv[j].y));
        }
#pragma unroll
        for (int m = 0; m < M; ++m) {
          double2 acc = csub(h[t], cv[m]);
          if (st.v) acc = cadd(acc, __ldg(st.v + ((size_t)l * M + m) * N + n0 + t));   // forcing part of w
#pragma unroll
          for (int j = 0; j < M; ++j) {
            const double q = g.dTQ[m * M + j];
            acc.x = fma(q, Au[j].x, acc.x);
            acc.y = fma(q, Au[j].y, acc.y);
          }
          U(l, m, t) = cscale(acc, sc);   // this row's u values at t are no longer needed
        }
#pragma unroll
        for (int j = 0; j < M; ++j) {
          lv[j] = cv[j];
          cv[j] = rv[j];
        }
      }
    }
    gp.sync();
    // (ii) L-point DIF FFT along l for the M*T columns, (iii) S_p^{-1} -> X
    fft_dif_g<3>(sm, M * T, 1, M * T, g.logL, tw, gp);
    // (iii) S_p^{-1} in place, one (p, m) row per item; the M rows of a slot sit on adjacent lanes
    // of one warp, so the reads of a slot precede its writes by a warp barrier (no group barrier)
    {
      constexpr int PPW = 32 / M;                 // slots per warp pass
      const int lane = gp.tid & 31, wg = gp.tid >> 5, nwg = gp.nt >> 5;
      const int pl = lane / M, m = lane - pl * M;
      for (int p0 = wg * PPW; p0 < L; p0 += nwg * PPW) {
        const int p = p0 + pl;
        const bool act = pl < PPW && p < L;
        double2 acc[T];
        if (act) {
          double2 srow[M];
#pragma unroll
          for (int j = 0; j < M; ++j) srow[j] = __ldg(at.Sinv + ((size_t)p * M + m) * M + j);
#pragma unroll
          for (int t = 0; t < T; ++t) {
            acc[t] = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < M; ++j) acc[t] = cfma(srow[j], U(p, j, t), acc[t]);
          }
        }
        __syncwarp();
        if (act) {
#pragma unroll
          for (int t = 0; t < T; ++t) U(p, m, t) = acc[t];
        }
      }
    }
    fence_proxy_async_smem();   // the generic writes of the slot before the TMA store reads it
    gp.sync();
    if (gp.tid == 0) {          // X[p][m][n0 .. n0 + T) <- the tile; refill once the store has read it
      tma_store_3d(&tmx, 2 * n0, 0, 0, sm);
      bulk_commit();
      bulk_wait_read();
      issue(k + NS);
    }
  }
  if (threadIdx.x % kFwdTmaGT == 0) bulk_wait_all();   // the last stores complete before exit
}

__device__ __forceinline__ unsigned long long dbl_bits(double v) { return (unsigned long long)__double_as_longlong(v); }

// PACK (Hermitian mode, 1 rank): unit q's solved lines at n' and n' + N/2 are node-transformed
// (G_k^{-1} S_k) and repacked into the slots of k and L - k (w = y(n') + i y(n' + N/2) and its
// conjugate counterpart); the inverse FFT's real / imaginary parts update u at n' and n' + N/2.
template <int M, bool NODE, bool PACK = false>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    bwd_kernel(const __grid_constant__ CUtensorMap tmx2, const __grid_constant__ CUtensorMap tmu, int tma, Geometry g,
               StaticTables st, AlphaTables at, const double2 *__restrict__ X2,
               double2 *__restrict__ u, int T, unsigned long long *diff_slot, int overwrite) {
  // tma (complex storage): the tile [L][M][T] is the unswizzled tensor box {2 T doubles, M nodes,
  // min(L, 256) steps} of X2 / u: tensor load in, and the update u += c leaves as a TMA tensor
  // reduce-add performed at the L2 (overwrite: a tensor store), as in tfft_bwd_tma_kernel
  extern __shared__ __align__(128) double2 sm[];
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t bar;
  const int lT = 31 - __clz(T);
  const int n0 = blockIdx.x * T;
  const int L = g.L;
  const int rows = L * M;
  const int all = rows * T;
  if (PACK) {
    for (int it = threadIdx.x; it < st.nsolve * T; it += blockDim.x) {
      const int t = it & (T - 1), q = it >> lT;
      const int p = __ldg(st.slots + q), kf = brev(p, g.logL), pc = brev((L - kf) & (L - 1), g.logL);
      double2 vt[M], vb[M];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const double2 *src = X2 + ((size_t)q * M + j) * g.N + n0 + t;
        vt[j] = __ldg(src);
        vb[j] = __ldg(src + g.N / 2);
      }
      const double2 *SG = at.SG + (size_t)p * M * M;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double2 yt = make_double2(0.0, 0.0), yb = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const double2 c = __ldg(SG + m * M + j);
          yt = cfma(c, vt[j], yt);
          yb = cfma(c, vb[j], yb);
        }
        sm[sidx<false>((p * M + m) * T + t)] = make_double2(yt.x - yb.y, yt.y + yb.x);               // yt + i yb
        if (pc != p) sm[sidx<false>((pc * M + m) * T + t)] = make_double2(yt.x + yb.y, yb.x - yt.y);  // conj yt + i conj yb
      }
    }
    __syncthreads();
  } else {
    if (tma) {
      if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        mbar_arrive_expect_tx(&bar, (unsigned)(all * sizeof(double2)));
        for (int lb = 0; lb < L; lb += 256) tma_load_3d(sm + (size_t)lb * M * T, &tmx2, 2 * n0, 0, lb, &bar);
      }
      __syncthreads();
      mbar_wait(&bar, 0);
    } else {
    // async tile load X2[p][m][n0..n0+T) -> sm, and an L2 prefetch of the u tile for the update
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
      const int t = idx & (T - 1), row = idx >> lT;
      cp_async16(sm + sidx<false>(idx), X2 + (size_t)row * g.N + n0 + t);
    }
    if (!overwrite)
      for (int row = threadIdx.x; row < rows; row += blockDim.x) prefetch_l2(u + (size_t)row * g.N + n0);
    cp_async_wait_all();
    __syncthreads();
    }
  }
  if (!NODE && st.twr) {  // P > 1: inverse four-step twiddle e^{+2 pi i rank kappa/L}
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x)
      sm[sidx<false>(idx)] = cmulc(sm[sidx<false>(idx)], __ldg(st.twr + (idx >> lT) / M));
    __syncthreads();
  }
  if (NODE && !PACK) {
    // (v-a) y = G_p^{-1} S_p x2 in place, one (p, t) per work item
    const int items = L * T;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int t = it & (T - 1), p = it >> lT;
      double2 v[M];
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = sm[sidx<false>((p * M + j) * T + t)];
      const double2 *SG = at.SG + (size_t)p * M * M;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) acc = cfma(__ldg(SG + m * M + j), v[j], acc);
        sm[sidx<false>((p * M + m) * T + t)] = acc;
      }
    }
    __syncthreads();
  }
  // (v-b) inverse DIT FFT from bit-reversed p to natural l
  fft_dit_inv<3, false>(sm, M * T, 1, M * T, L, g.logL, st.twL);   // (staging measured slower here)
  // (v-c) u += alpha^{-l/L}/L c, loads batched for memory-level parallelism
  double dmax = 0.0;
  constexpr int kB = 8;
  if (!PACK && tma) {
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
      const int row = idx >> lT, l = row / M;
      const double2 c = cscale(sm[idx], __ldg(at.scale_bwd + l));
      sm[idx] = c;
      if (l == L - 1 && diff_slot) {
        const double2 dd = overwrite ? csub(c, u[(size_t)row * g.N + n0 + (idx & (T - 1))]) : c;
        dmax = nanmax(dmax, hypot(dd.x, dd.y));
      }
    }
    fence_proxy_async_smem();
    __syncthreads();   // also: the old last-step values (overwrite form) were read before the store
    if (threadIdx.x == 0) {
      for (int lb = 0; lb < L; lb += 256) {
        if (overwrite) tma_store_3d(&tmu, 2 * n0, 0, lb, sm + (size_t)lb * M * T);
        else tma_reduce_add_3d(&tmu, 2 * n0, 0, lb, sm + (size_t)lb * M * T);
      }
      bulk_commit();
    }
  } else
  for (int base = threadIdx.x; base < all; base += kB * blockDim.x) {
    double2 uo[kB], uo2[kB];
    double sc[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int idx = base + k * blockDim.x;
      if (idx < all) {
        const int t = idx & (T - 1), row = idx >> lT;
        const bool need_old = !overwrite || (diff_slot && row / M == L - 1);
        if (PACK) {   // real storage
          const double *ur = (const double *)u + (size_t)row * g.N + n0 + t;
          uo[k] = make_double2(need_old ? ur[0] : 0.0, 0.0);
          uo2[k] = make_double2(need_old ? ur[g.N / 2] : 0.0, 0.0);
        } else {
          uo[k] = need_old ? u[(size_t)row * g.N + n0 + t] : make_double2(0.0, 0.0);
        }
        sc[k] = __ldg(at.scale_bwd + row / M);
      }
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int idx = base + k * blockDim.x;
      if (idx < all) {
        const int t = idx & (T - 1), row = idx >> lT;
        const double2 c = cscale(sm[sidx<false>(idx)], sc[k]);
        if (PACK) {   // real points n' (Re c) and n' + N/2 (Im c), stored real
          const double n1 = overwrite ? c.x : uo[k].x + c.x;
          const double n2 = overwrite ? c.y : uo2[k].x + c.y;
          double *ur = (double *)u + (size_t)row * g.N + n0 + t;
          ur[0] = n1;
          ur[g.N / 2] = n2;
          if (row / M == L - 1) dmax = nanmax(dmax, nanmax(fabs(n1 - uo[k].x), fabs(n2 - uo2[k].x)));
        } else {
          u[(size_t)row * g.N + n0 + t] = overwrite ? c : cadd(uo[k], c);   // direct form: u = C_a^{-1} r
          if (row / M == L - 1) {
            const double2 dd = overwrite ? csub(c, uo[k]) : c;
            dmax = nanmax(dmax, hypot(dd.x, dd.y));
          }
        }
      }
    }
  }
  if (diff_slot) {
    for (int o = 16; o > 0; o >>= 1) dmax = nanmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = nanmax(v, red[w]);
      atomicMax(diff_slot, dbl_bits(v));  // non-negative doubles order like their bit patterns
    }
  }
  if (!PACK && tma && threadIdx.x == 0) bulk_wait_read();   // the tile stays until the TMA unit has read it
}

// ---------------------------------------------------------------------------------------------
// 2-D time-transform tiles: one node m per CTA (the node transforms live in the row passes), so
// the tile is all l x T consecutive n with T = 64 KB / (16 L) (T = 8 for L = 512: 128-byte rows).
// Element (l, t) at sm[sidx<false>(l*T + t)]; CTA b covers node m = b / (N/T), n0 = (b % (N/T)) * T.

__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tfft_fwd_kernel(Geometry g, StaticTables st, double2 *__restrict__ X, int T) {
  extern __shared__ double2 sm[];
  const int lT = 31 - __clz(T);
  const int per = g.N / T;
  const int m = blockIdx.x / per;
  const int n0 = (blockIdx.x - m * per) * T;
  const size_t lstride = (size_t)g.M * g.N;
  double2 *base = X + (size_t)m * g.N + n0;
  const int all = g.L * T;
  for (int i = threadIdx.x; i < g.L; i += blockDim.x) sm[all + i] = __ldg(st.twL + i);   // time twiddles
  for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
    const int t = idx & (T - 1), l = idx >> lT;
    cp_async16(sm + sidx<false>(idx), base + (size_t)l * lstride + t);
  }
  cp_async_wait_all();
  __syncthreads();
  fft_dif<3, false>(sm, T, 1, T, g.L, g.logL, sm + all);   // twiddles staged behind the tile
  for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
    const int t = idx & (T - 1), p = idx >> lT;
    double2 v = sm[sidx<false>(idx)];
    if (st.twr) v = cmul(v, __ldg(st.twr + p));   // P > 1: four-step twiddle
    base[(size_t)p * lstride + t] = v;
  }
}

// PACK (Hermitian mode, real data): the time series of column n' < N/2 is w = y(n') + i y(n' + N/2);
// slot p of it is assembled from the unit planes of X2 (unit q = unitof[p]: y_k; -1 - q: conj y_k
// of the unit of L - k), and the real/imaginary parts of the inverse transform update the two
// real points n' and n' + N/2 of u (imaginary parts of u are kept at 0).
template <bool PACK>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tfft_bwd_kernel(Geometry g, StaticTables st, AlphaTables at, const double2 *__restrict__ X2,
                    double2 *__restrict__ u, int T, unsigned long long *diff_slot, int overwrite) {
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  const int lT = 31 - __clz(T);
  const int NC = PACK ? g.N / 2 : g.N;     // time-series columns
  const int per = NC / T;
  const int m = blockIdx.x / per;
  const int n0 = (blockIdx.x - m * per) * T;
  const size_t lstride = (size_t)g.M * g.N;
  // packed: the tile's first column as a point index and the partner offset of its pairs
  const bool xp = PACK && st.xpair;
  const int np0 = xp ? ((n0 >> (g.lognx - 1)) << g.lognx) + (n0 & (g.nx / 2 - 1)) : n0;
  const int poff = xp ? g.nx / 2 : g.N / 2;
  const double2 *xb = X2 + (size_t)m * g.N + (PACK ? np0 : n0);
  double2 *ub = u + (size_t)m * g.N + n0;
  const int all = g.L * T;
  if (PACK) {
    // one read of unit q's y_k (points n' and n' + N/2) fills both slots of the tile:
    // slot p_k <- y(n') + i y(n' + N/2), slot p_{L-k} <- conj y(n') + i conj y(n' + N/2)
    constexpr int kL = 4;
    const int units = st.nsolve * T;
    for (int i0 = threadIdx.x; i0 < units; i0 += kL * blockDim.x) {
      double2 a[kL], b[kL];
#pragma unroll
      for (int k = 0; k < kL; ++k) {
        const int idx = i0 + k * blockDim.x;
        if (idx < units) {
          const int t = idx & (T - 1), q = idx >> lT;
          const double2 *yp = xb + (size_t)q * g.M * g.N + t;
          a[k] = __ldg(yp);
          b[k] = __ldg(yp + poff);
        }
      }
#pragma unroll
      for (int k = 0; k < kL; ++k) {
        const int idx = i0 + k * blockDim.x;
        if (idx < units) {
          const int t = idx & (T - 1), q = idx >> lT;
          const int p = __ldg(st.slots + q), kf = brev(p, g.logL);
          const int pc = brev((g.L - kf) & (g.L - 1), g.logL);
          sm[sidx<false>(p * T + t)] = make_double2(a[k].x - b[k].y, a[k].y + b[k].x);          // a + i b
          if (pc != p) sm[sidx<false>(pc * T + t)] = make_double2(a[k].x + b[k].y, b[k].x - a[k].y);  // conj a + i conj b
        }
      }
    }
    __syncthreads();
  } else {
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
      const int t = idx & (T - 1), p = idx >> lT;
      cp_async16(sm + sidx<false>(idx), xb + (size_t)p * lstride + t);
    }
    cp_async_wait_all();
    __syncthreads();
  }
  if (st.twr) {  // P > 1: inverse four-step twiddle
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x)
      sm[sidx<false>(idx)] = cmulc(sm[sidx<false>(idx)], __ldg(st.twr + (idx >> lT)));
    __syncthreads();
  }
  fft_dit_inv<3, false>(sm, T, 1, T, g.L, g.logL, st.twL);   // (staging measured slower here)
  double dmax = 0.0;
  constexpr int kB = 8;
  for (int b0 = threadIdx.x; b0 < all; b0 += kB * blockDim.x) {
    double2 uo[kB], uo2[kB];
    double sc[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int idx = b0 + k * blockDim.x;
      if (idx < all) {
        const int t = idx & (T - 1), l = idx >> lT;
        const bool need_old = !overwrite || (diff_slot && l == g.L - 1);
        if (PACK) {   // real storage (u_dev holds doubles; same element offsets)
          const double *ur = (const double *)u + (size_t)m * g.N + np0 + (size_t)l * lstride + t;
          uo[k] = make_double2(need_old ? ur[0] : 0.0, 0.0);
          uo2[k] = make_double2(need_old ? ur[poff] : 0.0, 0.0);
        } else {
          uo[k] = need_old ? ub[(size_t)l * lstride + t] : make_double2(0.0, 0.0);
        }
        sc[k] = __ldg(at.scale_bwd + l);
      }
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int idx = b0 + k * blockDim.x;
      if (idx < all) {
        const int t = idx & (T - 1), l = idx >> lT;
        const double2 c = cscale(sm[sidx<false>(idx)], sc[k]);
        if (PACK) {
          // real points n' (Re c) and n' + N/2 (Im c), stored real
          const double n1 = overwrite ? c.x : uo[k].x + c.x;
          const double n2 = overwrite ? c.y : uo2[k].x + c.y;
          double *ur = (double *)u + (size_t)m * g.N + np0 + (size_t)l * lstride + t;
          ur[0] = n1;
          ur[poff] = n2;
          if (l == g.L - 1) dmax = nanmax(dmax, nanmax(fabs(n1 - uo[k].x), fabs(n2 - uo2[k].x)));
        } else {
          ub[(size_t)l * lstride + t] = overwrite ? c : cadd(uo[k], c);
          if (l == g.L - 1) {
            const double2 dd = overwrite ? csub(c, uo[k]) : c;
            dmax = nanmax(dmax, hypot(dd.x, dd.y));
          }
        }
      }
    }
  }
  if (diff_slot) {
    for (int o = 16; o > 0; o >>= 1) dmax = nanmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = nanmax(v, red[w]);
      atomicMax(diff_slot, dbl_bits(v));
    }
  }
}

// ---------------------------------------------------------------------------------------------
// TMA variants of the 2-D time tiles (complex storage, one rank or sharded; 2 T <= 256 doubles
// per box row).  The tile [L][T] is exactly the unswizzled box {2 T doubles, 1 node, min(L, 256)
// steps} of the 3-D map over X / x2 / u, so one thread moves it with cp.async.bulk.tensor (no
// per-thread address arithmetic or LSU traffic for the copies):
//   forward: tensor load, DIF, (P > 1: four-step twiddle), tensor store in place;
//   inverse: tensor load of x2, DIT, x alpha^{-l/L} / L in shared memory, and the update
//            u += c leaves as a TMA tensor REDUCTION (cp.reduce.async.bulk.tensor .add on the
//            FLOAT64 map, UTMAREDG): the fp64 add is performed at the L2, the old u never enters
//            the SM, and the CTA retires without waiting for a u round trip (the exposed latency
//            of tfft_bwd_kernel).  overwrite (direct form): a tensor store; the old last-step
//            values (T of them) are read early for the difference.
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tfft_fwd_tma_kernel(const __grid_constant__ CUtensorMap tmx, Geometry g, StaticTables st, int T) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ __align__(8) uint64_t bar;
  const int lT = 31 - __clz(T);
  const int per = g.N / T;
  const int m = blockIdx.x / per;
  const int n0 = (blockIdx.x - m * per) * T;
  const int all = g.L * T, LB = g.L < 256 ? g.L : 256;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
    mbar_arrive_expect_tx(&bar, (unsigned)(all * sizeof(double2)));
    for (int lb = 0; lb < g.L; lb += LB) tma_load_3d(sm + (size_t)lb * T, &tmx, 2 * n0, m, lb, &bar);
  }
  for (int i = threadIdx.x; i < g.L; i += blockDim.x) sm[all + i] = __ldg(st.twL + i);   // time twiddles
  __syncthreads();
  mbar_wait(&bar, 0);
  fft_dif<3, false>(sm, T, 1, T, g.L, g.logL, sm + all);
  if (st.twr) {   // P > 1: four-step twiddle
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) sm[idx] = cmul(sm[idx], __ldg(st.twr + (idx >> lT)));
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int lb = 0; lb < g.L; lb += LB) tma_store_3d(&tmx, 2 * n0, m, lb, sm + (size_t)lb * T);
    bulk_commit();
    bulk_wait_read();   // the tile must stay in shared memory until the TMA unit has read it
  }
}

__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tfft_bwd_tma_kernel(const __grid_constant__ CUtensorMap tmx2, const __grid_constant__ CUtensorMap tmu, Geometry g,
                        StaticTables st, AlphaTables at, const double2 *__restrict__ u, int T,
                        unsigned long long *diff_slot, int overwrite) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double red[32];
  __shared__ double2 uold[128];
  const int lT = 31 - __clz(T);
  const int per = g.N / T;
  const int m = blockIdx.x / per;
  const int n0 = (blockIdx.x - m * per) * T;
  const int all = g.L * T, LB = g.L < 256 ? g.L : 256;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
    mbar_arrive_expect_tx(&bar, (unsigned)(all * sizeof(double2)));
    for (int lb = 0; lb < g.L; lb += LB) tma_load_3d(sm + (size_t)lb * T, &tmx2, 2 * n0, m, lb, &bar);
  }
  if (overwrite && diff_slot && threadIdx.x < T)   // direct form: the old last-step values
    uold[threadIdx.x] = u[((size_t)(g.L - 1) * g.M + m) * g.N + n0 + threadIdx.x];
  __syncthreads();
  mbar_wait(&bar, 0);
  if (st.twr) {  // P > 1: inverse four-step twiddle
    for (int idx = threadIdx.x; idx < all; idx += blockDim.x) sm[idx] = cmulc(sm[idx], __ldg(st.twr + (idx >> lT)));
    __syncthreads();
  }
  fft_dit_inv<3, false>(sm, T, 1, T, g.L, g.logL, st.twL);
  double dmax = 0.0;
  for (int idx = threadIdx.x; idx < all; idx += blockDim.x) {
    const int l = idx >> lT;
    const double2 c = cscale(sm[idx], __ldg(at.scale_bwd + l));
    sm[idx] = c;
    if (l == g.L - 1) {
      const double2 dd = overwrite ? csub(c, uold[idx & (T - 1)]) : c;
      dmax = nanmax(dmax, hypot(dd.x, dd.y));
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int lb = 0; lb < g.L; lb += LB) {
      if (overwrite) tma_store_3d(&tmu, 2 * n0, m, lb, sm + (size_t)lb * T);
      else tma_reduce_add_3d(&tmu, 2 * n0, m, lb, sm + (size_t)lb * T);
    }
    bulk_commit();
  }
  if (diff_slot) {
    for (int o = 16; o > 0; o >>= 1) dmax = nanmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = nanmax(v, red[w]);
      atomicMax(diff_slot, dbl_bits(v));
    }
  }
  if (threadIdx.x == 0) bulk_wait_read();   // the tile must stay in shared memory until the TMA unit has read it
}

// ---------------------------------------------------------------------------------------------
// 2-D residual: X[l][m][n] = alpha^{l/L} (w - C u)[l][m][n] on spatial blocks BY x BX with a
// one-point halo staged in shared memory (all M nodes of one l per CTA).  Each warp stages whole
// halo rows (lanes along x: no index divisions), each thread then evaluates BX*BY/256 points.

// PACK (Hermitian mode): the CTA also evaluates the partner block BY rows lower by ny/2 and writes
// Z[l][m][n'] = alpha^{l/L} (Re r(n') + i Re r(n' + N/2)) for its top-half points n' (N/2 per plane).
// HW: halo width (1 for the 3-point operators, up to 3 for the kappa-6 / upwind-5 stencils);
// weights outside [-hx0, hx1] x [-hy0, hy1] are zero in g.wx / g.wy.
template <int M, bool PACK, int HW>
__global__ void __launch_bounds__(256, M <= 4 ? 4 : 2) residual2d_kernel(const __grid_constant__ CUtensorMap tmu, int tma,
                                                         Geometry g, StaticTables st, AlphaTables at,
                                                         const double2 *__restrict__ u,
                                                         double2 *__restrict__ X, int BX, int BY, int LG) {
  extern __shared__ __align__(128) double2 sm[];  // [1 + PACK][M][BY+2HW][BX+2HW]
  __shared__ __align__(8) uint64_t bar;
  const bool xp = PACK && st.xpair;   // packed partner (y, x + nx/2) instead of (y + ny/2, x)
  const int bxs = (xp ? g.nx / 2 : g.nx) / BX, bys = (PACK && !xp ? g.ny / 2 : g.ny) / BY;
  int b = blockIdx.x;
  // LG > 1: LG consecutive steps of one spatial block on consecutive CTAs, so the H-term plane
  // u_{l-1, M-1} of a block is read while the CTA of step l-1 streams the same lines (L2 hit)
  const int lo = LG > 1 ? b % LG : 0;
  if (LG > 1) b /= LG;
  const int bx = b % bxs; b /= bxs;
  const int by = b % bys;
  const int l = LG > 1 ? (b / bys) * LG + lo : b / bys;
  const int x0 = bx * BX, y0 = by * BY;
  const int W = BX + 2 * HW, H = BY + 2 * HW;
  const size_t plane = (size_t)M * g.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double sc = __ldg(at.scale_fwd + l);
  if constexpr (PACK) {
    // real storage: stage reals, real arithmetic; the CTA's block (hh = 0) and its partner ny/2
    // rows lower (hh = 1) give Z = Re r(n') + i Re r(n' + N/2)
    double *smr = (double *)sm;   // [2][M][H][W]
    const double *ur = (const double *)u + (size_t)l * plane;
    for (int r = warp; r < 2 * M * H; r += blockDim.x >> 5) {
      const int hh = r / (M * H), rr = r - hh * M * H;
      const int j = rr / H, yy = rr - j * H;
      const int y = (y0 + (xp ? 0 : hh * (g.ny / 2)) + yy - HW) & (g.ny - 1);
      const int xs = x0 + (xp ? hh * (g.nx / 2) : 0) - HW;
      const double *src = ur + (size_t)j * g.N + ((size_t)y << g.lognx);
      double *dst = smr + r * W;
      for (int xx = lane; xx < W; xx += 32) cp_async8(dst + xx, src + ((xs + xx) & (g.nx - 1)));
    }
    cp_async_wait_all();
    __syncthreads();
    for (int pt = threadIdx.x; pt < BX * BY; pt += blockDim.x) {
      const int ty = pt >> (31 - __clz(BX)), tx = pt & (BX - 1);   // BX: power of two
      const int n = ((y0 + ty) << g.lognx) + x0 + tx;
      double res[2][M];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int nn = n + hh * (xp ? g.nx / 2 : g.N / 2);
        // one rank: w (l = 0) or the H-term u_{l-1, M-1}
        const double base = l == 0 ? __ldg(st.u0 + nn).x : __ldg(ur - g.N + nn);
        double uc[M], Au[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const double *q = smr + ((hh * M + j) * H + ty + HW) * W + tx + HW;
          const double c = q[0];
          uc[j] = c;
          double acc = g.wx[3] * c;
#pragma unroll
          for (int o = -HW; o <= HW; ++o) {
            if (o == 0) continue;
            acc = fma(g.wx[3 + o], q[o], acc);
            acc = fma(g.wy[3 + o], q[o * W], acc);
          }
          Au[j] = acc;
        }
#pragma unroll
        for (int m = 0; m < M; ++m) {
          double acc = base - uc[m];
#pragma unroll
          for (int j = 0; j < M; ++j) acc = fma(g.dTQ[m * M + j], Au[j], acc);
          res[hh][m] = acc * sc;
        }
      }
#pragma unroll
      const int col = xp ? ((y0 + ty) << (g.lognx - 1)) + x0 + tx : n;   // packed column
#pragma unroll
      for (int m = 0; m < M; ++m) X[((size_t)l * M + m) * (g.N / 2) + col] = make_double2(res[0][m], res[1][m]);
    }
    return;
  } else {
  const double2 *ul = u + (size_t)l * plane;
  // a block whose halo does not wrap around the periodic boundary is one tensor box {2 W doubles, H
  // rows, M nodes} of u: one thread hands it to the TMA unit; the blocks on the boundary (2 of the
  // nx / BX block columns, 2 of the ny / BY block rows) stage their rows with cp.async
  const bool box = tma && x0 >= HW && x0 + BX + HW <= g.nx && y0 >= HW && y0 + BY + HW <= g.ny;
  if (box) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_init_fence();
      mbar_arrive_expect_tx(&bar, (unsigned)(M * H * W * sizeof(double2)));
      tma_load_3d(sm, &tmu, 2 * (x0 - HW), y0 - HW, l * M, &bar);
    }
  } else {
    for (int r = warp; r < M * H; r += blockDim.x >> 5) {
      const int j = r / H, yy = r - j * H;
      const int y = (y0 + yy - HW) & (g.ny - 1);
      const double2 *src = ul + (size_t)j * g.N + ((size_t)y << g.lognx);
      double2 *dst = sm + r * W;
      for (int xx = lane; xx < W; xx += 32) cp_async16(dst + xx, src + ((x0 + xx - HW) & (g.nx - 1)));
    }
  }
  // the H-term block (last node of step l - 1, or u0 for global step 0) is staged with the tile, so
  // the point loop below has no global load whose latency it would expose
  double2 *hb = sm + M * H * W;   // [BY][BX]
  {
    const int jj = l - st.prev_shift;
    const double2 *hsrc = jj < 0 ? st.u0 : st.prev_base + (long long)jj * st.prev_stride;
    for (int r = warp; r < BY; r += blockDim.x >> 5) {
      const double2 *src = hsrc + ((size_t)(y0 + r) << g.lognx) + x0;
      for (int xx = lane; xx < BX; xx += 32) cp_async16(hb + r * BX + xx, src + xx);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (box) mbar_wait(&bar, 0);
  for (int pt = threadIdx.x; pt < BX * BY; pt += blockDim.x) {
    const int ty = pt / BX, tx = pt - ty * BX;
    const int n = ((y0 + ty) << g.lognx) + x0 + tx;
    const double2 base = hb[pt];
    double2 uc[M], Au[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double2 *q = sm + (j * H + ty + HW) * W + tx + HW;
      const double2 c = q[0];
      uc[j] = c;
      double2 acc = make_double2(g.wx[3] * c.x, g.wx[3] * c.y);
#pragma unroll
      for (int o = -HW; o <= HW; ++o) {
        if (o == 0) continue;
        const double2 a = q[o], d = q[o * W];
        acc.x = fma(g.wx[3 + o], a.x, acc.x);
        acc.y = fma(g.wx[3 + o], a.y, acc.y);
        acc.x = fma(g.wy[3 + o], d.x, acc.x);
        acc.y = fma(g.wy[3 + o], d.y, acc.y);
      }
      Au[j] = acc;
    }
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
      X[(size_t)l * plane + (size_t)m * g.N + n] = cscale(acc, sc);
    }
  }
  }
}

// ---------------------------------------------------------------------------------------------
// 1-D spatial solves: (I - s A) x = y, A cyclic tridiagonal with constant coefficients.
// PCR level j (h = 2^j) on the circulant system: y_i <- y_i - p_j y_{i-h} - q_j y_{i+h} with
// p_j = a_j/b_j, q_j = c_j/b_j; last level (h = N/2, i-h == i+h): y_i <- y_i - p y_{i+h}; then
// x = y / e_final.  Level coefficients come from the host (long double, row sum e = a+b+c carried,
// DESIGN.md reading R6).  The level operators are circulant, hence commute: the two-pass scheme
// applies the large strides (closed on residue classes mod R) first, then the small strides on
// contiguous chunks with halos.

// One PCR level update y - p y_{i-h} - q y_{i+h}.  The level coefficients of the heat family are
// symmetric (q = p at every level: a' = -a^2/b, c' = -c^2/b keep a = c) and those of centred
// advection antisymmetric at level 0 (q = -p) and symmetric after; sym = +1 / -1 then needs one
// complex product instead of two (used by the chunk pass; the register class pass measured
// slower with the extra branch).
__device__ __forceinline__ int pcr_sym(double2 p, double2 q) {
  if (p.x == q.x && p.y == q.y) return 1;
  if (p.x == -q.x && p.y == -q.y) return -1;
  return 0;
}
__device__ __forceinline__ double2 pcr_update(int sym, double2 p, double2 q, double2 lv, double2 rv, double2 y) {
  if (sym > 0) return cfms(p, cadd(lv, rv), y);
  if (sym < 0) return cfms(p, csub(lv, rv), y);
  return cfms(q, rv, cfms(p, lv, y));
}

constexpr int kPcrThreads = 256;
constexpr int kPcrIPT = 16;   // items per thread held in registers per level

// Lines of length nq at element stride R (residue classes mod R), T consecutive classes per CTA.
// Applies coefficient levels j_off .. nlev-1 (the last is the pair level) and multiplies by 1/e.
// Line indices run over the solved units (Hermitian mode: k <= L/2); the factor tables are indexed
// by the unit's slot: tline = slots[line / M] M + line % M.
__device__ __forceinline__ int table_line(const Geometry &g, const int *slots, int line) {
  return __ldg(slots + line / g.M) * g.M + line % g.M;
}

template <int F>
__global__ void __launch_bounds__(kPcrThreads) pcr_classes_kernel(const Geometry g, AlphaTables at,
                                                                  double2 *__restrict__ X, int R, int T,
                                                                  int j_off, const double2 *__restrict__ r0,
                                                                  const int *__restrict__ slots) {
  extern __shared__ double2 sm[];  // [nq][T]
  const int lT = 31 - __clz(T);
  const int N = g.N;
  const int nq = N / R;
  const int lognq = g.logN - j_off;
  const int groups = R / T;
  const int line = blockIdx.x / groups;
  const int rr = (blockIdx.x - line * groups) * T;
  double2 *xl = X + (size_t)line * N;
  const int tline = table_line(g, slots, line);
  const int items = nq * T;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int tt = it & (T - 1), q = it >> lT;
    sm[it] = r0 ? cmul(__ldg(at.sig + tline), __ldg(r0 + (size_t)q * R + rr + tt)) : xl[(size_t)q * R + rr + tt];
  }
  __syncthreads();
  const double2 *coef = at.pcr + (size_t)tline * g.logN * F * 2;   // F == g.nfac
  for (int jf = 0; jf < lognq * F; ++jf) {   // level jj, factor f (all circulant: any order)
    const int jj = jf / F;
    const int j = j_off + jj;
    const double2 pj = __ldg(coef + 2 * (j * F + jf % F)), qj = __ldg(coef + 2 * (j * F + jf % F) + 1);
    const int h = 1 << jj;
    const bool pair = (jj == lognq - 1);
    double2 nv[kPcrIPT];
#pragma unroll
    for (int k = 0; k < kPcrIPT; ++k) {
      const int it = threadIdx.x + k * kPcrThreads;
      if (it < items) {
        const int tt = it & (T - 1), q = it >> lT;
        const double2 yc = sm[it];
        const double2 yp = sm[((q + h) & (nq - 1)) * T + tt];
        double2 v = csub(yc, cmul(pair ? pj : qj, yp));
        if (!pair) v = csub(v, cmul(pj, sm[((q - h) & (nq - 1)) * T + tt]));
        nv[k] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPcrIPT; ++k) {
      const int it = threadIdx.x + k * kPcrThreads;
      if (it < items) sm[it] = nv[k];
    }
    __syncthreads();
  }
  const double2 ie = __ldg(at.inv_e + tline);
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int tt = it & (T - 1), q = it >> lT;
    xl[(size_t)q * R + rr + tt] = cmul(sm[it], ie);
  }
}

// one block-arrangement PCR level with compile-time stride H (< E: only the 2H edge values move
// between lanes; >= E: whole neighbours H/E lanes away)
template <int E, int H>
__device__ __forceinline__ void pcr_block_level(double2 (&y)[E], int b, int S, double2 pj, double2 qj) {
  double2 nv[E];
  if constexpr (H < E) {
    const int left = (b + S - 1) & (S - 1), right = (b + 1) & (S - 1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      double2 lv, rv;
      if (e >= H) {
        lv = y[e - H];
      } else {
        lv.x = __shfl_sync(0xffffffffu, y[e - H + E].x, left, S);
        lv.y = __shfl_sync(0xffffffffu, y[e - H + E].y, left, S);
      }
      if (e + H < E) {
        rv = y[e + H];
      } else {
        rv.x = __shfl_sync(0xffffffffu, y[e + H - E].x, right, S);
        rv.y = __shfl_sync(0xffffffffu, y[e + H - E].y, right, S);
      }
      nv[e] = cfms(qj, rv, cfms(pj, lv, y[e]));
    }
  } else {
    constexpr int d = H / E;
    const int bl = (b + S - d) & (S - 1), br = (b + d) & (S - 1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      double2 lv, rv;
      lv.x = __shfl_sync(0xffffffffu, y[e].x, bl, S);
      lv.y = __shfl_sync(0xffffffffu, y[e].y, bl, S);
      rv.x = __shfl_sync(0xffffffffu, y[e].x, br, S);
      rv.y = __shfl_sync(0xffffffffu, y[e].y, br, S);
      nv[e] = cfms(qj, rv, cfms(pj, lv, y[e]));
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) y[e] = nv[e];
}

// Register-resident variant of the class pass (two-pass scheme, nq = N/R <= 32*E): E class
// elements per thread.  Levels with stride h' < S = nq/E run in a BLOCK arrangement (thread holds
// q in [b E, (b+1) E) of one column; neighbours across the block edge come from lanes b-1/b+1 by
// warp shuffle); then one shared-memory transposition to a CLASS arrangement (thread holds
// q = c + S k), where every stride h' >= S is closed in registers (cyclic in k).  Large strides
// are applied last, so the 1/e scaling and the store happen from the class arrangement
// (coalesced over the T columns).  Level operators commute (circulant), so the order is free.
template <int E, int F>
__global__ void __launch_bounds__(256, 3) pcr_reg_kernel(const Geometry g, AlphaTables at, double2 *__restrict__ X,
                                                         int R, int T, int j_off, const double2 *__restrict__ r0,
                                                         const int *__restrict__ slots) {
  extern __shared__ double2 sm[];  // [nq][T], swizzled
  const int N = g.N;
  const int nq = N / R;
  const int lognq = g.logN - j_off;
  const int S = nq / E;                 // lanes per column in the block arrangement
  const int logS = 31 - __clz(S);
  const int lT = 31 - __clz(T);
  const int groups = R / T;
  const int line = blockIdx.x / groups;
  const int rr = (blockIdx.x - line * groups) * T;
  double2 *xl = X + (size_t)line * N;
  const int tline = table_line(g, slots, line);
  const int items = nq * T;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int tt = it & (T - 1), q = it >> lT;
    if (r0) sm[swz(it)] = cmul(__ldg(at.sig + tline), __ldg(r0 + (size_t)q * R + rr + tt));  // direct form
    else cp_async16(sm + swz(it), xl + (size_t)q * R + rr + tt);
  }
  cp_async_wait_all();
  __syncthreads();
  const double2 *coef = at.pcr + (size_t)tline * g.logN * F * 2;   // F == g.nfac
  double2 y[E];
  {  // block arrangement: thread -> (column, block b); the S lanes of a column are consecutive
    const int b = threadIdx.x & (S - 1), col = threadIdx.x >> logS;
#pragma unroll
    for (int e = 0; e < E; ++e) y[e] = sm[swz(((b * E + e) << lT) + col)];
    const double2 *cb = coef + 2 * j_off * F;
#define PINT_BLK(H, JJ) \
    if ((H) < S) _Pragma("unroll") for (int f = 0; f < F; ++f) \
      pcr_block_level<E, H>(y, b, S, __ldg(cb + 2 * ((JJ) * F + f)), __ldg(cb + 2 * ((JJ) * F + f) + 1));
    PINT_BLK(1, 0) PINT_BLK(2, 1) PINT_BLK(4, 2) PINT_BLK(8, 3) PINT_BLK(16, 4)
#undef PINT_BLK
#pragma unroll
    for (int e = 0; e < E; ++e) sm[swz(((b * E + e) << lT) + col)] = y[e];
  }
  __syncthreads();
  // class arrangement: thread -> (column fastest, class c); holds q = c + S k
  const int col = threadIdx.x & (T - 1), c = threadIdx.x >> lT;
#pragma unroll
  for (int k = 0; k < E; ++k) y[k] = sm[swz(((c + (k << logS)) << lT) + col)];
  for (int jf = logS * F; jf < lognq * F; ++jf) {   // strides h' = S 2^i, i.e. 2^i in k (cyclic over E)
    const int jj = jf / F;
    const int hk = 1 << (jj - logS);
    const double2 *cj = coef + 2 * ((j_off + jj) * F + jf % F);
    const double2 pj = __ldg(cj), qj = __ldg(cj + 1);
    const bool pair = (jj == lognq - 1);
    double2 nv[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const double2 rv = y[(k + hk) & (E - 1)];
      if (pair) nv[k] = cfms(pj, rv, y[k]);
      else nv[k] = cfms(qj, rv, cfms(pj, y[(k - hk) & (E - 1)], y[k]));
    }
#pragma unroll
    for (int k = 0; k < E; ++k) y[k] = nv[k];
  }
  const double2 ie = __ldg(at.inv_e + tline);
#pragma unroll
  for (int k = 0; k < E; ++k) xl[(size_t)(c + (k << logS)) * R + rr + col] = cmul(y[k], ie);
}

// Small-stride levels 0..jA-1 (each for all F factors) on contiguous chunks of C with halos of
// H >= F (2^jA - 1) (redundant halo computation, out of place X -> Y).
constexpr int kChunkThreads = 512;
constexpr int kChunkIPT = 10;

__global__ void __launch_bounds__(kChunkThreads) pcr_chunk_kernel(const Geometry g, AlphaTables at,
                                                                  const double2 *__restrict__ X,
                                                                  double2 *__restrict__ Y, int C, int H,
                                                                  int jA, const int *__restrict__ slots) {
  extern __shared__ double2 sm[];  // [C + 2H]
  const int N = g.N;
  const int chunks = N / C;
  const int line = blockIdx.x / chunks;
  const int n0 = (blockIdx.x - line * chunks) * C;
  const double2 *xl = X + (size_t)line * N;
  const int S = C + 2 * H;
  for (int i = threadIdx.x; i < S; i += blockDim.x) sm[i] = __ldg(xl + ((n0 - H + i) & (N - 1)));
  __syncthreads();
  const int F = g.nfac;
  const double2 *coef = at.pcr + (size_t)table_line(g, slots, line) * g.logN * F * 2;
  int lo = 0;
  for (int jf = 0; jf < jA * F; ++jf) {
    const int h = 1 << (jf / F);
    lo += h;  // valid region after this (level, factor): [lo, S - lo)
    const double2 pj = __ldg(coef + 2 * jf), qj = __ldg(coef + 2 * jf + 1);
    const int sym = pcr_sym(pj, qj);
    const int cnt = S - 2 * lo;
    double2 nv[kChunkIPT];
#pragma unroll
    for (int k = 0; k < kChunkIPT; ++k) {
      const int i = lo + threadIdx.x + k * kChunkThreads;
      if (i < lo + cnt) nv[k] = pcr_update(sym, pj, qj, sm[i - h], sm[i + h], sm[i]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kChunkIPT; ++k) {
      const int i = lo + threadIdx.x + k * kChunkThreads;
      if (i < lo + cnt) sm[i] = nv[k];
    }
    __syncthreads();
  }
  double2 *yl = Y + (size_t)line * N;
  for (int i = threadIdx.x; i < C; i += blockDim.x) yl[n0 + i] = sm[H + i];
}

// ---------------------------------------------------------------------------------------------
// 2-D spatial solves by FFT: row DIF (x) -> column pass [DIF (y), * 1/((1 - s lambda) nx ny),
// DIT (y)] -> row DIT (x).  Spectral positions are bit-reversed between the passes.

constexpr int kFftThreads = 256;

// Row pass with the node transform of frequency p fused in: one CTA per (p, group of YG rows y),
// holding the M rows (p, m, y) of every y of the group.  Forward: x1 = S_p^{-1} x, then x-DIF FFT.
// Inverse: x-DIT inverse FFT, then y = G_p^{-1} S_p x2.  All threads of a CTA share p, so the
// M x M table loads are warp-uniform (broadcast).
template <int M, bool INV, bool NODE>
__global__ void __launch_bounds__(kFftThreads, kSpaceMinBlocks)
    fft2d_rows_kernel(const Geometry g, StaticTables st, AlphaTables at, double2 *__restrict__ X, int YG) {
  extern __shared__ double2 sm[];  // [YG][M][nx], swizzled
  const int nx = g.nx;
  const int ygroups = g.ny / YG;
  const int p = blockIdx.x / ygroups;
  const int y0 = (blockIdx.x - p * ygroups) * YG;
  const size_t plane = (size_t)M * g.N;
  double2 *xp = X + (size_t)p * plane;
  const int items = YG * M * nx;
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int x = i & (nx - 1), r = i >> g.lognx;
    const int m = r % M, yy = r / M;
    cp_async16(sm + swz(i), xp + (size_t)m * g.N + ((size_t)(y0 + yy) << g.lognx) + x);
  }
  cp_async_wait_all();
  __syncthreads();
  const double2 *tab = (INV ? at.SG : at.Sinv) + (size_t)p * M * M;
  if (!INV) {
    if (NODE) for (int c = threadIdx.x; c < YG * nx; c += blockDim.x) {
      const int x = c & (nx - 1), yy = c >> g.lognx;
      double2 v[M];
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = sm[swz((yy * M + j) * nx + x)];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) acc = cfma(__ldg(tab + m * M + j), v[j], acc);
        sm[swz((yy * M + m) * nx + x)] = acc;
      }
    }
    __syncthreads();
    fft_dif<4, true>(sm, YG * M, nx, 1, nx, g.lognx, st.twx);
  } else {
    fft_dit_inv<4, true>(sm, YG * M, nx, 1, nx, g.lognx, st.twx);
    if (NODE) for (int c = threadIdx.x; c < YG * nx; c += blockDim.x) {
      const int x = c & (nx - 1), yy = c >> g.lognx;
      double2 v[M];
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = sm[swz((yy * M + j) * nx + x)];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) acc = cfma(__ldg(tab + m * M + j), v[j], acc);
        sm[swz((yy * M + m) * nx + x)] = acc;
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int x = i & (nx - 1), r = i >> g.lognx;
    const int m = r % M, yy = r / M;
    xp[(size_t)m * g.N + ((size_t)(y0 + yy) << g.lognx) + x] = sm[swz(i)];
  }
}

constexpr int kColThreads = 512;

__global__ void __launch_bounds__(kColThreads, 1)
    fft2d_cols_kernel(const Geometry g, StaticTables st, AlphaTables at, double2 *__restrict__ X, int T) {
  extern __shared__ double2 sm[];  // [ny][T] (T >= 8: contiguous quarter-warps, no swizzle)
  const int lT = 31 - __clz(T);
  const int nx = g.nx, ny = g.ny;
  const int groups = nx / T;
  const int line = blockIdx.x / groups;           // line = p*M + m
  const int kx0 = (blockIdx.x - line * groups) * T;
  double2 *xl = X + (size_t)line * g.N;
  const int items = ny * T;
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int tt = i & (T - 1), y = i >> lT;
    cp_async16(sm + sidx<false>(i), xl + (size_t)y * nx + kx0 + tt);
  }
  cp_async_wait_all();
  __syncthreads();
  const int blast = fft_dif_but_last<4, false>(sm, T, 1, T, g.logny, st.twy);
  const double2 s = __ldg(at.shift + line);
  const double inv_n = 1.0 / ((double)nx * (double)ny);
  // x2 = x1 / (1 - s (lambda_x + lambda_y)) / (nx ny), applied in the fused middle groups
  auto divide = [&](int tt, int py, double2 v) -> double2 {
    const int kx = brev(kx0 + tt, g.lognx), ky = brev(py, g.logny);
    const double2 lam = cadd(__ldg(st.lamx + kx), __ldg(st.lamy + ky));
    const double2 sl = cmul(s, lam);
    const double dr = 1.0 - sl.x, di = -sl.y;
    const double q = dr * dr + di * di;             // > 0 (Re s > 0, Re lambda <= 0)
    double rq = __drcp_rn(q);                        // reciprocal + one Newton step
    rq = fma(rq, fma(-q, rq, 1.0), rq);
    const double den = inv_n * rq;
    return make_double2((v.x * dr + v.y * di) * den, (v.y * dr - v.x * di) * den);
  };
  if (blast == 1) fused_middle<1, false>(sm, T, 1, T, g.logny, divide);
  else if (blast == 2) fused_middle<2, false>(sm, T, 1, T, g.logny, divide);
  else if (blast == 3) fused_middle<3, false>(sm, T, 1, T, g.logny, divide);
  else fused_middle<4, false>(sm, T, 1, T, g.logny, divide);
  fft_dit_inv_from<4, false>(sm, T, 1, T, g.logny, st.twy, 1);
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int tt = i & (T - 1), y = i >> lT;
    xl[(size_t)y * nx + kx0 + tt] = sm[sidx<false>(i)];
  }
}

// ---------------------------------------------------------------------------------------------
// Direct form (Alg. 1 as printed): r = (C_a - C) u + w = w - alpha e_1 (x) H u_L
// has one non-zero block, r0 = u0 - alpha u_{L-1,M-1} replicated over the nodes; its
// scaled time DFT is r0 at every frequency, so the forward transform costs one N-vector.

__global__ void direct_r0_kernel(Geometry g, StaticTables st, AlphaTables at, const double2 *__restrict__ u,
                                 double2 *__restrict__ r0) {
  const size_t ul = ((size_t)(g.L - 1) * g.M + (g.M - 1)) * g.N;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < g.N; n += gridDim.x * blockDim.x) {
    const double2 a = __ldg(st.u0 + n), b = u_at(u, ul + n, st.packed != 0);
    r0[n] = make_double2(a.x - at.alpha * b.x, a.y - at.alpha * b.y);
  }
}

// one plane: x-DIF of YG rows per CTA (in place, bit-reversed kx positions)
__global__ void __launch_bounds__(kFftThreads) plane_rows_dif_kernel(const Geometry g, StaticTables st,
                                                                     double2 *__restrict__ P, int YG) {
  extern __shared__ double2 sm[];
  const int nx = g.nx;
  double2 *base = P + (size_t)blockIdx.x * YG * nx;
  const int items = YG * nx;
  for (int i = threadIdx.x; i < items; i += blockDim.x) cp_async16(sm + swz(i), base + i);
  cp_async_wait_all();
  __syncthreads();
  fft_dif<4, true>(sm, YG, nx, 1, nx, g.lognx, st.twx);
  for (int i = threadIdx.x; i < items; i += blockDim.x) base[i] = sm[swz(i)];
}

// one plane: y-DIF of T columns per CTA (in place, bit-reversed ky positions)
__global__ void __launch_bounds__(kFftThreads) plane_cols_dif_kernel(const Geometry g, StaticTables st,
                                                                     double2 *__restrict__ P, int T) {
  extern __shared__ double2 sm[];
  const int lT = 31 - __clz(T);
  const int kx0 = blockIdx.x * T;
  const int items = g.ny * T;
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int tt = i & (T - 1), y = i >> lT;
    cp_async16(sm + swz(i), P + (size_t)y * g.nx + kx0 + tt);
  }
  cp_async_wait_all();
  __syncthreads();
  fft_dif<4, true>(sm, T, 1, T, g.ny, g.logny, st.twy);
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int tt = i & (T - 1), y = i >> lT;
    P[(size_t)y * g.nx + kx0 + tt] = sm[swz(i)];
  }
}

// synthesized column pass: x2_{km} spectrum = sig_km r0hat / (1 - s_km lambda) / (nx ny), then the
// y-DIT inverse; writes the (line, all y, T columns) tile of X (no read of X)
__global__ void __launch_bounds__(kColThreads, 1)
    cols_direct_kernel(const Geometry g, StaticTables st, AlphaTables at, const double2 *__restrict__ spec,
                       double2 *__restrict__ X, int T) {
  extern __shared__ double2 sm[];  // [ny][T]
  const int lT = 31 - __clz(T);
  const int nx = g.nx, ny = g.ny;
  const int groups = nx / T;
  const int line = blockIdx.x / groups;
  const int kx0 = (blockIdx.x - line * groups) * T;
  double2 *xl = X + (size_t)line * g.N;
  const int items = ny * T;
  const double2 s = __ldg(at.shift + line);
  const double2 sg = cscale(__ldg(at.sig + line), 1.0 / ((double)nx * (double)ny));
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int tt = i & (T - 1), py = i >> lT;
    const int kx = brev(kx0 + tt, g.lognx), ky = brev(py, g.logny);
    const double2 lam = cadd(__ldg(st.lamx + kx), __ldg(st.lamy + ky));
    const double2 sl = cmul(s, lam);
    const double dr = 1.0 - sl.x, di = -sl.y;
    const double q = dr * dr + di * di;
    double rq = __drcp_rn(q);
    rq = fma(rq, fma(-q, rq, 1.0), rq);
    const double2 v = cmul(sg, __ldg(spec + (size_t)py * nx + kx0 + tt));
    sm[i] = make_double2((v.x * dr + v.y * di) * rq, (v.y * dr - v.x * di) * rq);
  }
  __syncthreads();
  fft_dit_inv<4, false>(sm, T, 1, T, ny, g.logny, st.twy);
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int tt = i & (T - 1), y = i >> lT;
    xl[(size_t)y * nx + kx0 + tt] = sm[i];
  }
}

// ---------------------------------------------------------------------------------------------
// Multi-rank pieces (time-sharded cyclic distribution, four-step time FFT).
// Rank g owns global steps l = g + P j (j < Ll = L/P).  After the local Ll-point DIF FFT (slot p,
// kappa = bitrev_Ll(p)) and the twiddle e^{-2 pi i g kappa / L}, chunk d (p in [d Lc, (d+1) Lc),
// Lc = Ll/P) goes to rank d.  Rank d then holds, for its local positions pl < Lc, the P values
// y_g (g = source rank) and forms x_{kappa + Ll q} = sum_g e^{-2 pi i g q/P} y_g (q < P), stored at
// slot sigma = q Lc + pl of the local frequency order (its factor tables are built for that order).

__global__ void halo_pack_kernel(Geometry g, const double2 *__restrict__ u, double2 *__restrict__ hsend) {
  const long long total = (long long)g.L * g.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long l = i / g.N, n = i - l * g.N;
    hsend[i] = __ldg(u + (l * g.M + (g.M - 1)) * (long long)g.N + n);
  }
}

// forward: in = receive buffer [src g][pl][m][n] -> out[sigma][m][n] with S_sigma^{-1} applied
// inverse: in[sigma][m][n] -> G_sigma^{-1} S_sigma, inverse P-point DFT -> out = send buffer
//          [dst g][pl][m][n]
template <int M, int P, bool INV>
__global__ void __launch_bounds__(256) xdft_kernel(Geometry g, StaticTables st, AlphaTables at,
                                                   const double2 *__restrict__ in, double2 *__restrict__ out,
                                                   int pl0, int npl) {
  const int Lc = g.L / P;
  const long long total = (long long)npl * g.N;           // band pl0 .. pl0 + npl of the chunk slots
  const long long chunk = (long long)Lc * M * g.N;       // elements per peer chunk
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int pl = pl0 + (int)(i / g.N);
    const long long n = i - (long long)(pl - pl0) * g.N;
    double2 x[P][M];
    if (!INV) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double2 v[P];
#pragma unroll
        for (int gg = 0; gg < P; ++gg) v[gg] = __ldg(in + gg * chunk + ((long long)pl * M + m) * g.N + n);
#pragma unroll
        for (int q = 0; q < P; ++q) {
          double2 acc = v[0];
#pragma unroll
          for (int gg = 1; gg < P; ++gg) acc = cfma(v[gg], __ldg(st.twP + (gg * q) % P), acc);
          x[q][m] = acc;
        }
      }
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const int sig = q * Lc + pl;
        const double2 *S = at.Sinv + (size_t)sig * M * M;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < M; ++j) acc = cfma(__ldg(S + m * M + j), x[q][j], acc);
          out[((long long)sig * M + m) * g.N + n] = acc;
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const int sig = q * Lc + pl;
        double2 v[M];
#pragma unroll
        for (int j = 0; j < M; ++j) v[j] = __ldg(in + ((long long)sig * M + j) * g.N + n);
        const double2 *S = at.SG + (size_t)sig * M * M;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < M; ++j) acc = cfma(__ldg(S + m * M + j), v[j], acc);
          x[q][m] = acc;
        }
      }
#pragma unroll
      for (int gg = 0; gg < P; ++gg) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          double2 acc = x[0][m];
#pragma unroll
          for (int q = 1; q < P; ++q) acc = cfma(x[q][m], cmulc(make_double2(1.0, 0.0), __ldg(st.twP + (gg * q) % P)), acc);
          out[gg * chunk + ((long long)pl * M + m) * g.N + n] = acc;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// residual norms and initialisation

template <int M, bool P2 = true>
__global__ void __launch_bounds__(256) resnorm_kernel(Geometry g, StaticTables st,
                                                      const double2 *__restrict__ u, double *partial) {
  __shared__ double s2[32], sm_[32];
  double acc2 = 0.0, accm = 0.0;
  const long long total = (long long)g.L * g.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(i / g.N), n = (int)(i - (long long)l * g.N);
    double2 r[M];
    if (!P2) residual_point<M, false, 3, false>(g, st, u, l, n, r);
    else if (st.packed) residual_point<M, true>(g, st, u, l, n, r);
    else residual_point<M, false>(g, st, u, l, n, r);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double a2 = r[m].x * r[m].x + r[m].y * r[m].y;
      acc2 += a2;
      accm = nanmax(accm, sqrt(a2));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
    accm = nanmax(accm, __shfl_xor_sync(0xffffffffu, accm, o));
  }
  if ((threadIdx.x & 31) == 0) { s2[threadIdx.x >> 5] = acc2; sm_[threadIdx.x >> 5] = accm; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += s2[w]; b = nanmax(b, sm_[w]); }
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
  }
}

__global__ void reduce_partials_kernel(const double *partial, int nblocks, double *out) {
  // one warp, fixed order -> deterministic
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += 32) { a += partial[2 * i]; b = nanmax(b, partial[2 * i + 1]); }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b = nanmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if (threadIdx.x == 0) { out[0] = sqrt(a); out[1] = b; }
}

__global__ void init_iterate_kernel(Geometry g, const double2 *__restrict__ u0, double2 *__restrict__ u, int real) {
  const long long total = (long long)g.L * g.M * g.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    if (real) ((double *)u)[i] = __ldg(u0 + (i % g.N)).x;
    else u[i] = __ldg(u0 + (i % g.N));
  }
}

// ||w||_inf with a forcing attached (Alg. 2's gamma): w_0 = u0 + v_0 on every node of global
// step 0 (rank 0's local step 0), w_l = v_l otherwise; NaN-propagating max into out (as bits)
__global__ void __launch_bounds__(256) w_inf_kernel(Geometry g, StaticTables st, unsigned long long *out) {
  __shared__ double red[8];
  double m = 0.0;
  const long long total = (long long)g.L * g.M * g.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    double2 v = __ldg(st.v + i);
    if (st.rank == 0 && i < (long long)g.M * g.N) v = cadd(v, __ldg(st.u0 + (i % g.N)));
    m = nanmax(m, hypot(v.x, v.y));
  }
  for (int o = 16; o > 0; o >>= 1) m = nanmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = nanmax(m, red[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(m));   // non-negative: bit order = value order
  }
}

// storage conversion of the iterate (pint_set_hermitian): complex <-> real through a scratch
// vector (in-place compaction would race)
__global__ void real_parts_kernel(const double2 *__restrict__ src, double *__restrict__ dst, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i].x;
}
__global__ void complex_from_real_kernel(const double *__restrict__ src, double2 *__restrict__ dst, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = make_double2(src[i], 0.0);
}

// ---------------------------------------------------------------------------------------------
// host-side launch logic

static thread_local Recorder *g_rec = nullptr;
void set_recorder(Recorder *r) { g_rec = r; }
void record_launch(cudaStream_t s) {
  if (g_rec && g_rec->n < g_rec->cap) cudaEventRecord(g_rec->ev[g_rec->n++], s);
}
static inline void rec(cudaStream_t s) {
  if (g_rec && g_rec->n < g_rec->cap) cudaEventRecord(g_rec->ev[g_rec->n++], s);
}

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

size_t fwd_smem_bytes(const Geometry &g, int T) { return (size_t)g.L * g.M * T * sizeof(double2); }

// the 1-D backward tile moved by the TMA unit (bwd_kernel, tma = 1): complex storage, box rows of
// 2 T <= 256 doubles, L <= 256 or a multiple of 256.  PINT_BWD_TMA=0 (experiments build): A/B.
static bool bwd1d_tma_ok(const Geometry &g, const StaticTables &st, int T) {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_BWD_TMA");
    v = (e && !atoi(e)) ? 0 : 1;
  }
  return v == 1 && g.dim == 1 && g.pow2 && !st.packed && T >= 1 && 2 * T <= 256 && g.N % T == 0 && g.M <= 8 &&
         (g.L <= 256 || g.L % 256 == 0) && tma_encode_fn() != nullptr;
}
// the TMA-staged 1-D forward tile (fwd1d_tma_kernel): one rank, complex storage, 3-point stencil,
// T = 4, L <= 256 (one step per thread), 128-byte aligned halo arrays, >= 3 CTAs per SM
bool fwd1d_tma_ok(const Geometry &g, const StaticTables &st, int T) {
  return g.dim == 1 && g.pow2 && st.P == 1 && !st.packed && g.hw <= 1 && T == 4 && g.N >= 8 && g.L >= 8 &&
         g.L <= 256 && (g.L * g.M) % 32 == 0 && g.M <= 4 && 2048 + (size_t)g.L * 16 + 2 * (size_t)g.L * g.M * 6 * sizeof(double2) <= 227 * 1024 &&
         tma_encode_fn() != nullptr && !experiment_env("PINT_FWD_LEGACY");
}

// 2-D path selection: default = all-node time tiles + the persistent spatial pipeline
// (spatial2d.cu); PINT_LEGACY2D=1 selects the six-pass path (A/B measurements only).
static bool legacy_pipe() {   // A/B: the fused persistent spatial2d kernel instead of the pipelined passes
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_LEGACY_PIPE");
    v = (e && atoi(e)) ? 1 : 0;
  }
  return v == 1;
}
// The pipelined (TMA ring) time transforms measured slower than the one-tile-per-CTA kernels on
// config 5 (forward 16.2 vs 14.9 ms, inverse 31.9 vs 21.2 ms: a third of the threads per SM keep
// fewer u loads in flight); they stay an A/B option (PINT_TFFT_PIPE=1, experiments build).
static bool legacy_tfft() {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_TFFT_PIPE");
    v = (e && atoi(e)) ? 0 : 1;
  }
  return v == 1;
}
// TMA variants of the 2-D time tiles (tfft_fwd_tma_kernel / tfft_bwd_tma_kernel): complex storage,
// box rows of 2 T <= 256 doubles, L <= 256 or a multiple of 256.  PINT_TFFT_TMA=0 (experiments
// build) selects the per-thread copies for A/B runs.
static bool tfft_tma_ok(const Geometry &g, const StaticTables &st, int T) {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_TFFT_TMA");
    v = (e && !atoi(e)) ? 0 : 1;
  }
  return v == 1 && g.dim == 2 && g.pow2 && !st.packed && T >= 1 && 2 * T <= 256 && T <= g.N && g.N % T == 0 &&
         (g.L <= 256 || g.L % 256 == 0) && tma_encode_fn() != nullptr;
}
// the inverse's TMA variant alone can be switched off (PINT_TFFT_BWD_TMA=0, experiments build)
static bool tfft_bwd_tma_ok(const Geometry &g, const StaticTables &st, int T) {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_TFFT_BWD_TMA");
    v = (e && !atoi(e)) ? 0 : 1;
  }
  return v == 1 && tfft_tma_ok(g, st, T);
}
// 3-D map over a [L][M][N] complex array as doubles {2N, M, L}, box {2 T doubles, 1 node, min(L, 256) steps}
static bool time_tile_map(const Geometry &g, const double2 *base, int T, CUtensorMap &tm) {
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_fn());
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * g.N, (cuuint64_t)g.M, (cuuint64_t)g.L};
  const cuuint64_t strides[2] = {(cuuint64_t)g.N * 16, (cuuint64_t)g.M * g.N * 16};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * T), 1, (cuuint32_t)(g.L < 256 ? g.L : 256)};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool legacy2d() {
  static int v = -1;
  if (v < 0) {
    const char *e = experiment_env("PINT_LEGACY2D");
    v = (e && atoi(e)) ? 1 : 0;
  }
  return v == 1;
}
// register-engine 2-D path (spatial2d.cu) for the grids it is instantiated for; the generic
// smem-engine kernels below serve every other 2-D shape
static bool reg2d(const Geometry &g) {
  return g.dim == 2 && !legacy2d() && spatial2d_supported(g) && g.logL >= 2 && g.logL <= 10;
}
bool reg2d_path(const Geometry &g) { return reg2d(g); }

// the 1-D two-pass solve runs on the pipelined passes of pcr1d.cu (correction form)
bool pcr1d_path(const Geometry &g, const LaunchCfg &lc) {
  return g.dim == 1 && lc.pcr_mode == 1 && pcr1d_pipe_supported(g, lc.pcr_R) && !experiment_env("PINT_PCR_LEGACY");
}

LaunchCfg choose_launch(const Geometry &g) {
  LaunchCfg lc{};
  // forward/backward tile: as many spatial points as fit ~100 KB (2 CTAs per SM), <= 16
  int T = 16;
  while (T > 1 && fwd_smem_bytes(g, T) > 64 * 1024) T >>= 1;
  if (const char *e = experiment_env("PINT_FWD_T")) T = atoi(e);   // tuning experiments only
  while (T > g.N) T >>= 1;
  lc.fwd_T = T;
  // backward tile: measured on config 3 (L = 256, M = 3): T = 8 (96 KB) 0.63 ms vs T = 4 0.75 ms
  // (the forward tile, which also evaluates the stencil, prefers T = 4 at 3 CTAs per SM)
  int TB = 16;
  while (TB > 1 && fwd_smem_bytes(g, TB) > 100 * 1024) TB >>= 1;
  if (const char *e = experiment_env("PINT_BWD_T")) TB = atoi(e);   // tuning experiments only
  while (TB > g.N) TB >>= 1;
  lc.bwd_T = TB;
  int T2 = 32;
  while (T2 > 1 && (size_t)g.L * T2 * sizeof(double2) > 64 * 1024) T2 >>= 1;
  while (T2 > g.N) T2 >>= 1;
  while (T2 > 1 && g.N % T2) T2 >>= 1;   // generic grids: T must divide N
  lc.tfft_T = T2;
  if (g.dim == 1) {
    if (g.N <= 4096) {
      lc.pcr_mode = 0;
      lc.pcr_R = 1;
      lc.pcr_T = 1;
    } else {
      lc.pcr_mode = 1;
      int jA = g.logN / 2;            // R = 2^jA classes of length N/R
      // pipelined passes (pcr1d.cu): classes of 256 points (strides >= N/256 in the class pass)
      if (pcr1d_pipe_supported(g, 1 << (g.logN - 8)) && !experiment_env("PINT_PCR_LEGACY")) jA = g.logN - 8;
      lc.pcr_chunk = g.nfac > 1 ? 2048 : 4096;
      // The chunk kernel updates at most kChunkThreads * kChunkIPT values per level, so the tile
      // C + 2 F R (chunk + halos) must fit it (every nfac: N = 2^20 with F = 1 gives R = 1024 and
      // a 6144-value tile at C = 4096).  Lower jA while the class length N/R stays <= 4096 (the
      // class pass's tile), then shrink the chunk.
      const int cap = kChunkThreads * kChunkIPT;
      while (jA > 1 && lc.pcr_chunk + 2 * g.nfac * (1 << jA) > cap && (g.N >> (jA - 1)) <= 4096) --jA;
      while (lc.pcr_chunk > 256 && lc.pcr_chunk + 2 * g.nfac * (1 << jA) > cap) lc.pcr_chunk >>= 1;
      lc.pcr_R = 1 << jA;
      int nq = g.N / lc.pcr_R;
      int t = 4096 / nq;
      if (t > lc.pcr_R) t = lc.pcr_R;
      if (t < 1) t = 1;
      lc.pcr_T = t;
      if (lc.pcr_chunk > g.N) lc.pcr_chunk = g.N;
    }
  }
  return lc;
}

bool hermitian_pipe_path(const Geometry &g) { return reg2d(g) && spatial_pipe_geometry(g) && !legacy_pipe(); }

static bool pipe2d(const Geometry &g, const StaticTables &st) {
  return reg2d(g) && spatial_pipe_supported(g, st) && !legacy_pipe();
}
bool pipe2d_geometry(const Geometry &g) { return reg2d(g) && spatial_pipe_geometry(g); }

int launches_per_iteration(const Geometry &g, const LaunchCfg &lc, const StaticTables &st) {
  if (!g.pow2) return generic_launches(g);
  if (g.dim == 2) return pipe2d(g, st) ? (spatial_fused_supported(g, st) ? 4 : 6) : (reg2d(g) ? 4 : 6);
  return lc.pcr_mode == 0 ? 3 : 4;
}

const char *kernel_name(const Geometry &g, const LaunchCfg &lc, const StaticTables &st, int i) {
  static const char *k1a[] = {"fwd_kernel", "pcr_classes_kernel", "bwd_kernel"};
  static const char *k1b[] = {"fwd_kernel", "pcr_classes_kernel", "pcr_chunk_kernel", "bwd_kernel"};
  static const char *k1p[] = {"fwd_kernel", "pcr_cls_pipe_kernel", "pcr_chunk_pipe_kernel", "bwd_kernel"};
  if (g.dim == 1 && i == 0 && fwd1d_tma_ok(g, st, lc.fwd_T)) return "fwd1d_tma_kernel";
  static const char *k2[] = {"residual2d_kernel", "tfft_fwd_kernel", "fft2d_rows_kernel<fwd>", "fft2d_cols_kernel",
                             "fft2d_rows_kernel<inv>", "tfft_bwd_kernel"};
  static const char *k2p[] = {"residual2d_kernel", "tfft_fwd_kernel", "spatial2d_kernel", "tfft_bwd_kernel"};
  static const char *k2q[] = {"residual2d_kernel", "tfft_fwd_kernel", "rows_pipe_kernel<fwd>", "cols_pipe_kernel",
                              "rows_pipe_kernel<inv>", "tfft_bwd_kernel"};
  static const char *k2t[] = {"residual2d_kernel", "tfft_pipe_kernel<fwd>", "rows_pipe_kernel<fwd>", "cols_pipe_kernel",
                              "rows_pipe_kernel<inv>", "tfft_pipe_kernel<inv>"};
  const int n = launches_per_iteration(g, lc, st);
  if (i < 0 || i >= n) return "";
  if (!g.pow2) return generic_kernel_name(g, i);
  static const char *k2f[] = {"residual2d_kernel", "tfft_fwd_kernel", "spatial_fused_kernel", "tfft_bwd_kernel"};
  if (g.dim == 2) {
    if (pipe2d(g, st) && spatial_fused_supported(g, st)) return k2f[i];
    if (pipe2d(g, st)) {
      if (tfft_pipe_supported(g, st) && !legacy_tfft()) return k2t[i];
      if (tfft_tma_ok(g, st, lc.tfft_T)) {
        if (i == 1) return "tfft_fwd_tma_kernel";
        if (i == n - 1 && tfft_bwd_tma_ok(g, st, lc.tfft_T)) return "tfft_bwd_tma_kernel";
      }
      return k2q[i];
    }
    const char *nm = reg2d(g) ? k2p[i] : k2[i];
    if (tfft_pipe_supported(g, st) && !legacy_tfft()) {   // time transforms pipelined, spatial legacy
      if (i == 1) return "tfft_pipe_kernel<fwd>";
      if (i == n - 1) return "tfft_pipe_kernel<inv>";
    }
    if (tfft_tma_ok(g, st, lc.tfft_T)) {
      if (i == 1) return "tfft_fwd_tma_kernel";
      if (i == n - 1 && tfft_bwd_tma_ok(g, st, lc.tfft_T)) return "tfft_bwd_tma_kernel";
    }
    return nm;
  }
  return lc.pcr_mode == 0 ? k1a[i] : (pcr1d_path(g, lc) ? k1p[i] : k1b[i]);
}

static cudaError_t set_smem(const void *fn, size_t bytes, bool max_carveout = false) {
  // always opt in: static shared memory (reduction scratch) adds to the dynamic bytes
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess || !max_carveout) return e;
  // largest shared-memory carveout (residual tiles: 4 CTAs of 42 KB per SM)
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

static cudaError_t launch_pcr_classes(const Geometry &g, const AlphaTables &at, double2 *X, int R, int T, int jOff,
                                      const double2 *r0, const int *slots, int grid, size_t smem, cudaStream_t s) {
  cudaError_t e;
#define PINT_PCRCL(F_)                                                                          \
  if ((e = set_smem((const void *)pcr_classes_kernel<F_>, smem)) != cudaSuccess) return e;      \
  pcr_classes_kernel<F_><<<grid, kPcrThreads, smem, s>>>(g, at, X, R, T, jOff, r0, slots);
  if (g.nfac == 1) { PINT_PCRCL(1) } else if (g.nfac == 2) { PINT_PCRCL(2) } else { PINT_PCRCL(3) }
#undef PINT_PCRCL
  return cudaGetLastError();
}

template <int E>
static cudaError_t launch_pcr_reg(const Geometry &g, const AlphaTables &at, double2 *X, int R, int T, int jOff,
                                  const double2 *r0, const int *slots, int grid, size_t smem, cudaStream_t s) {
  cudaError_t e;
#define PINT_PCRREG(F_)                                                                       \
  if ((e = set_smem((const void *)pcr_reg_kernel<E, F_>, smem)) != cudaSuccess) return e;     \
  pcr_reg_kernel<E, F_><<<grid, 256, smem, s>>>(g, at, X, R, T, jOff, r0, slots);
  if (g.nfac == 1) { PINT_PCRREG(1) } else if (g.nfac == 2) { PINT_PCRREG(2) } else { PINT_PCRREG(3) }
#undef PINT_PCRREG
  return cudaGetLastError();
}


#define PINT_DISPATCH_M(M_, ...)       \
  switch (M_) {                        \
    case 1: { constexpr int MM = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int MM = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int MM = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int MM = 4; __VA_ARGS__; } break; \
    case 5: { constexpr int MM = 5; __VA_ARGS__; } break; \
    case 6: { constexpr int MM = 6; __VA_ARGS__; } break; \
    case 7: { constexpr int MM = 7; __VA_ARGS__; } break; \
    default: { constexpr int MM = 8; __VA_ARGS__; } break; \
  }

// 2-D residual block: BX x BY points, BX*BY <= 256
static void residual_block(const Geometry &g, int &BX, int &BY) {
  BX = g.nx < 64 ? g.nx : 64;     // 64 x 8 points per CTA (halo overhead 66*10/512 = 1.29)
  BY = 512 / BX;
  if (BY > g.ny) BY = g.ny;
}

cudaError_t launch_forward(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                           const AlphaTables &at, const Buffers &b, cudaStream_t s) {
  if (!g.pow2) {   // generic grids (generic.cu): residual, then the time DFT on T | N columns
    cudaError_t e = launch_generic_residual(g, st, at, b.u, b.X, s);
    if (e != cudaSuccess) return e;
    const int T2 = lc.tfft_T;
    const size_t sm2 = (size_t)g.L * (T2 + 1) * sizeof(double2);
    if ((e = set_smem((const void *)tfft_fwd_kernel, sm2)) != cudaSuccess) return e;
    tfft_fwd_kernel<<<g.M * (g.N / T2), kTileThreads, sm2, s>>>(g, st, b.X, T2);
    rec(s);
    return cudaGetLastError();
  }
  int T = lc.fwd_T;
  if (st.packed) while (T > g.N / 2) T >>= 1;
  const size_t smem = fwd_smem_bytes(g, T) + (size_t)g.L * sizeof(double2);   // + staged twiddles
  const int grid = (st.packed ? g.N / 2 : g.N) / T;
  cudaError_t e = cudaSuccess;
  if (g.dim == 1 && fwd1d_tma_ok(g, st, T)) {   // TMA-staged tile (the product 1-D path)
    CUtensorMap tmu, tmh, tmx;
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_fn());
    const cuuint64_t dims[3] = {(cuuint64_t)2 * g.N, (cuuint64_t)g.M, (cuuint64_t)g.L};
    const cuuint64_t strides[2] = {(cuuint64_t)g.N * 16, (cuuint64_t)g.M * g.N * 16};
    const cuuint32_t es[3] = {1, 1, 1};
    const cuuint32_t BL = (cuuint32_t)g.L;
    const cuuint32_t boxu[3] = {2 * 4, (cuuint32_t)g.M, BL}, boxh[3] = {2, (cuuint32_t)g.M, BL};
    if (!enc ||
        enc(&tmu, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)b.u, dims, strides, boxu, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&tmh, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)b.u, dims, strides, boxh, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)b.X, dims, strides, boxu, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
    const size_t slot = (size_t)g.L * g.M * (4 + 2) * sizeof(double2);
    const size_t head = 1024 + (((size_t)g.L * sizeof(double2) + 1023) & ~(size_t)1023);
    int NS = 3;
    while (NS > 2 && 1024 + head + NS * slot > 227 * 1024) --NS;
    const size_t sm1 = 1024 + head + NS * slot;
    const int ntiles = g.N / 4;
    int grid = num_sms();
    if (grid > ntiles) grid = ntiles;
    switch (g.M) {
#define PINT_FWDT(MM_)                                                                                        \
  case MM_:                                                                                                   \
    e = set_smem((const void *)fwd1d_tma_kernel<MM_>, sm1);                                                   \
    if (e == cudaSuccess)                                                                                     \
      fwd1d_tma_kernel<MM_><<<grid, kFwdTmaGT * kFwdTmaG, sm1, s>>>(tmu, tmh, tmx, g, st, at, NS, ntiles);          \
    break;
      PINT_FWDT(1) PINT_FWDT(2) PINT_FWDT(3) default: PINT_FWDT(4)
#undef PINT_FWDT
    }
    rec(s);
  } else if (g.dim == 1) {
#define PINT_FWD1(NODE_, PACK_, HW_)                                                              \
  e = set_smem((const void *)fwd_kernel<MM, true, NODE_, PACK_, HW_>, smem);                       \
  if (e == cudaSuccess) fwd_kernel<MM, true, NODE_, PACK_, HW_><<<grid, kTileThreads, smem, s>>>(g, st, at, b.u, b.X, T);
    const bool wide = g.hw > 1;   // the 5-/7-point stencils (reading R14)
    PINT_DISPATCH_M(g.M, {
      if (st.packed) {
        if (wide) { PINT_FWD1(true, true, 3) } else { PINT_FWD1(true, true, 1) }
      } else if (st.P == 1) {
        if (wide) { PINT_FWD1(true, false, 3) } else { PINT_FWD1(true, false, 1) }
      } else {
        if (wide) { PINT_FWD1(false, false, 3) } else { PINT_FWD1(false, false, 1) }
      }
    });
#undef PINT_FWD1
    rec(s);
  } else {
    const bool pk = st.packed != 0;   // Hermitian mode: two real points per complex time series
    int BX, BY;
    residual_block(g, BX, BY);
    const bool xp = pk && st.xpair;
    if (pk && !xp && BY > g.ny / 2) BY = g.ny / 2;
    if (xp && BX > g.nx / 2) BX = g.nx / 2;
    const int hw = g.hw < 1 ? 1 : g.hw;
    auto rbytes = [&](int bx, int by) {   // tile + (complex storage) the staged H-term block
      return (size_t)g.M * (bx + 2 * hw) * (by + 2 * hw) * (pk ? 2 * sizeof(double) : sizeof(double2)) +
             (pk ? 0 : (size_t)bx * by * sizeof(double2));
    };
    while (rbytes(BX, BY) > 200 * 1024) {   // wide halos at large M: smaller blocks
      if (BY > 1) BY >>= 1;
      else BX >>= 1;
    }
    const size_t rs = rbytes(BX, BY);
    const int rgrid = g.L * ((xp ? g.nx / 2 : g.nx) / BX) * ((pk && !xp ? g.ny / 2 : g.ny) / BY);
    // step-grouped block order where a plane no longer fits L2 comfortably (config 5: 16 MB planes,
    // 14.3 -> 13.6 ms measured in round 1; config 4's 4 MB planes: slower, so not there)
    int lg = (size_t)g.N * sizeof(double2) >= ((size_t)8 << 20) ? 8 : 1;
    while (lg > 1 && g.L % lg) lg >>= 1;
    // complex storage: the halo tile of an interior block is one tensor box of u (TMA); PINT_RES_TMA=0
    // (experiments build) keeps the cp.async staging everywhere for A/B runs
    CUtensorMap tmu{};
    int tma = 0;
    if (!pk && 2 * (BX + 2 * hw) <= 256 && BY + 2 * hw <= 256 && g.M <= 256) {
      const char *ev = experiment_env("PINT_RES_TMA");
      auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_fn());
      const cuuint64_t dims[3] = {(cuuint64_t)2 * g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.L * g.M};
      const cuuint64_t strides[2] = {(cuuint64_t)g.nx * 16, (cuuint64_t)g.N * 16};
      const cuuint32_t box[3] = {(cuuint32_t)(2 * (BX + 2 * hw)), (cuuint32_t)(BY + 2 * hw), (cuuint32_t)g.M};
      const cuuint32_t es[3] = {1, 1, 1};
      tma = enc && !(ev && !atoi(ev)) &&
            enc(&tmu, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)b.u, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
#define PINT_RES2D(MM_, PK_, HW_)                                                                   \
  e = set_smem((const void *)residual2d_kernel<MM_, PK_, HW_>, rs, true);                            \
  if (e == cudaSuccess) residual2d_kernel<MM_, PK_, HW_><<<rgrid, 256, rs, s>>>(tmu, tma, g, st, at, b.u, b.X, BX, BY, lg);
    PINT_DISPATCH_M(g.M, {
      if (pk) {
        if (hw == 1) { PINT_RES2D(MM, true, 1) } else if (hw == 2) { PINT_RES2D(MM, true, 2) } else { PINT_RES2D(MM, true, 3) }
      } else {
        if (hw == 1) { PINT_RES2D(MM, false, 1) } else if (hw == 2) { PINT_RES2D(MM, false, 2) } else { PINT_RES2D(MM, false, 3) }
      }
    });
#undef PINT_RES2D
    rec(s);
    if (e != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (!pk && tfft_pipe_supported(g, st) && !legacy_tfft()) {   // pipelined (TMA ring) time FFT
      e = launch_tfft_pipe(g, st, &at, b.X, nullptr, b.u, false, nullptr, 0, s);
      rec(s);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
    Geometry gt = g;                  // time transform over N (or N/2 packed columns)
    if (pk) gt.N = g.N / 2;
    int T2 = lc.tfft_T;
    while (T2 > gt.N) T2 >>= 1;
    const size_t sm2 = (size_t)g.L * (T2 + 1) * sizeof(double2);   // tile + staged twiddles
    if (T2 == lc.tfft_T && tfft_tma_ok(gt, st, T2)) {   // tile moved by the TMA unit
      CUtensorMap tmx;
      if (!time_tile_map(gt, b.X, T2, tmx)) return cudaErrorNotSupported;
      e = set_smem((const void *)tfft_fwd_tma_kernel, sm2);
      if (e == cudaSuccess) tfft_fwd_tma_kernel<<<g.M * (gt.N / T2), kTileThreads, sm2, s>>>(tmx, gt, st, T2);
    } else {
      e = set_smem((const void *)tfft_fwd_kernel, sm2);
      if (e == cudaSuccess) tfft_fwd_kernel<<<g.M * (gt.N / T2), kTileThreads, sm2, s>>>(gt, st, b.X, T2);
    }
    rec(s);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_solve(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                         const AlphaTables &at, const Buffers &b, cudaStream_t s, double2 **out) {
  cudaError_t e = cudaSuccess;
  if (!g.pow2) {   // generic grids: node transforms + mixed-radix FFT-diagonal solves (generic.cu)
    *out = b.X;
    return launch_generic_solve(g, st, at, b.X, s);
  }
  const int lines = st.nsolve * g.M;   // solved units x nodes (Hermitian mode: k <= L/2)
  if (g.dim == 1) {
    if (lc.pcr_mode == 0) {
      const size_t smem = (size_t)g.N * sizeof(double2);
      if ((e = launch_pcr_classes(g, at, b.X, 1, 1, 0, nullptr, st.slots, lines, smem, s)) != cudaSuccess) return e;
      rec(s);
      *out = b.X;
    } else {
      const int R = lc.pcr_R, T = lc.pcr_T;
      const int jOff = __builtin_ctz((unsigned)R);
      if (pcr1d_path(g, lc)) {   // pipelined class + chunk passes (pcr1d.cu), each launch recorded
        *out = b.Y;
        return launch_pcr1d_pipe(g, at, b.X, b.Y, st.slots, lines, R, s, st.sm_reserve);
      }
      const int nq = g.N / R;
      size_t smem = (size_t)nq * T * sizeof(double2);
      constexpr int E = 8;
      const int Sr = nq / E, Tr = Sr > 0 ? 256 / Sr : 0;
      if (nq >= E && Sr <= 32 && Tr >= 1 && Tr <= R) {
        const size_t smr = (size_t)nq * Tr * sizeof(double2);
        if ((e = launch_pcr_reg<E>(g, at, b.X, R, Tr, jOff, nullptr, st.slots, lines * (R / Tr), smr, s)) != cudaSuccess)
          return e;
      } else {
        if ((e = launch_pcr_classes(g, at, b.X, R, T, jOff, nullptr, st.slots, lines * (R / T), smem, s)) != cudaSuccess) return e;
      }
      rec(s);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      const int C = lc.pcr_chunk, H = R * g.nfac;
      if (C + 2 * H > kChunkThreads * kChunkIPT) return cudaErrorInvalidConfiguration;   // see choose_launch
      smem = (size_t)(C + 2 * H) * sizeof(double2);
      if ((e = set_smem((const void *)pcr_chunk_kernel, smem)) != cudaSuccess) return e;
      pcr_chunk_kernel<<<lines * (g.N / C), kChunkThreads, smem, s>>>(g, at, b.X, b.Y, C, H, jOff, st.slots);
      rec(s);
      *out = b.Y;
    }
  } else if (pipe2d(g, st) && spatial_fused_supported(g, st)) {
    e = launch_spatial_fused(g, st, at, b.X, b.Y, b.sync, s);   // R, C, I items in one launch
    *out = b.X;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  } else if (pipe2d(g, st)) {
    e = launch_spatial_pipe(g, st, at, b.X, b.Y, s);   // R, C, I: three launches, each recorded
    *out = b.X;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  } else if (reg2d(g)) {
    e = launch_spatial2d(g, st, at, b.X, nullptr, b.sync, st.nsolve * g.M, s);
    rec(s);
    *out = b.X;
    if (e != cudaSuccess) return e;
  } else {
    // row passes: one frequency p and YG rows y per CTA (M*YG*nx <= 4096 elements = 64 KB)
    int YG = 4096 / (g.M * g.nx);
    if (YG < 1) YG = 1;
    if (YG > g.ny) YG = g.ny;
    while (g.ny % YG) YG >>= 1;
    const size_t smem = (size_t)YG * g.M * g.nx * sizeof(double2);
    const unsigned rgrid = (unsigned)(g.L * (g.ny / YG));
    PINT_DISPATCH_M(g.M, {
      if (st.P == 1) {
        e = set_smem((const void *)fft2d_rows_kernel<MM, false, true>, smem);
        if (e == cudaSuccess) e = set_smem((const void *)fft2d_rows_kernel<MM, true, true>, smem);
        if (e == cudaSuccess) fft2d_rows_kernel<MM, false, true><<<rgrid, kFftThreads, smem, s>>>(g, st, at, b.X, YG);
      } else {
        e = set_smem((const void *)fft2d_rows_kernel<MM, false, false>, smem);
        if (e == cudaSuccess) e = set_smem((const void *)fft2d_rows_kernel<MM, true, false>, smem);
        if (e == cudaSuccess) fft2d_rows_kernel<MM, false, false><<<rgrid, kFftThreads, smem, s>>>(g, st, at, b.X, YG);
      }
    });
    rec(s);
    if (e != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int T = 8192 / g.ny;                 // 128 KB tile, one 512-thread CTA per SM
    if (T < 1) T = 1;
    if (T > g.nx) T = g.nx;
    if (T > 16) T = 16;
    size_t smc = (size_t)g.ny * T * sizeof(double2);
    if ((e = set_smem((const void *)fft2d_cols_kernel, smc)) != cudaSuccess) return e;
    fft2d_cols_kernel<<<lines * (g.nx / T), kColThreads, smc, s>>>(g, st, at, b.X, T);
    rec(s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    PINT_DISPATCH_M(g.M, {
      if (st.P == 1) fft2d_rows_kernel<MM, true, true><<<rgrid, kFftThreads, smem, s>>>(g, st, at, b.X, YG);
      else fft2d_rows_kernel<MM, true, false><<<rgrid, kFftThreads, smem, s>>>(g, st, at, b.X, YG);
    });
    rec(s);
    *out = b.X;
  }
  return cudaGetLastError();
}

cudaError_t launch_backward(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                            const AlphaTables &at, const Buffers &b, const double2 *x2,
                            double *diff_slot, cudaStream_t s, int overwrite) {
  int T = lc.bwd_T;
  if (st.packed) while (T > g.N / 2) T >>= 1;
  const size_t smem = fwd_smem_bytes(g, T);
  const int grid = (st.packed && g.dim == 1 ? g.N / 2 : g.N) / T;
  cudaError_t e = cudaSuccess;
  if (!g.pow2) {   // generic grids: G^{-1} S was applied by the solve; inverse DFT on T | N columns
    const int T2 = lc.tfft_T;
    const size_t sm2 = (size_t)g.L * T2 * sizeof(double2);
    e = set_smem((const void *)tfft_bwd_kernel<false>, sm2);
    if (e == cudaSuccess)
      tfft_bwd_kernel<false><<<g.M * (g.N / T2), kTileThreads, sm2, s>>>(g, st, at, x2, b.u, T2,
                                                                           (unsigned long long *)diff_slot, overwrite);
  } else if (g.dim == 1) {
    // complex storage: tile in by a tensor load, u += c out as a TMA reduce-add (bwd1d_tma_ok)
    CUtensorMap tmx2{}, tmu{};
    int tma = 0;
    if (bwd1d_tma_ok(g, st, T)) {
      auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_fn());
      const cuuint64_t dims[3] = {(cuuint64_t)2 * g.N, (cuuint64_t)g.M, (cuuint64_t)g.L};
      const cuuint64_t strides[2] = {(cuuint64_t)g.N * 16, (cuuint64_t)g.M * g.N * 16};
      const cuuint32_t box[3] = {(cuuint32_t)(2 * T), (cuuint32_t)g.M, (cuuint32_t)(g.L < 256 ? g.L : 256)};
      const cuuint32_t es[3] = {1, 1, 1};
      tma = enc(&tmx2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)x2, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
            enc(&tmu, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)b.u, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    PINT_DISPATCH_M(g.M, {
      if (st.packed) {
        e = set_smem((const void *)bwd_kernel<MM, true, true>, smem);
        if (e == cudaSuccess)
          bwd_kernel<MM, true, true><<<grid, kTileThreads, smem, s>>>(tmx2, tmu, 0, g, st, at, x2, b.u, T, (unsigned long long *)diff_slot, overwrite);
      } else if (st.P == 1) {
        e = set_smem((const void *)bwd_kernel<MM, true>, smem);
        if (e == cudaSuccess)
          bwd_kernel<MM, true><<<grid, kTileThreads, smem, s>>>(tmx2, tmu, tma, g, st, at, x2, b.u, T, (unsigned long long *)diff_slot, overwrite);
      } else {
        e = set_smem((const void *)bwd_kernel<MM, false>, smem);
        if (e == cudaSuccess)
          bwd_kernel<MM, false><<<grid, kTileThreads, smem, s>>>(tmx2, tmu, tma, g, st, at, x2, b.u, T, (unsigned long long *)diff_slot, overwrite);
      }
    });
  } else if (st.packed) {
    int T2 = lc.tfft_T;
    while (T2 > g.N / 2) T2 >>= 1;
    const size_t sm2 = (size_t)g.L * T2 * sizeof(double2);
    e = set_smem((const void *)tfft_bwd_kernel<true>, sm2);
    if (e == cudaSuccess)
      tfft_bwd_kernel<true><<<g.M * (g.N / 2 / T2), kTileThreads, sm2, s>>>(
          g, st, at, unit_planes(g, b.X), b.u, T2, (unsigned long long *)diff_slot, overwrite);
  } else if (tfft_pipe_supported(g, st) && !legacy_tfft()) {   // pipelined (TMA ring) inverse time FFT
    e = launch_tfft_pipe(g, st, &at, b.X, x2, b.u, true, (unsigned long long *)diff_slot, overwrite, s);
  } else {
    const int T2 = lc.tfft_T;
    const size_t sm2 = (size_t)g.L * T2 * sizeof(double2);
    if (tfft_bwd_tma_ok(g, st, T2)) {   // TMA tile in, u += c as a TMA reduce-add (overwrite: a store)
      CUtensorMap tmx2, tmu;
      if (!time_tile_map(g, x2, T2, tmx2) || !time_tile_map(g, b.u, T2, tmu)) return cudaErrorNotSupported;
      e = set_smem((const void *)tfft_bwd_tma_kernel, sm2);
      if (e == cudaSuccess)
        tfft_bwd_tma_kernel<<<g.M * (g.N / T2), kTileThreads, sm2, s>>>(tmx2, tmu, g, st, at, b.u, T2,
                                                                        (unsigned long long *)diff_slot, overwrite);
    } else {
      e = set_smem((const void *)tfft_bwd_kernel<false>, sm2);
      if (e == cudaSuccess)
        tfft_bwd_kernel<false><<<g.M * (g.N / T2), kTileThreads, sm2, s>>>(g, st, at, x2, b.u, T2,
                                                                             (unsigned long long *)diff_slot, overwrite);
    }
  }
  rec(s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int launches_per_iteration_direct(const Geometry &g, const LaunchCfg &lc, const StaticTables &st) {
  // r0, plane rows, plane cols, [spatial2d | synthesized cols, rows<inv>], bwd
  if (g.dim == 2) return pipe2d(g, st) ? 7 : reg2d(g) ? 5 : 6;
  return lc.pcr_mode == 0 ? 3 : 4;            // r0, pcr (1 or 2), bwd
}

const char *kernel_name_direct(const Geometry &g, const LaunchCfg &lc, const StaticTables &st, int i) {
  static const char *k1a[] = {"direct_r0_kernel", "pcr_classes_kernel", "bwd_kernel"};
  static const char *k1b[] = {"direct_r0_kernel", "pcr_classes_kernel", "pcr_chunk_kernel", "bwd_kernel"};
  static const char *k2[] = {"direct_r0_kernel", "plane_rows_dif_kernel", "plane_cols_dif_kernel",
                             "cols_direct_kernel", "fft2d_rows_kernel<inv>", "tfft_bwd_kernel"};
  static const char *k2p[] = {"direct_r0_kernel", "plane_rows_dif_kernel", "plane_cols_dif_kernel",
                              "spatial2d_kernel", "tfft_bwd_kernel"};
  static const char *k2q[] = {"direct_r0_kernel", "plane_rows_dif_kernel", "plane_cols_dif_kernel", "spec_blocked_kernel",
                              "cols_pipe_kernel<synth>", "rows_pipe_kernel<inv>", "tfft_bwd_kernel"};
  const int n = launches_per_iteration_direct(g, lc, st);
  if (i < 0 || i >= n) return "";
  if (g.dim == 2) {
    if (i == n - 1 && tfft_pipe_supported(g, st) && !legacy_tfft()) return "tfft_pipe_kernel<inv>";
    if (i == n - 1 && !st.packed && tfft_bwd_tma_ok(g, st, lc.tfft_T)) return "tfft_bwd_tma_kernel";
    if (pipe2d(g, st)) return k2q[i];
    return reg2d(g) ? k2p[i] : k2[i];
  }
  return lc.pcr_mode == 0 ? k1a[i] : k1b[i];
}

cudaError_t launch_direct_r0(const Geometry &g, const StaticTables &st, const AlphaTables &at, const Buffers &b,
                             double2 *r0, cudaStream_t s) {
  int blocks = (g.N + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  direct_r0_kernel<<<blocks, 256, 0, s>>>(g, st, at, b.u, r0);
  rec(s);
  return cudaGetLastError();
}

cudaError_t launch_direct_front(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                const AlphaTables &at, const Buffers &b, double2 *r0, cudaStream_t s) {
  cudaError_t e = launch_direct_r0(g, st, at, b, r0, s);
  if (e != cudaSuccess) return e;
  return launch_direct_spectrum(g, lc, st, at, b, r0, s);
}

cudaError_t launch_direct_spectrum(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                   const AlphaTables &at, const Buffers &b, double2 *r0, cudaStream_t s) {
  (void)lc;
  cudaError_t e = cudaSuccess;
  if (g.dim == 1) return e;
  int YG = 4096 / g.nx;
  if (YG < 1) YG = 1;
  if (YG > g.ny) YG = g.ny;
  size_t smr = (size_t)YG * g.nx * sizeof(double2);
  if ((e = set_smem((const void *)plane_rows_dif_kernel, smr)) != cudaSuccess) return e;
  plane_rows_dif_kernel<<<g.ny / YG, kFftThreads, smr, s>>>(g, st, r0, YG);
  rec(s);
  int Tp = 4096 / g.ny;
  if (Tp < 1) Tp = 1;
  if (Tp > g.nx) Tp = g.nx;
  size_t smc = (size_t)g.ny * Tp * sizeof(double2);
  if ((e = set_smem((const void *)plane_cols_dif_kernel, smc)) != cudaSuccess) return e;
  plane_cols_dif_kernel<<<g.nx / Tp, kFftThreads, smc, s>>>(g, st, r0, Tp);
  rec(s);
  if (reg2d(g)) return cudaGetLastError();   // the synthesized column pass runs inside spatial2d
  int T = 8192 / g.ny;
  if (T < 1) T = 1;
  if (T > g.nx) T = g.nx;
  if (T > 16) T = 16;
  size_t smd = (size_t)g.ny * T * sizeof(double2);
  if ((e = set_smem((const void *)cols_direct_kernel, smd)) != cudaSuccess) return e;
  cols_direct_kernel<<<g.L * g.M * (g.nx / T), kColThreads, smd, s>>>(g, st, at, r0, b.X, T);
  rec(s);
  return cudaGetLastError();
}

cudaError_t launch_sequential_step(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                                   const Buffers &b, double2 *r0, double2 *out, cudaStream_t s) {
  int YG = 4096 / g.nx;
  if (YG < 1) YG = 1;
  if (YG > g.ny) YG = g.ny;
  cudaError_t e;
  size_t smr = (size_t)YG * g.nx * sizeof(double2);
  if ((e = set_smem((const void *)plane_rows_dif_kernel, smr)) != cudaSuccess) return e;
  plane_rows_dif_kernel<<<g.ny / YG, kFftThreads, smr, s>>>(g, st, r0, YG);
  int Tp = 4096 / g.ny;
  if (Tp < 1) Tp = 1;
  if (Tp > g.nx) Tp = g.nx;
  size_t smc = (size_t)g.ny * Tp * sizeof(double2);
  if ((e = set_smem((const void *)plane_cols_dif_kernel, smc)) != cudaSuccess) return e;
  plane_cols_dif_kernel<<<g.nx / Tp, kFftThreads, smc, s>>>(g, st, r0, Tp);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return launch_spatial2d(g, st, at, out, r0, b.sync, g.M, s);
}

cudaError_t launch_direct_solve(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                const AlphaTables &at, const Buffers &b, const double2 *r0, cudaStream_t s,
                                double2 **out) {
  cudaError_t e = cudaSuccess;
  const int lines = st.nsolve * g.M;   // solved units x nodes (Hermitian mode: k <= L/2)
  if (pipe2d(g, st) && b.Y != b.X) {   // synthesized C pass + I pass (each launch recorded)
    *out = b.X;
    e = launch_spatial_pipe(g, st, at, b.X, b.Y, s, r0);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  if (reg2d(g)) {
    e = launch_spatial2d(g, st, at, b.X, r0, b.sync, st.nsolve * g.M, s);
    rec(s);
    *out = b.X;
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  if (g.dim == 2) {
    int YG = 4096 / (g.M * g.nx);
    if (YG < 1) YG = 1;
    if (YG > g.ny) YG = g.ny;
    while (g.ny % YG) YG >>= 1;
    const size_t smem = (size_t)YG * g.M * g.nx * sizeof(double2);
    const unsigned rgrid = (unsigned)(g.L * (g.ny / YG));
    PINT_DISPATCH_M(g.M, {   // P > 1: G^{-1} S lives in the inverse cross-rank DFT
      if (st.P == 1) {
        e = set_smem((const void *)fft2d_rows_kernel<MM, true, true>, smem);
        if (e == cudaSuccess) fft2d_rows_kernel<MM, true, true><<<rgrid, kFftThreads, smem, s>>>(g, st, at, b.X, YG);
      } else {
        e = set_smem((const void *)fft2d_rows_kernel<MM, true, false>, smem);
        if (e == cudaSuccess) fft2d_rows_kernel<MM, true, false><<<rgrid, kFftThreads, smem, s>>>(g, st, at, b.X, YG);
      }
    });
    rec(s);
    *out = b.X;
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  if (lc.pcr_mode == 0) {
    const size_t smem = (size_t)g.N * sizeof(double2);
    if ((e = launch_pcr_classes(g, at, b.X, 1, 1, 0, r0, st.slots, lines, smem, s)) != cudaSuccess) return e;
    rec(s);
    *out = b.X;
    return cudaGetLastError();
  }
  const int R = lc.pcr_R, T = lc.pcr_T;
  const int jOff = __builtin_ctz((unsigned)R);
  const int nq = g.N / R;
  constexpr int E = 8;
  const int Sr = nq / E, Tr = Sr > 0 ? 256 / Sr : 0;
  if (nq >= E && Sr <= 32 && Tr >= 1 && Tr <= R) {
    const size_t smr = (size_t)nq * Tr * sizeof(double2);
    if ((e = launch_pcr_reg<E>(g, at, b.X, R, Tr, jOff, r0, st.slots, lines * (R / Tr), smr, s)) != cudaSuccess)
      return e;
  } else {
    const size_t smem = (size_t)nq * T * sizeof(double2);
    if ((e = launch_pcr_classes(g, at, b.X, R, T, jOff, r0, st.slots, lines * (R / T), smem, s)) != cudaSuccess) return e;
  }
  rec(s);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int C = lc.pcr_chunk, H = R * g.nfac;
  const size_t smc = (size_t)(C + 2 * H) * sizeof(double2);
  if ((e = set_smem((const void *)pcr_chunk_kernel, smc)) != cudaSuccess) return e;
  pcr_chunk_kernel<<<lines * (g.N / C), kChunkThreads, smc, s>>>(g, at, b.X, b.Y, C, H, jOff, st.slots);
  rec(s);
  *out = b.Y;
  return cudaGetLastError();
}

// U_m = sum_j V_mj y_j (the node basis back-transform of a sequential step)
template <int M>
__global__ void seq_node_mix_kernel(const double2 *__restrict__ V, const double2 *__restrict__ y,
                                    double2 *__restrict__ out, int N) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    double2 v[M];
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = __ldg(y + (size_t)j * N + n);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < M; ++j) acc = cfma(__ldg(V + m * M + j), v[j], acc);
      out[(size_t)m * N + n] = acc;
    }
  }
}

cudaError_t launch_sequential_step_1d(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                      const AlphaTables &at, const Buffers &b, double2 *r0, double2 *out,
                                      cudaStream_t s) {
  double2 *y = nullptr;
  cudaError_t e = launch_direct_solve(g, lc, st, at, b, r0, s, &y);
  if (e != cudaSuccess) return e;
  const int blocks = (g.N + 255) / 256 < num_sms() * 4 ? (g.N + 255) / 256 : num_sms() * 4;
  PINT_DISPATCH_M(g.M, { seq_node_mix_kernel<MM><<<blocks, 256, 0, s>>>(at.SG, y, out, g.N); });
  return cudaGetLastError();
}

cudaError_t launch_residual_norm(const Geometry &g, const StaticTables &st, const Buffers &b,
                                 double *out2, cudaStream_t s) {
  const long long total = (long long)g.L * g.N;
  int blocks = (int)((total + 255) / 256);
  const int cap = 148 * 8;  // partials scratch is sized for 148*8 blocks (pint_abi.cpp layout)
  if (blocks > cap) blocks = cap;
  PINT_DISPATCH_M(g.M, {
    if (g.pow2) resnorm_kernel<MM><<<blocks, 256, 0, s>>>(g, st, b.u, b.red);
    else resnorm_kernel<MM, false><<<blocks, 256, 0, s>>>(g, st, b.u, b.red);
  });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  reduce_partials_kernel<<<1, 32, 0, s>>>(b.red, blocks, out2);
  return cudaGetLastError();
}

cudaError_t launch_halo_pack(const Geometry &g, const Buffers &b, double2 *hsend, cudaStream_t s) {
  const long long total = (long long)g.L * g.N;
  long long blocks = (total + 255) / 256;
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
  halo_pack_kernel<<<(int)blocks, 256, 0, s>>>(g, b.u, hsend);
  rec(s);
  return cudaGetLastError();
}

cudaError_t launch_xdft(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                        const double2 *in, double2 *out, bool inverse, cudaStream_t s, int pl0, int npl) {
  if (npl < 0) npl = g.L / st.P - pl0;
  const long long total = (long long)npl * g.N;
  long long blocks = (total + 255) / 256;
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
  cudaError_t e = cudaErrorInvalidValue;
#define PINT_XDFT(PP)                                                                          \
  if (st.P == PP) {                                                                            \
    PINT_DISPATCH_M(g.M, {                                                                     \
      if constexpr (MM * PP <= 32) {                                                           \
        if (inverse) xdft_kernel<MM, PP, true><<<(int)blocks, 256, 0, s>>>(g, st, at, in, out, pl0, npl); \
        else xdft_kernel<MM, PP, false><<<(int)blocks, 256, 0, s>>>(g, st, at, in, out, pl0, npl);       \
        e = cudaGetLastError();                                                                \
      }                                                                                        \
    });                                                                                        \
  }
  PINT_XDFT(2)
  PINT_XDFT(4)
  PINT_XDFT(8)
#undef PINT_XDFT
  rec(s);
  return e;
}

__global__ void square_first_kernel(const double *in, double *out) { out[0] = in[0] * in[0]; }
__global__ void sqrt_into_kernel(const double *in, double *out) { out[0] = sqrt(in[0]); }
cudaError_t launch_square_first(const double *in, double *out, cudaStream_t s) {
  square_first_kernel<<<1, 1, 0, s>>>(in, out);
  return cudaGetLastError();
}
cudaError_t launch_sqrt_into(const double *in, double *out, cudaStream_t s) {
  sqrt_into_kernel<<<1, 1, 0, s>>>(in, out);
  return cudaGetLastError();
}

cudaError_t launch_w_inf(const Geometry &g, const StaticTables &st, double *out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  w_inf_kernel<<<num_sms() * 4, 256, 0, s>>>(g, st, (unsigned long long *)out);
  return cudaGetLastError();
}

cudaError_t launch_init_iterate(const Geometry &g, const StaticTables &st, const Buffers &b, cudaStream_t s) {
  const long long total = (long long)g.L * g.M * g.N;
  long long blocks = (total + 255) / 256;
  if (blocks > num_sms() * 32) blocks = num_sms() * 32;
  init_iterate_kernel<<<(int)blocks, 256, 0, s>>>(g, st.u0, b.u, st.packed);
  return cudaGetLastError();
}

cudaError_t launch_storage_convert(const Geometry &g, const Buffers &b, bool to_real, cudaStream_t s) {
  const long long n = (long long)g.L * g.M * g.N;
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  double *tmp = (double *)b.X;   // scratch: X holds >= L M N complex values
  if (to_real) {
    real_parts_kernel<<<blocks, 256, 0, s>>>(b.u, tmp, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync((void *)b.u, tmp, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  }
  cudaError_t e = cudaMemcpyAsync(tmp, (const void *)b.u, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  complex_from_real_kernel<<<blocks, 256, 0, s>>>(tmp, b.u, n);
  return cudaGetLastError();
}

}  // namespace pint
