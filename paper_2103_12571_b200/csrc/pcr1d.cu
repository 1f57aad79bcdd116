// 1-D spatial solves (north star step (iv), Alg. 1) as two pipelined
// persistent passes of parallel cyclic reduction on the constant-coefficient cyclic tridiagonal
// (I - d_km dT A) x = y (row sum carried in the host's level coefficients, reading R6).
//
// PCR level j (stride h = 2^j): y_i <- y_i - p_j y_{i-h} - q_j y_{i+h}; the last level (h = N/2)
// y_i <- y_i - p y_{i+h}; then x = y / e.  The level operators are circulants, so they commute
// and the two-pass split of kernels.cu holds: the strides h >= R are closed on residue classes
// mod R (class pass, in place on X), the strides h < R run on contiguous chunks with a halo of
// R - 1 points each side (chunk pass, X -> Y).  These kernels implement the split for classes of
// NQ = 256 points (N = 256 R, R <= 256) and the 3-point operators (one tridiagonal factor);
// other shapes keep the smem kernels of kernels.cu.
//
// Both passes are persistent (one CTA per SM) with a ring of shared-memory slots filled by the
// TMA unit (class pass: a tensor-map box of 8 consecutive classes x 256 rows, 128-byte swizzle;
// chunk pass: 1-D bulk copies of the chunk and its halos) completing on one mbarrier per slot,
// G consumer groups taking alternate items, and the group that has finished reading a slot
// refilling it with the CTA's item k + NS (ring order = item order).  The levels run on values
// held in registers, 16 per thread:
//   class pass:  CLASS arrangement (thread holds q = beta + 16 k of one class column): strides
//                h' = 16, 32, 64, 128 are cyclic shifts of k, closed in registers; one shared-
//                memory transposition to the BLOCK arrangement (q = 16 b + e), strides 1, 2, 4, 8
//                with the edge values from lanes b -/+ 1 by width-16 warp shuffles; x = y / e is
//                stored from registers;
//   chunk pass:  COMB arrangement (thread holds p = 256 B + beta + 16 e of the tile): strides
//                16 .. 128 are shifts of e, the edge teeth come through the slot (natural
//                positions); a transposition to the BLOCK arrangement (p = 16 t + e, swizzled
//                positions) for strides 1 .. 8, edges again through the slot; a transposition
//                back to the comb arrangement for coalesced stores of the chunk's core.
// Levels whose stencil reaches outside the tile read clamped positions: their results fall in
// the halo, which the chunk pass never stores (radius of the strides < R is R - 1 <= H).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"
#include "internal.h"

namespace pint {

namespace {

constexpr int kE = 16;        // values per thread
constexpr int kNQ = 256;      // class length of the class pass
constexpr int kTC = 8;        // class columns per class-pass item (128-byte rows)
constexpr int kCH = 256;      // chunk halo (>= R - 1)
// shared-memory header of both kernels: NS mbarriers, NS slot tags, then per slot the item's level
// coefficients (up to 8 levels x (p, q)) and 1/e, brought by the same bulk copies as the data
constexpr int kHdrCoef = 128;             // byte offset of the coefficient area
constexpr int kCoefPerSlot = 17;          // double2: 16 level coefficients + 1/e
constexpr int kHdrBytes = 4096;           // NS <= 8

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// wait for CTA-local item k in slot k mod NS (slot tags: see ring_wait in spatial2d.cu)
__device__ __forceinline__ void slot_wait(uint64_t *bar, volatile int *slot_item, int k, int NS) {
  while (slot_item[k % NS] != k) __nanosleep(32);
  mbar_wait(bar, (unsigned)((k / NS) & 1));
}

__device__ __forceinline__ unsigned char *align_1024(unsigned char *p) {
  const unsigned a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

__device__ __forceinline__ int tline_of(const Geometry &g, const int *slots, int line) {
  return __ldg(slots + line / g.M) * g.M + line % g.M;
}

// One PCR update; sym = +1: q == p (heat family, and centred advection after level 0), -1: q == -p
// (centred advection, level 0), 0: general.  sym is uniform over the CTA.
__device__ __forceinline__ double2 lvl_update(int sym, double2 p, double2 q, double2 lv, double2 rv, double2 y) {
  if (sym > 0) return cfms(p, cadd(lv, rv), y);
  if (sym < 0) return cfms(p, csub(lv, rv), y);
  return cfms(q, rv, cfms(p, lv, y));
}
__device__ __forceinline__ int lvl_sym(double2 p, double2 q) {
  if (p.x == q.x && p.y == q.y) return 1;
  if (p.x == -q.x && p.y == -q.y) return -1;
  return 0;
}
// compile-time level form: SYM = true for the centred 3-point operators (heat: q == p at every
// level; centred advection: q == -p at level 0, q == p after), sg = q / p in {+1, -1}; SYM =
// false: the general two-product update
template <bool SYM>
__device__ __forceinline__ double2 upd(double2 p, double2 q, double sg, double2 lv, double2 rv, double2 y) {
  if constexpr (SYM) return cfms(p, make_double2(fma(sg, rv.x, lv.x), fma(sg, rv.y, lv.y)), y);
  else return cfms(q, rv, cfms(p, lv, y));
}

// cyclic in-register level over the 16 values (shift S in k), PAIR: y - p y_{k+S} only
template <int S, bool PAIR, bool SYM>
__device__ __forceinline__ void cyc_level(double2 (&y)[kE], double2 p, double2 q) {
  double2 nv[kE];
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const double2 rv = y[(k + S) & (kE - 1)];
    nv[k] = PAIR ? cfms(p, rv, y[k]) : upd<SYM>(p, q, 1.0, y[(k - S) & (kE - 1)], rv, y[k]);
  }
#pragma unroll
  for (int k = 0; k < kE; ++k) y[k] = nv[k];
}

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src, 16), __shfl_sync(0xffffffffu, v.y, src, 16));
}

// block level (stride H < 16) on q = 16 b + e, edges from lanes b -/+ 1 (cyclic over 16 lanes)
template <int H, bool SYM>
__device__ __forceinline__ void blk_level(double2 (&y)[kE], int b, double2 p, double2 q, double sg) {
  const int left = (b + 15) & 15, right = (b + 1) & 15;
  double2 lx[H], rx[H];
#pragma unroll
  for (int e = 0; e < H; ++e) {
    lx[e] = shfl2(y[kE - H + e], left);   // left neighbour's y[16 - H + e] = position 16 b + e - H
    rx[e] = shfl2(y[e], right);           // right neighbour's y[e]        = position 16 b + 16 + e
  }
  double2 nv[kE];
#pragma unroll
  for (int e = 0; e < kE; ++e) {
    const double2 lv = e >= H ? y[e - H] : lx[e];
    const double2 rv = e + H < kE ? y[e + H] : rx[e + H - kE];
    nv[e] = upd<SYM>(p, q, sg, lv, rv, y[e]);
  }
#pragma unroll
  for (int e = 0; e < kE; ++e) y[e] = nv[e];
}

// transposition layout of the class pass: element (q, col) of a [256][8] slot at
// q * 8 + (col ^ ((q ^ (q >> 4)) & 7)) -- conflict-free for q = beta + 16 k (8 consecutive beta)
// and for q = 16 b + e (8 consecutive b)
__device__ __forceinline__ int cls_sw(int q, int col) { return (q << 3) + (col ^ ((q ^ (q >> 4)) & 7)); }

// ---- class pass --------------------------------------------------------------------------------
// item = (line, r0): classes r0 .. r0 + 7 of `line`, rows q = 0..255 at element stride R.
// Slot = TMA box [256 rows][8 columns] with the 128-byte swizzle (16-byte unit u of row q at
// u ^ (q & 7)).  Thread t of a group: column col = t >> 4, lane-in-column beta / b = t & 15.
// The slot's coefficient area receives the line's levels jOff .. jOff + 7 and 1/e with the data.
template <int G, bool SYM>
__global__ void __launch_bounds__(G * kTC * 16, 1)
    pcr_cls_pipe_kernel(const __grid_constant__ CUtensorMap tm, const Geometry g, AlphaTables at,
                        double2 *__restrict__ X, const int *__restrict__ slots, int R, int jOff, int NS, int nitems) {
  constexpr int GT = kTC * 16;                       // 128 threads per group
  constexpr int SLOT = kNQ * kTC;                    // 2048 values = 32 KB
  extern __shared__ __align__(1024) unsigned char smraw_[];
  unsigned char *smraw = align_1024(smraw_);
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smraw + 64);
  double2 *coefs = reinterpret_cast<double2 *>(smraw + kHdrCoef);
  double2 *ring = reinterpret_cast<double2 *>(smraw + kHdrBytes);
  const int gid = threadIdx.x / GT, t = threadIdx.x - gid * GT;
  const int col = t >> 4, bb = t & 15;
  const int groups = R / kTC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      slot_item[s] = -1;
    }
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= nitems) return;
    const int line = it / groups, r0 = (it - line * groups) * kTC;
    const int tl = tline_of(g, slots, line);
    uint64_t *bar = full + k % NS;
    double2 *cf = coefs + (k % NS) * kCoefPerSlot;
    mbar_arrive_expect_tx(bar, (unsigned)((SLOT + kCoefPerSlot) * sizeof(double2)));
    tma_load_3d(ring + (size_t)(k % NS) * SLOT, &tm, 2 * r0, 0, line, bar);
    bulk_g2s(cf, at.pcr + ((size_t)tl * g.logN + jOff) * 2, 16 * sizeof(double2), bar);
    bulk_g2s(cf + 16, at.inv_e + tl, sizeof(double2), bar);
    slot_item[k % NS] = k;
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  for (int k = gid;; k += G) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= nitems) break;
    const int line = it / groups, r0 = (it - line * groups) * kTC;
    double2 *slot = ring + (size_t)(k % NS) * SLOT;
    const double2 *cf = coefs + (k % NS) * kCoefPerSlot;
    slot_wait(full + k % NS, slot_item, k, NS);
    double2 y[kE];
    // class arrangement: q = beta + 16 k (TMA swizzle: unit col ^ (q & 7))
#pragma unroll
    for (int kk = 0; kk < kE; ++kk) {
      const int q = bb + 16 * kk;
      y[kk] = slot[(q << 3) + (col ^ (q & 7))];
    }
    {
      double2 p = cf[8], q = cf[9];
      cyc_level<1, false, SYM>(y, p, q);
      p = cf[10], q = cf[11];
      cyc_level<2, false, SYM>(y, p, q);
      p = cf[12], q = cf[13];
      cyc_level<4, false, SYM>(y, p, q);
      p = cf[14];
      cyc_level<8, true, SYM>(y, p, p);   // h = N/2: the pair level
    }
    bar_sync(1 + gid, GT);   // the group's reads of the TMA layout are done
#pragma unroll
    for (int kk = 0; kk < kE; ++kk) slot[cls_sw(bb + 16 * kk, col)] = y[kk];
    bar_sync(1 + gid, GT);
#pragma unroll
    for (int e = 0; e < kE; ++e) y[e] = slot[cls_sw(16 * bb + e, col)];
    double2 c0[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c0[i] = cf[i];
    const double2 ie = cf[16];
    fence_proxy_async_smem();   // generic reads of the slot before the refill's async writes
    bar_sync(1 + gid, GT);
    if (t == 0) issue(k + NS);
    // class-pass levels are j >= jOff >= 5: symmetric in SYM mode (sg = 1)
    blk_level<1, SYM>(y, bb, c0[0], c0[1], 1.0);
    blk_level<2, SYM>(y, bb, c0[2], c0[3], 1.0);
    blk_level<4, SYM>(y, bb, c0[4], c0[5], 1.0);
    blk_level<8, SYM>(y, bb, c0[6], c0[7], 1.0);
    double2 *xl = X + (size_t)line * g.N + r0 + col;
#pragma unroll
    for (int e = 0; e < kE; ++e) xl[(size_t)(16 * bb + e) * R] = cmul(y[e], ie);
  }
}

// ---- chunk pass --------------------------------------------------------------------------------
// item = (line, chunk c): tile position p in [0, CT = CC + 512) holds line point c CC - 256 + p
// (mod N).  Levels j = 0 .. jA - 1 (h = 2^j <= 128).  Comb arrangement: B = t >> 4, beta = t & 15,
// p = 256 B + beta + 16 e.  Block arrangement: p = 16 t + e at swizzled positions
// chk_sw(p) = p ^ ((p >> 4) & 7) (conflict-free for both arrangements).
__device__ __forceinline__ int chk_sw(int p) { return p ^ ((p >> 4) & 7); }

// comb level: shift S in e (stride 16 S); neighbours' teeth read from natural positions p -/+ 16 S
template <int S, int CT, bool SYM>
__device__ __forceinline__ void comb_level(double2 (&y)[kE], const double2 *tile, int p0, double2 p, double2 q,
                                           double sg) {
  constexpr int h = 16 * S;
  double2 nv[kE];
#pragma unroll
  for (int e = 0; e < kE; ++e) {
    const int pe = p0 + 16 * e;
    const double2 lv = e >= S ? y[e - S] : tile[pe - h >= 0 ? pe - h : pe];
    const double2 rv = e + S < kE ? y[e + S] : tile[pe + h < CT ? pe + h : pe];
    nv[e] = upd<SYM>(p, q, sg, lv, rv, y[e]);
  }
#pragma unroll
  for (int e = 0; e < kE; ++e) y[e] = nv[e];
}
// block level: stride H < 16 on p = 16 t + e; neighbours' edge values from swizzled positions
template <int H, int CT, bool SYM>
__device__ __forceinline__ void chunk_blk_level(double2 (&y)[kE], const double2 *tile, int t, double2 p, double2 q,
                                                double sg) {
  double2 nv[kE];
#pragma unroll
  for (int e = 0; e < kE; ++e) {
    const int pe = 16 * t + e;
    const double2 lv = e >= H ? y[e - H] : tile[chk_sw(pe - H >= 0 ? pe - H : pe)];
    const double2 rv = e + H < kE ? y[e + H] : tile[chk_sw(pe + H < CT ? pe + H : pe)];
    nv[e] = upd<SYM>(p, q, sg, lv, rv, y[e]);
  }
#pragma unroll
  for (int e = 0; e < kE; ++e) y[e] = nv[e];
}

// Exchanges ping-pong between the slot and a second buffer of the group: a level reads its
// neighbours' values from `src` and publishes the edge values the next level needs into `dst`
// (comb: natural positions; block: swizzled), one group barrier, then the buffers swap roles.  A
// write to a buffer always follows the barrier after which every read of it is complete.
template <int S, int CT>
__device__ __forceinline__ void comb_publish(const double2 (&y)[kE], double2 *dst, int p0) {
#pragma unroll
  for (int e = 0; e < kE; ++e)
    if (e < S || e >= kE - S) dst[p0 + 16 * e] = y[e];
}
template <int H>
__device__ __forceinline__ void blk_publish(const double2 (&y)[kE], double2 *dst, int t) {
#pragma unroll
  for (int e = 0; e < kE; ++e)
    if (e < H || e >= kE - H) dst[chk_sw(16 * t + e)] = y[e];
}

template <int CC, int G, bool SYM>
__global__ void __launch_bounds__(G * (CC + 2 * kCH) / kE, 1)
    pcr_chunk_pipe_kernel(const Geometry g, AlphaTables at, const double2 *__restrict__ X, double2 *__restrict__ Y,
                          const int *__restrict__ slots, int jA, int NS, int nitems) {
  constexpr int CT = CC + 2 * kCH, GT = CT / kE;
  extern __shared__ __align__(1024) unsigned char smraw_[];
  unsigned char *smraw = align_1024(smraw_);
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  volatile int *slot_item = reinterpret_cast<volatile int *>(smraw + 64);
  double2 *coefs = reinterpret_cast<double2 *>(smraw + kHdrCoef);
  double2 *ring = reinterpret_cast<double2 *>(smraw + kHdrBytes);
  const int gid = threadIdx.x / GT, t = threadIdx.x - gid * GT;
  const int B = t >> 4, beta = t & 15;
  const int N = g.N;
  const int chunks = N / CC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      slot_item[s] = -1;
    }
    mbar_init_fence();
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= nitems) return;
    const int line = it / chunks, c = it - line * chunks;
    const int tl = tline_of(g, slots, line);
    const double2 *xl = X + (size_t)line * N;
    uint64_t *bar = full + k % NS;
    double2 *dst = ring + (size_t)(k % NS) * CT;
    mbar_arrive_expect_tx(bar, (unsigned)((CT + 2 * jA) * sizeof(double2)));
    const int start = c * CC - kCH;
    if (start < 0) {   // wrap at the line start
      bulk_g2s(dst, xl + N + start, (unsigned)(-start * sizeof(double2)), bar);
      bulk_g2s(dst - start, xl, (unsigned)((CT + start) * sizeof(double2)), bar);
    } else if (start + CT > N) {   // wrap at the line end
      const int n1 = N - start;
      bulk_g2s(dst, xl + start, (unsigned)(n1 * sizeof(double2)), bar);
      bulk_g2s(dst + n1, xl, (unsigned)((CT - n1) * sizeof(double2)), bar);
    } else {
      bulk_g2s(dst, xl + start, (unsigned)(CT * sizeof(double2)), bar);
    }
    bulk_g2s(coefs + (k % NS) * kCoefPerSlot, at.pcr + (size_t)tl * g.logN * 2, (unsigned)(2 * jA * sizeof(double2)), bar);
    slot_item[k % NS] = k;
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NS; ++k) issue(k);
  const int gbar = 1 + gid;
  const int p0 = 256 * B + beta;
  double2 *edge = ring + (size_t)NS * CT + (size_t)gid * CT;   // the group's second exchange buffer
  for (int k = gid;; k += G) {
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= nitems) break;
    const int line = it / chunks, c = it - line * chunks;
    double2 *tile = ring + (size_t)(k % NS) * CT;
    const double2 *cf = coefs + (k % NS) * kCoefPerSlot;
    slot_wait(full + k % NS, slot_item, k, NS);
    double2 y[kE];
#pragma unroll
    for (int e = 0; e < kE; ++e) y[e] = tile[p0 + 16 * e];
    const double2 *src = tile;
    double2 *dst = edge;
    auto flip = [&]() {
      bar_sync(gbar, GT);
      double2 *tmp = const_cast<double2 *>(src);
      src = dst;
      dst = tmp;
    };
    // comb levels j = 4 .. jA - 1 (h = 16 .. 128); the first reads the loaded tile as is
    if (jA > 4) {
      comb_level<1, CT, SYM>(y, src, p0, cf[8], cf[9], 1.0);
      if (jA > 5) { comb_publish<2, CT>(y, dst, p0); flip(); }
    }
    if (jA > 5) {
      comb_level<2, CT, SYM>(y, src, p0, cf[10], cf[11], 1.0);
      if (jA > 6) { comb_publish<4, CT>(y, dst, p0); flip(); }
    }
    if (jA > 6) {
      comb_level<4, CT, SYM>(y, src, p0, cf[12], cf[13], 1.0);
      if (jA > 7) { comb_publish<8, CT>(y, dst, p0); flip(); }
    }
    if (jA > 7) comb_level<8, CT, SYM>(y, src, p0, cf[14], cf[15], 1.0);
    // transposition comb -> block (swizzled positions) into the buffer nobody reads now
#pragma unroll
    for (int e = 0; e < kE; ++e) dst[chk_sw(p0 + 16 * e)] = y[e];
    flip();
#pragma unroll
    for (int e = 0; e < kE; ++e) y[e] = src[chk_sw(16 * t + e)];
    // block levels j = 0 .. min(jA, 4) - 1 (h = 1 .. 8); the first reads the transposed values
    if (jA > 0) {
      const double2 p = cf[0], q = cf[1];
      chunk_blk_level<1, CT, SYM>(y, src, t, p, q, (p.x != q.x || p.y != q.y) ? -1.0 : 1.0);
      if (jA > 1) { blk_publish<2>(y, dst, t); flip(); }
    }
    if (jA > 1) {
      chunk_blk_level<2, CT, SYM>(y, src, t, cf[2], cf[3], 1.0);
      if (jA > 2) { blk_publish<4>(y, dst, t); flip(); }
    }
    if (jA > 2) {
      chunk_blk_level<4, CT, SYM>(y, src, t, cf[4], cf[5], 1.0);
      if (jA > 3) { blk_publish<8>(y, dst, t); flip(); }
    }
    if (jA > 3) chunk_blk_level<8, CT, SYM>(y, src, t, cf[6], cf[7], 1.0);
    // transposition block -> comb for coalesced stores of the core (blocks B = 1 .. CC/256)
#pragma unroll
    for (int e = 0; e < kE; ++e) dst[chk_sw(16 * t + e)] = y[e];
    flip();
#pragma unroll
    for (int e = 0; e < kE; ++e) y[e] = src[chk_sw(p0 + 16 * e)];
    fence_proxy_async_smem();
    bar_sync(gbar, GT);
    if (t == 0) issue(k + NS);
    if (B >= 1 && B <= CC / 256) {
      double2 *yl = Y + (size_t)line * N + (size_t)c * CC - kCH;
#pragma unroll
      for (int e = 0; e < kE; ++e) yl[p0 + 16 * e] = y[e];
    }
  }
}

constexpr int kClsG = 2, kClsNS = 4;              // class pass: 2 groups of 128 threads, 4 x 32 KB slots
constexpr int kChkCC = 2048, kChkG = 2, kChkNS = 3;  // chunk pass: 2 groups of 160 threads, 3 x 40 KB slots
                                                     // + a 40 KB exchange buffer per group

}  // namespace

void *tma_encode_fn() {
  static void *fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = ptr;
  }
  return fn;
}

bool pcr1d_pipe_supported(const Geometry &g, int R) {
  return g.dim == 1 && g.pow2 && g.nfac == 1 && g.N >= 8192 && g.N <= 65536 && g.N == kNQ * R && R >= 32 &&
         kCH >= R - 1;
}

cudaError_t launch_pcr1d_pipe(const Geometry &g, const AlphaTables &at, double2 *X, double2 *Y, const int *slots,
                              int lines, int R, cudaStream_t s, int sm_reserve) {
  if (!pcr1d_pipe_supported(g, R)) return cudaErrorNotSupported;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sm_reserve > 0 && sms > 2 * sm_reserve) sms -= sm_reserve;   // NCCL ranks: leave SMs to the comm kernels
  const int jA = __builtin_ctz((unsigned)R);
  const bool sym = g.op == 0 || g.op == 1;   // centred 3-point heat / advection (see upd)
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_fn());
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tm;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)2 * R, (cuuint64_t)kNQ, (cuuint64_t)lines};
    const cuuint64_t strides[2] = {(cuuint64_t)R * 16, (cuuint64_t)g.N * 16};
    const cuuint32_t box[3] = {2 * kTC, kNQ, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return cudaErrorNotSupported;
  }
  cudaError_t e;
  {
    const size_t smem = 1024 + kHdrBytes + (size_t)kClsNS * kNQ * kTC * sizeof(double2);
    const void *fn = sym ? (const void *)pcr_cls_pipe_kernel<kClsG, true> : (const void *)pcr_cls_pipe_kernel<kClsG, false>;
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
    const int nitems = lines * (R / kTC);
    if (sym) pcr_cls_pipe_kernel<kClsG, true><<<sms, kClsG * kTC * 16, smem, s>>>(tm, g, at, X, slots, R, jA, kClsNS, nitems);
    else pcr_cls_pipe_kernel<kClsG, false><<<sms, kClsG * kTC * 16, smem, s>>>(tm, g, at, X, slots, R, jA, kClsNS, nitems);
    record_launch(s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  {
    constexpr int CT = kChkCC + 2 * kCH;
    const size_t smem = 1024 + kHdrBytes + (size_t)(kChkNS + kChkG) * CT * sizeof(double2);
    const void *fn = sym ? (const void *)pcr_chunk_pipe_kernel<kChkCC, kChkG, true>
                         : (const void *)pcr_chunk_pipe_kernel<kChkCC, kChkG, false>;
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
    const int nitems = lines * (g.N / kChkCC);
    if (sym)
      pcr_chunk_pipe_kernel<kChkCC, kChkG, true><<<sms, kChkG * CT / kE, smem, s>>>(g, at, X, Y, slots, jA, kChkNS, nitems);
    else
      pcr_chunk_pipe_kernel<kChkCC, kChkG, false><<<sms, kChkG * CT / kE, smem, s>>>(g, at, X, Y, slots, jA, kChkNS, nitems);
    record_launch(s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace pint
