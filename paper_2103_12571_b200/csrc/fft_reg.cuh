// Register-resident radix-16 FFT engine for power-of-two lines of N = 2^LOGN complex fp64
// values, 4 <= N <= 4096 (time axis L, spatial axes nx, ny).
//
// Plan: N = R0 R1 R2 with R_i = 2^{B_i}, B0 = min(4, LOGN), B1 = min(4, LOGN - B0), B2 = rest
// (at most 3 passes).  A line is handled by TPL = N / E threads, E = R0 values per thread.  Pass i
// works on blocks of m_i = N / (R0..R_{i-1}) positions at stride s_i = m_i / R_i: butterfly
// g = tau + TPL u (u < E / R_i) is (block beta = g / s_i, offset j = g % s_i) and owns positions
// beta m_i + j + s_i t, t < R_i.  DIF pass: in-register radix-R DFT (slot t receives frequency
// bitrev(t)), then slot t *= w_{m_i}^{j bitrev(t)}; the product over the passes leaves frequency
// bitrev_N(P) at position P (natural in, bit-reversed out: the order the paper keeps).
// The inverse (DIT) pass undoes a DIF pass on the same position sets (conjugate twiddle, then the
// inverse radix-R DFT from bit-reversed slots), passes in reverse order, unnormalised (N x).
//
// Between passes the values go through shared memory (one write, one barrier, one read per
// pass); a radix-2/4 third pass runs across lanes with warp shuffles instead (SHL).  Element P of a line lives at swizzled offset F(P): F XORs the low three 16-byte slot
// bits with higher position bits so that every quarter-warp access of every pass of the plan is
// bank-conflict free (tests/test_fft_plan.py checks it).  Twiddles: per-pass tables of the
// powers tw_i[k s_i + j] = w_{m_i}^{j 2^k}, k < B_i (host long double, staged in shared memory,
// lanes read consecutive j or broadcast); the other exponents j r are formed in registers by a
// short product chain from the nearest power of two below r (<= 7 complex products, error a few
// ulp), which trades 11 of 15 shared-memory loads per radix-16 butterfly for fp64 work.
// Exchanges synchronise only the threads of one line (warp or named barrier), never the CTA.
#pragma once
#include "device_common.cuh"

namespace pint {
namespace rfft {

__host__ __device__ constexpr int ilog2_ct(int r) { return r <= 1 ? 0 : 1 + ilog2_ct(r >> 1); }

template <int LOGN_, int MAXB = 4>
struct Plan {
  static constexpr int LOGN = LOGN_;
  static constexpr int N = 1 << LOGN;
  static constexpr int B0 = LOGN < MAXB ? LOGN : MAXB;
  static constexpr int B1 = (LOGN - B0) < MAXB ? (LOGN - B0) : MAXB;
  static constexpr int B2 = LOGN - B0 - B1;
  static_assert(B2 <= MAXB, "plan needs more than three passes");
  static constexpr int NP = B2 > 0 ? 3 : (B1 > 0 ? 2 : 1);
  static constexpr int E = 1 << B0;
  static constexpr int TPL = N / E;
  static constexpr int BL = NP == 3 ? B2 : (NP == 2 ? B1 : B0);   // radix (log2) of the last pass
  // Option: three-pass plans with a radix-2/4 last pass can run it across the 2^B2 lanes that hold
  // one block (warp shuffles, values stay at their pass-1 positions), saving the third shared-memory
  // exchange.  Parity-green, but measured slower on config 5 (spatial2d 89 vs 79-84 ms: the shuffle
  // window costs ~500 B of register spills at the 128-register cap), so it is off.
  static constexpr bool SHL = false && NP == 3 && B2 <= 2;
  static constexpr int b(int p) { return p == 0 ? B0 : (p == 1 ? B1 : B2); }
  static constexpr int logm(int p) { return p == 0 ? LOGN : (p == 1 ? LOGN - B0 : LOGN - B0 - B1); }
  static constexpr int logs(int p) { return logm(p) - b(p); }
  static constexpr int twcount(int p) { return b(p) << logs(p); }
  static constexpr int twoff(int p) { return p == 0 ? 0 : (p == 1 ? twcount(0) : twcount(0) + twcount(1)); }
  static constexpr int twsize() {
    return twcount(0) + (NP > 1 ? twcount(1) : 0) + (NP > 2 ? twcount(2) : 0);
  }
};

// swizzled offset of position p inside a line (see header)
template <class P>
__device__ __forceinline__ int F(int p) {
  int h = 0;
  if constexpr (P::NP >= 2) {
    constexpr int bl = P::BL;
    constexpr int sh = bl > 3 ? bl : 3;
    constexpr int mk = bl >= 3 ? 7 : ((1 << bl) - 1);
    h ^= (p >> sh) & mk;
  }
  if constexpr (P::NP == 3 && P::B2 < 3) {
    constexpr int lm1 = P::logm(1);
    h ^= ((p >> lm1) & ((8 >> P::B2) - 1)) << P::B2;
  }
  return p ^ h;
}

// position of value (u, t) of thread tau in pass PASS
template <class P, int PASS>
__device__ __forceinline__ int pos(int tau, int u, int t) {
  constexpr int lm = P::logm(PASS), ls = P::logs(PASS);
  const int g = tau + P::TPL * u;
  return ((g >> ls) << lm) + (g & ((1 << ls) - 1)) + (t << ls);
}

template <class P, int PASS>
__device__ __forceinline__ void to_smem(const double2 (&v)[P::E], double2 *line, int tau) {
  constexpr int R = 1 << P::b(PASS);
#pragma unroll
  for (int u = 0; u < P::E / R; ++u)
#pragma unroll
    for (int t = 0; t < R; ++t) line[F<P>(pos<P, PASS>(tau, u, t))] = v[u * R + t];
}

template <class P, int PASS>
__device__ __forceinline__ void from_smem(double2 (&v)[P::E], const double2 *line, int tau) {
  constexpr int R = 1 << P::b(PASS);
#pragma unroll
  for (int u = 0; u < P::E / R; ++u)
#pragma unroll
    for (int t = 0; t < R; ++t) v[u * R + t] = line[F<P>(pos<P, PASS>(tau, u, t))];
}

// slot t of a radix-2^B butterfly carries frequency bitrev_B(t), i.e. exponent r = brev(t);
// multiply every slot by w^{j r} (CONJ: w^{-j r}) with w^{j 2^k} = tp[k s].  Within each block
// [hb, 2 hb) the other powers come from two interleaved product chains (even and odd offsets,
// step w^{2j}): depth <= hb / 2 and five live values, error a few ulp.
template <int B, bool CONJ>
__device__ __forceinline__ void apply_twiddles(double2 *x, const double2 *tp, int s) {
  constexpr int R = 1 << B;
  auto ld = [&](int k) {
    double2 w = tp[k * s];
    if (CONJ) w.y = -w.y;
    return w;
  };
  const double2 w1 = ld(0);
  x[brev_ct<B>(1)] = cmul(x[brev_ct<B>(1)], w1);
  if constexpr (B >= 2) {
    const double2 w2 = ld(1);
    x[brev_ct<B>(2)] = cmul(x[brev_ct<B>(2)], w2);
    x[brev_ct<B>(3)] = cmul(x[brev_ct<B>(3)], cmul(w2, w1));
#pragma unroll
    for (int k = 2; k < B; ++k) {
      const int hb = 1 << k;
      const double2 wh = ld(k);
      double2 we = wh, wo = cmul(wh, w1);
#pragma unroll
      for (int o = 0; o < hb; o += 2) {
        if (o > 0) {
          we = cmul(we, w2);
          wo = cmul(wo, w2);
        }
        x[brev_ct<B>(hb + o)] = cmul(x[brev_ct<B>(hb + o)], we);
        x[brev_ct<B>(hb + o + 1)] = cmul(x[brev_ct<B>(hb + o + 1)], wo);
      }
    }
  }
  (void)R;
}

// DIF pass PASS on the thread's values; tw = the plan's twiddle table (shared memory)
template <class P, int PASS>
__device__ __forceinline__ void dif(double2 (&v)[P::E], int tau, const double2 *tw) {
  constexpr int b = P::b(PASS), R = 1 << b, ls = P::logs(PASS), s = 1 << ls;
#pragma unroll
  for (int u = 0; u < P::E / R; ++u) {
    reg_dif<b>(v + u * R);
    if constexpr (ls > 0) {
      const int j = (tau + P::TPL * u) & (s - 1);
      apply_twiddles<b, false>(v + u * R, tw + P::twoff(PASS) + j, s);
    }
  }
}

// inverse (DIT) of DIF pass PASS: conjugate twiddles, then the inverse radix-R DFT
template <class P, int PASS>
__device__ __forceinline__ void dit(double2 (&v)[P::E], int tau, const double2 *tw) {
  constexpr int b = P::b(PASS), R = 1 << b, ls = P::logs(PASS), s = 1 << ls;
#pragma unroll
  for (int u = 0; u < P::E / R; ++u) {
    if constexpr (ls > 0) {
      const int j = (tau + P::TPL * u) & (s - 1);
      apply_twiddles<b, true>(v + u * R, tw + P::twoff(PASS) + j, s);
    }
    reg_dit_inv<b>(v + u * R);
  }
}

// barrier over the TPL threads of line l (TPL <= 32: the warp; else named barrier 1 + l)
template <class P>
__device__ __forceinline__ void line_sync(int l) {
  constexpr int TPL = P::TPL;
  if constexpr (TPL <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + l), "r"(TPL) : "memory");
  }
}

// SHL plans: the last pass (radix R = 2^B2, blocks of R consecutive positions) across the R lanes
// j = tau mod R that hold one block (pass 1 left position beta m1 + j + R t in lane (beta, j),
// value t).  DIF stage with half h: the lower lane keeps a + b, the upper (b_partner - own) w_{2h}^e
// (e = j mod h); after the stages lane j holds the block's DFT at bitrev(j), i.e. exactly what the
// shared-memory pass leaves at that position.  lane_dit undoes it (conjugate twiddle, unnormalised).
template <class P>
__device__ __forceinline__ void lane_dif(double2 (&v)[P::E], int tau) {
  constexpr int BR = P::B2;
  const int j = tau & ((1 << BR) - 1);
#pragma unroll
  for (int st = 0; st < BR; ++st) {
    const int h = (1 << BR) >> (st + 1);
    const bool low = (j & h) == 0;
    const bool rot = h == 2 && (j & 1);   // w_4^1 = -i (only non-trivial twiddle for R <= 4)
#pragma unroll
    for (int t0 = 0; t0 < P::E; t0 += 4) {
#pragma unroll
      for (int t = t0; t < t0 + 4; ++t) {
        double2 r;
        r.x = __shfl_xor_sync(0xffffffffu, v[t].x, h);
        r.y = __shfl_xor_sync(0xffffffffu, v[t].y, h);
        if (low) {
          v[t] = cadd(v[t], r);
        } else {
          const double2 d = csub(r, v[t]);
          v[t] = rot ? make_double2(d.y, -d.x) : d;
        }
      }
      asm volatile("" ::: "memory");   // bound the shuffle window (register pressure)
    }
  }
}
template <class P>
__device__ __forceinline__ void lane_dit(double2 (&v)[P::E], int tau) {
  constexpr int BR = P::B2;
  const int j = tau & ((1 << BR) - 1);
#pragma unroll
  for (int st = BR - 1; st >= 0; --st) {
    const int h = (1 << BR) >> (st + 1);
    const bool low = (j & h) == 0;
    const bool rot = h == 2 && (j & 1);   // conj(w_4^1) = +i
#pragma unroll
    for (int t0 = 0; t0 < P::E; t0 += 4) {
#pragma unroll
      for (int t = t0; t < t0 + 4; ++t) {
        double2 w = v[t];
        if (!low && rot) w = make_double2(-w.y, w.x);
        double2 r;
        r.x = __shfl_xor_sync(0xffffffffu, w.x, h);
        r.y = __shfl_xor_sync(0xffffffffu, w.y, h);
        v[t] = low ? cadd(w, r) : csub(r, w);
      }
      asm volatile("" ::: "memory");
    }
  }
}

// Forward transform of a line whose values sit in shared memory at `line` (swizzled, natural
// order).  Returns with the values of the LAST pass in registers (positions pos<NP-1>).
// Contains NP - 1 exchanges; the first statement is a read, so the caller must have barriered
// after filling the line; ends without a trailing barrier.
template <class P>
__device__ __forceinline__ void forward_regs(double2 (&v)[P::E], double2 *line, int l, int tau,
                                             const double2 *tw) {
  // Exchanges need one barrier each: every thread writes pass i's values back to exactly the
  // positions pos<i>(tau, .) it read them from (from_smem<P, i>), so a write can never clobber a
  // position another thread of the line has still to read (the position sets of the threads are
  // disjoint); only the read of pass i + 1 must wait for all writes (RAW).
  dif<P, 0>(v, tau, tw);
  if constexpr (P::NP >= 2) {
    to_smem<P, 0>(v, line, tau);
    line_sync<P>(l);
    from_smem<P, 1>(v, line, tau);
    dif<P, 1>(v, tau, tw);
  }
  if constexpr (P::NP >= 3 && P::SHL) {
    lane_dif<P>(v, tau);
  } else if constexpr (P::NP >= 3) {
    to_smem<P, 1>(v, line, tau);
    line_sync<P>(l);
    from_smem<P, 2>(v, line, tau);
    dif<P, 2>(v, tau, tw);
  }
}
// forward_regs starting from pass-0 values that sit (natural order, swizzled) in `line`; the
// values must have been read from pos<0> positions of this thread (from_smem<P, 0> below), which
// is what makes the write-back of pass 0 barrier-free
template <class P>
__device__ __forceinline__ void forward_from_smem(double2 (&v)[P::E], double2 *line, int l, int tau,
                                                  const double2 *tw) {
  from_smem<P, 0>(v, line, tau);
  forward_regs<P>(v, line, l, tau, tw);
}

// Inverse transform starting from the last pass's positions in registers; ends with the values
// of pass 0 (natural positions tau + TPL t) in registers.  Uses `line` for the exchanges: the
// caller must make sure nobody still reads it, or that every thread's values came from its own
// last-pass positions of `line` (the forward transform), so that the first write-back clobbers
// nothing another thread still reads.  The last read (pass 0) is not followed by a barrier: a
// caller that writes `line` afterwards must write pos<P, 0> positions (to_smem<P, 0>) or sync.
template <class P>
__device__ __forceinline__ void inverse_in_regs(double2 (&v)[P::E], double2 *line, int l, int tau,
                                                const double2 *tw) {
  if constexpr (P::NP >= 3 && P::SHL) {
    lane_dit<P>(v, tau);
  } else if constexpr (P::NP >= 3) {
    dit<P, 2>(v, tau, tw);
    to_smem<P, 2>(v, line, tau);
    line_sync<P>(l);
    from_smem<P, 1>(v, line, tau);
  }
  if constexpr (P::NP >= 2) {
    dit<P, 1>(v, tau, tw);
    to_smem<P, 1>(v, line, tau);   // pos<1> positions: the ones this thread just read
    line_sync<P>(l);
    from_smem<P, 0>(v, line, tau);
  }
  dit<P, 0>(v, tau, tw);
}

// Natural position of pass-0 value t of thread tau: tau + TPL t.
template <class P>
__device__ __forceinline__ int natural_pos(int tau, int t) { return tau + P::TPL * t; }

// S-layout: storage slot of last-pass value (u, t) of thread tau in spectral (bit-reversed
// position) data kept in global memory: slot q = t * (N / R_L) + beta, beta = tau + TPL u; the
// lanes of a warp write consecutive slots.  slot_to_pos inverts it.
// (SHL plans: register i = u R_L + t stays at pass-1 position pos<1>(tau, 0, i); slot q = i TPL + tau.)
template <class P>
__device__ __forceinline__ int s_slot(int tau, int u, int t) {
  if constexpr (P::SHL) return ((u << P::BL) + t) * P::TPL + tau;   // register i = u R_L + t
  else return (t << (P::LOGN - P::BL)) + tau + P::TPL * u;
}
template <class P>
__device__ __forceinline__ int slot_to_pos(int q) {
  if constexpr (P::SHL) {
    return pos<P, 1>(q % P::TPL, 0, q / P::TPL);
  } else {
    constexpr int sh = P::LOGN - P::BL;
    return ((q & ((1 << sh) - 1)) << P::BL) + (q >> sh);
  }
}
// position of last-pass value (u, t) of thread tau (its frequency is bitrev_N of it)
template <class P>
__device__ __forceinline__ int last_pos(int tau, int u, int t) {
  if constexpr (P::SHL) return pos<P, 1>(tau, 0, (u << P::BL) + t);
  else return pos<P, P::NP - 1>(tau, u, t);
}

}  // namespace rfft
}  // namespace pint
